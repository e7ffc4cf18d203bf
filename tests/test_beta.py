"""The general outer-product gate G_t = alpha_t^T beta_t through the C ABI (gla_chunk_fwd_beta /
gla_chunk_bwd_beta / gla_recurrent_step_beta) vs the fp64 two-gate oracle (oracle/gla_beta_oracle.c, pinned in
tests/test_oracle_beta.py) on identical seeded inputs.  Normwise per-(b,h) errors (R11): 1e-5 for fp32
inputs (the fp32 CUDA-core path), 2e-2 for bf16 inputs.  CPU-side: the ABI validation of the new entry points."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_06635_b200 import binding as G
from tests.helpers import nerr_slices


def beta_problem(B, H, T, K, V, seed=0, gate="std", beta_gate="std", dtype=torch.float32, h0=False, dfinal=False):
    p = synth.problem(B, H, T, K, V, seed=seed, gate=gate, dtype=dtype)
    p["lb"] = synth.gates(beta_gate, B, H, T, V, seed=seed + 77)
    p["h0"] = synth.state(B, H, K, V, seed) if h0 else None
    p["dfinal"] = synth.state(B, H, K, V, seed + 1000, scale=0.5) if dfinal else None
    return p


def f64(t):
    return None if t is None else t.double().numpy()


def run_gpu(p, C, c):
    d = {n: (t.cuda().contiguous() if isinstance(t, torch.Tensor) else t) for n, t in p.items()}
    o, fs = G.chunk_fwd_beta(d["q"], d["k"], d["v"], d["g"], d["lb"], C, c, d["h0"], True)
    grads = G.chunk_bwd_beta(d["q"], d["k"], d["v"], d["g"], d["lb"], d["do"], C, c, d["h0"], d["dfinal"], True)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), fs.cpu().numpy(), [g.float().cpu().numpy() for g in grads]


def run_oracle(p):
    a = [f64(p[n]) for n in ("q", "k", "v", "g", "lb")]
    o, fs = oracle.fwd_beta(*a, h0=f64(p["h0"]))
    grads = oracle.bwd_beta(*a, f64(p["do"]), h0=f64(p["h0"]), d_final=f64(p["dfinal"]))
    return o, fs, grads


NAMES = ("dq", "dk", "dv", "dlog_alpha", "dlog_beta", "dh0")


def check(p, C, c, tol):
    o, fs, g = run_gpu(p, C, c)
    ro, rfs, rg = run_oracle(p)
    errs = {"o": nerr_slices(o, ro), "final_state": nerr_slices(fs, rfs)}
    for n, a, b in zip(NAMES, g, rg):
        assert np.all(np.isfinite(a)), n
        errs[n] = nerr_slices(a, b)
    print("beta", p.get("gate_kind", "std"), C, c, " ".join(f"{n}={e:.2e}" for n, e in errs.items()))
    bad = {n: e for n, e in errs.items() if not e < tol}
    assert not bad, bad


@pytest.mark.gpu
@pytest.mark.parametrize("C,c", [(16, 4), (32, 8), (64, 16), (8, 8)])
def test_beta_fp32_chunk_plans(C, c):
    check(beta_problem(2, 2, 128, 32, 48, seed=1, h0=True, dfinal=True), C, c, 1e-5)


@pytest.mark.gpu
@pytest.mark.parametrize("gate,beta_gate", [("std", "std"), ("strong", "strong"), ("ones", "std"), ("std", "ones"),
                                            ("mixed", "const"), ("near1", "strong")])
def test_beta_fp32_gate_distributions(gate, beta_gate):
    check(beta_problem(1, 2, 192, 64, 64, seed=3, gate=gate, beta_gate=beta_gate, h0=True, dfinal=True), 64, 16, 1e-5)


@pytest.mark.gpu
def test_beta_bf16_inputs_340m_head():
    """bf16 inputs at a 340M-shaped head (K=128, V=256), T = 512 (several chunks, several V tiles)."""
    check(beta_problem(1, 2, 512, 128, 256, seed=5, dtype=torch.bfloat16, dfinal=True), 64, 16, 2e-2)


@pytest.mark.gpu
def test_beta_ones_equals_alpha_only_path():
    """log beta = 0: the two-gate entry points reproduce gla_chunk_fwd / gla_chunk_bwd on the SIMT path."""
    p = beta_problem(1, 2, 128, 32, 64, seed=7, h0=True, dfinal=True)
    p["lb"] = torch.zeros_like(p["lb"])
    d = {n: (t.cuda() if isinstance(t, torch.Tensor) else t) for n, t in p.items()}
    o1, f1 = G.chunk_fwd(d["q"], d["k"], d["v"], d["g"], 32, 8, d["h0"], True, "simt")
    o2, f2 = G.chunk_fwd_beta(d["q"], d["k"], d["v"], d["g"], d["lb"], 32, 8, d["h0"], True)
    assert torch.allclose(o1, o2, rtol=1e-6, atol=1e-6) and torch.allclose(f1, f2, rtol=1e-6, atol=1e-6)
    g1 = G.chunk_bwd(d["q"], d["k"], d["v"], d["g"], d["do"], 32, 8, d["h0"], d["dfinal"], True, "simt")
    g2 = G.chunk_bwd_beta(d["q"], d["k"], d["v"], d["g"], d["lb"], d["do"], 32, 8, d["h0"], d["dfinal"], True)
    for a, b in zip((g2[0], g2[1], g2[2], g2[3], g2[5]), g1):
        assert nerr_slices(a.cpu().numpy(), b.cpu().numpy()) < 1e-5


@pytest.mark.gpu
def test_beta_decode_steps_match_oracle():
    B, H, K, V, T = 2, 2, 64, 96, 12
    p = beta_problem(B, H, T, K, V, seed=9, dtype=torch.float32)
    d = {n: (t.cuda() if isinstance(t, torch.Tensor) else t) for n, t in p.items()}
    st = torch.zeros(B, H, K, V, device="cuda")
    rst = np.zeros((B, H, K, V))
    for t in range(T):
        o = G.recurrent_step_beta(*(d[n][:, :, t].contiguous() for n in ("q", "k", "v", "g", "lb")), st)
        ro, rst = oracle.step_beta(*(f64(p[n][:, :, t]) for n in ("q", "k", "v", "g", "lb")), rst)
        assert nerr_slices(o.cpu().numpy(), ro) < 1e-5
    assert nerr_slices(st.cpu().numpy(), rst) < 1e-5


def test_beta_abi_validation_no_launch():
    """CPU: the two-gate entry points validate before any launch (TC path refused, plan errors, workspace)."""
    L = G.lib()
    d = G._Desc(1, 1, 64, 16, 32, 16, 4, G.FP32, G.FP32, G.PATHS["tc"])
    assert L.gla_chunk_fwd_beta(ctypes.byref(d), *([None] * 9), 0, None) == 6      # GLA_ERR_UNSUPPORTED
    d = G._Desc(1, 1, 60, 16, 32, 16, 4, G.FP32, G.FP32, G.PATHS["simt"])
    assert L.gla_chunk_fwd_beta(ctypes.byref(d), *([None] * 9), 0, None) == 2      # GLA_ERR_PLAN (16 does not divide 60)
    d = G._Desc(1, 1, 64, 16, 32, 16, 4, G.FP32, G.FP32, G.PATHS["simt"])
    assert L.gla_chunk_bwd_beta(ctypes.byref(d), *([None] * 15), 0, None) == 5     # GLA_ERR_NULL
    assert L.gla_beta_workspace_size(ctypes.byref(d)) > 0
