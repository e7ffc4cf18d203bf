"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle on identical seeded inputs.

Tolerances (north_star / DESIGN.md R11): normwise per (b,h) slice, 1e-5 for the fp32 SIMT ("debug")
path with fp32 inputs, 2e-2 for bf16 inputs with fp32 accumulation.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2312_06635_b200 import binding as G
from tests.helpers import cuda, gpu_bwd, gpu_fwd, nerr_slices, oracle_bwd, oracle_fwd, problem

pytestmark = pytest.mark.gpu

F32_TOL = 1e-5
BF16_TOL = 2e-2
NAMES = ("dq", "dk", "dv", "dlog_alpha", "dh0")


def check_fwd(p, C, c, path, tol):
    o, fs = gpu_fwd(cuda(p), C, c, path)
    ro, rfs = oracle_fwd(p)
    assert np.all(np.isfinite(o)) and np.all(np.isfinite(fs))
    eo, ef = nerr_slices(o, ro), nerr_slices(fs, rfs)
    assert eo < tol, ("o", eo)
    assert ef < tol, ("final_state", ef)
    return eo, ef


def dg_scale(p, ref):
    """Per-slice scale of d log alpha's defining terms q.dq and k.dk (R12): d log alpha is the
    reverse cumsum of (q.dq - k.dk) (plus a final-state term), so its rounding error is bounded relative to
    these summands, not to the (possibly e^-30-small) result."""
    q, k = p["q"].double().numpy(), p["k"].double().numpy()
    a = np.abs(q * ref[0]).reshape(q.shape[0] * q.shape[1], -1).max(1)
    b = np.abs(k * ref[1]).reshape(q.shape[0] * q.shape[1], -1).max(1)
    return np.maximum(a, b)


def check_bwd(p, C, c, path, tol):
    return check_bwd_outputs(p, gpu_bwd(cuda(p), C, c, path), path, tol)


def check_bwd_outputs(p, got, path, tol):
    """got = (dq, dk, dv, d log alpha, dh0) as numpy arrays, checked against the fp64 oracle."""
    ref = oracle_bwd(p)
    errs = {}
    for n, a, b in zip(NAMES, got, ref):
        assert np.all(np.isfinite(a)), n
        errs[n] = nerr_slices(a, b)
    # d log alpha: error relative to max(|d log alpha|, |q.dq|, |k.dk|) per slice
    a, b = got[3].astype(np.float64), ref[3]
    BH = b.shape[0] * b.shape[1]
    den = np.maximum(np.abs(b).reshape(BH, -1).max(1), dg_scale(p, ref))
    errs["dlog_alpha"] = float(np.max(np.abs(a - b).reshape(BH, -1).max(1) / den))
    errs["dlog_alpha_strict"] = nerr_slices(a, b)
    print(f"check_bwd path={path} gate={p.get('gate_kind', 'std')} " +
          " ".join(f"{n}={e:.2e}" for n, e in errs.items()))
    bad = {n: e for n, e in errs.items() if e >= tol and n != "dlog_alpha_strict"}
    assert not bad, bad
    # The plain normwise bar holds for every gate except `extreme` (log alpha = -30): there the true d log alpha
    # is ~1e-13 while its defining summands q.dq, k.dk are O(1) (ratio ~1e13, measured with the oracle), so only
    # the summand-relative bar above is meaningful (R12).
    if p.get("gate_kind") != "extreme":
        assert errs["dlog_alpha_strict"] < tol, errs
    return errs


# ---- fp32 SIMT path ("fp32 debug build"), tolerance 1e-5 -------------------------------------------------
@pytest.mark.parametrize("C,c", [(16, 4), (16, 16), (16, 1), (64, 16), (32, 8)])
def test_simt_fwd_tiny_config(C, c):
    """BJ config 1: B=1, H=1, T=64, d_k=16, d_v=32, chunk 16, fp32."""
    p = problem(1, 1, 64, 16, 32, seed=0, dtype=torch.float32)
    check_fwd(p, C, c, "simt", F32_TOL)


@pytest.mark.parametrize("gate", synth.GATES)
def test_simt_fwd_gate_distributions(gate):
    p = problem(2, 2, 128, 40, 72, seed=1, gate=gate, dtype=torch.float32, h0=True)   # ragged K/V tiles
    check_fwd(p, 64, 16, "simt", F32_TOL)


@pytest.mark.parametrize("gate", ["std", "strong", "extreme", "ones"])
def test_simt_bwd(gate):
    p = problem(2, 1, 128, 48, 80, seed=2, gate=gate, dtype=torch.float32, h0=True, dfinal=True)
    p["gate_kind"] = gate
    check_bwd(p, 32, 8, "simt", F32_TOL)


def test_simt_bwd_tiny_config():
    p = problem(1, 1, 64, 16, 32, seed=3, dtype=torch.float32)
    check_bwd(p, 16, 4, "simt", F32_TOL)


# ---- bf16 inputs ---------------------------------------------------------------------------------------
@pytest.mark.parametrize("path", ["simt", "auto"])
@pytest.mark.parametrize("gate", ["std", "strong", "extreme"])
def test_bf16_fwd_bwd_340m_heads(path, gate):
    """340M per-head shapes (K=128, V=256), several chunks."""
    p = problem(1, 2, 256, 128, 256, seed=4, gate=gate, dtype=torch.bfloat16, h0=True, dfinal=True)
    p["gate_kind"] = gate
    check_fwd(p, 64, 16, path, BF16_TOL)
    check_bwd(p, 64, 16, path, BF16_TOL)


@pytest.mark.parametrize("path", ["simt", "auto"])
def test_bf16_fwd_bwd_1p3b_heads(path):
    """1.3B per-head shapes (K=256, V=512)."""
    p = problem(1, 2, 192, 256, 512, seed=5, dtype=torch.bfloat16)
    check_fwd(p, 64, 16, path, BF16_TOL)
    check_bwd(p, 64, 16, path, BF16_TOL)


def test_bf16_gates():
    p = problem(1, 2, 128, 64, 128, seed=6, dtype=torch.bfloat16)
    p["g"] = p["g"].to(torch.bfloat16)
    check_fwd(p, 64, 16, "auto", BF16_TOL)
    check_bwd(p, 64, 16, "auto", BF16_TOL)


# ---- decode, segments, determinism ---------------------------------------------------------------------
@pytest.mark.parametrize("dtype,tol,B,H,T,K,V", [(torch.float32, F32_TOL, 2, 2, 64, 64, 96),
                                                  (torch.bfloat16, BF16_TOL, 2, 2, 64, 64, 96),
                                                  (torch.bfloat16, BF16_TOL, 80, 4, 8, 32, 256),    # wide tiles
                                                  (torch.bfloat16, BF16_TOL, 16, 4, 8, 64, 128),    # narrow tiles
                                                  (torch.bfloat16, BF16_TOL, 1, 4, 16, 256, 512)])  # B = 1 decode shape
def test_recurrent_step_matches_oracle_and_chunk_fwd(dtype, tol, B, H, T, K, V):
    p = problem(B, H, T, K, V, seed=7, dtype=dtype, h0=True)
    pc = cuda(p)
    st = pc["h0"].clone()
    outs = []
    for t in range(T):
        outs.append(G.recurrent_step(pc["q"][:, :, t].contiguous(), pc["k"][:, :, t].contiguous(),
                                     pc["v"][:, :, t].contiguous(), pc["g"][:, :, t].contiguous(), st))
    o = torch.stack(outs, 2).float().cpu().numpy()
    ro, rfs = oracle_fwd(p)
    assert nerr_slices(o, ro) < tol
    assert nerr_slices(st.cpu().numpy(), rfs) < tol


def test_state_summary_and_combine():
    B, H, T, K, V = 2, 2, 128, 32, 64
    p = problem(B, H, T, K, V, seed=8, dtype=torch.float32)
    pc = cuda(p)
    S, D = G.state_summary(pc["k"], pc["v"], pc["g"], 32, 8)
    _, rfs = oracle.fwd(p["q"].double().numpy(), p["k"].double().numpy(), p["v"].double().numpy(),
                        p["g"].double().numpy())
    assert nerr_slices(S.cpu().numpy(), rfs) < F32_TOL
    np.testing.assert_allclose(D.cpu().numpy(), p["g"].double().sum(2).numpy(), rtol=1e-5, atol=1e-5)
    h = synth.state(B, H, K, V, 3).cuda()
    out = G.state_combine(h, D, S)
    ref = np.exp(D.double().cpu().numpy())[..., None] * h.double().cpu().numpy() + S.double().cpu().numpy()
    assert nerr_slices(out.cpu().numpy(), ref) < 1e-6
    dh = G.dstate_summary(pc["q"], pc["do"], pc["g"], 32, 8)
    rdh = oracle.bwd(*(p[n].double().numpy() for n in ("q", "k", "v", "g", "do")))[4]
    assert nerr_slices(dh.cpu().numpy(), rdh) < F32_TOL


def test_two_segment_scan_equals_single_pass():
    """Sequence split in two segments: summary -> combine -> fwd(h0) reproduces the single pass."""
    B, H, T, K, V = 1, 2, 256, 64, 64
    p = problem(B, H, T, K, V, seed=9, dtype=torch.float32)
    pc = cuda(p)
    h = T // 2
    seg = [{n: pc[n][:, :, s].contiguous() for n in ("q", "k", "v", "g")} for s in (slice(0, h), slice(h, T))]
    S0, D0 = G.state_summary(seg[0]["k"], seg[0]["v"], seg[0]["g"], 64, 16)
    H1 = G.state_combine(torch.zeros_like(S0), D0, S0)
    o1, _ = G.chunk_fwd(seg[1]["q"], seg[1]["k"], seg[1]["v"], seg[1]["g"], 64, 16, H1, False, "simt")
    ro, _ = oracle_fwd(p)
    assert nerr_slices(o1.cpu().numpy(), ro[:, :, h:]) < F32_TOL


@pytest.mark.parametrize("path", ["simt", "auto"])
def test_deterministic(path):
    p = cuda(problem(1, 2, 128, 64, 128, seed=10))
    a = G.chunk_fwd(p["q"], p["k"], p["v"], p["g"], 64, 16, None, True, path)
    b = G.chunk_fwd(p["q"], p["k"], p["v"], p["g"], 64, 16, None, True, path)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    ga = G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 64, 16, path=path)
    gb = G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 64, 16, path=path)
    for x, y in zip(ga[:4], gb[:4]):
        assert torch.equal(x, y)


def test_zero_length_and_empty():
    q = torch.zeros(1, 2, 0, 16, device="cuda")
    v = torch.zeros(1, 2, 0, 32, device="cuda")
    h0 = torch.randn(1, 2, 16, 32, device="cuda")
    o, fs = G.chunk_fwd(q, q, v, q, 16, 4, h0, True, "simt")
    assert o.numel() == 0 and torch.equal(fs, h0)


def test_autograd_wrapper():
    p = cuda(problem(1, 1, 64, 32, 64, seed=11, dtype=torch.float32))
    q, k, v, g = (p[n].clone().requires_grad_(True) for n in ("q", "k", "v", "g"))
    o, fs = G.gla(q, k, v, g, None, 16, 4, "simt")
    (o * p["do"]).sum().backward()
    dq, dk, dv, dg, _ = G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 16, 4, path="simt")
    assert torch.equal(q.grad, dq) and torch.equal(g.grad, dg)


# ---- chunk sizes beyond the tensor-core path's 64 (the f4 sweep's plans), fp32 SIMT ------------------------
@pytest.mark.parametrize("C,c", [(128, 16), (128, 128), (128, 32), (8, 2)])
def test_simt_large_and_small_chunks(C, c):
    p = problem(1, 2, 256, 64, 128, seed=4, dtype=torch.float32, h0=True, dfinal=True)
    check_fwd(p, C, c, "simt", F32_TOL)
    check_bwd(p, C, c, "simt", F32_TOL)
