"""Shared test helpers: seeded problems on the GPU vs the fp64 oracle, normwise per-(b,h) errors.

Error metric (reading R11): for each output tensor and each (b,h) slice,
err = max_i |x_i - y_i| / max_i |y_i|; a test asserts the max over slices.  Elementwise relative error is not
used: it is meaningless on this operator (near-zero entries; d log alpha row 0 is exactly 0).
"""
import numpy as np
import torch

import oracle
import synth
from paper_2312_06635_b200 import binding as G


def nerr_slices(x, y):
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    B, H = y.shape[:2]
    xs = x.reshape(B * H, -1)
    ys = y.reshape(B * H, -1)
    den = np.maximum(np.max(np.abs(ys), axis=1), 1e-30)
    return float(np.max(np.max(np.abs(xs - ys), axis=1) / den))


def problem(B, H, T, K, V, seed=0, gate="std", dtype=torch.bfloat16, h0=False, dfinal=False):
    p = synth.problem(B, H, T, K, V, seed=seed, gate=gate, dtype=dtype)
    p["h0"] = synth.state(B, H, K, V, seed) if h0 else None
    p["dfinal"] = synth.state(B, H, K, V, seed + 1000, scale=0.5) if dfinal else None
    return p


def cuda(p):
    return {k: (v.cuda().contiguous() if isinstance(v, torch.Tensor) else v) for k, v in p.items()}


def f64(t):
    return None if t is None else t.double().numpy()


def oracle_fwd(p):
    return oracle.fwd(f64(p["q"]), f64(p["k"]), f64(p["v"]), f64(p["g"]), h0=f64(p["h0"]))


def oracle_bwd(p):
    return oracle.bwd(f64(p["q"]), f64(p["k"]), f64(p["v"]), f64(p["g"]), f64(p["do"]), h0=f64(p["h0"]),
                      d_final=f64(p["dfinal"]))


def gpu_fwd(pc, C, c, path):
    o, fs = G.chunk_fwd(pc["q"], pc["k"], pc["v"], pc["g"], C, c, pc["h0"], True, path)
    torch.cuda.synchronize()
    return o.float().cpu().numpy(), fs.cpu().numpy()


def gpu_bwd(pc, C, c, path):
    dq, dk, dv, dg, dh0 = G.chunk_bwd(pc["q"], pc["k"], pc["v"], pc["g"], pc["do"], C, c, pc["h0"], pc["dfinal"],
                                      True, path)
    torch.cuda.synchronize()
    return [t.float().cpu().numpy() for t in (dq, dk, dv, dg, dh0)]
