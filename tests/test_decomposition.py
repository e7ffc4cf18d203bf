"""The chunk-wise two-level decomposition (what the kernels implement) equals the recurrent oracle
in fp64.  Pins DESIGN.md's readings R1-R6 before any GPU code runs."""
import numpy as np
import pytest

import oracle
from tests.chunk_ref import chunk_bwd, chunk_fwd


def nerr(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("C,c,tau", [(16, 4, 16.0), (32, 16, 1.0), (16, 16, 4.0), (8, 1, 1.0)])
def test_chunk_forward_equals_oracle(C, c, tau):
    rng = np.random.default_rng(C * 100 + c)
    T, K, V = 64, 6, 5
    q, k, v = (rng.standard_normal((T, d)) for d in (K, K, V))
    g = -np.log1p(np.exp(-rng.standard_normal((T, K)))) / tau
    h0 = rng.standard_normal((K, V))
    o, H = chunk_fwd(q, k, v, g, C, c, h0)
    oo, fs = oracle.fwd(q[None, None], k[None, None], v[None, None], g[None, None], h0=h0[None, None])
    assert nerr(o, oo[0, 0]) < 1e-12
    assert nerr(H, fs[0, 0]) < 1e-12


def test_chunk_forward_extreme_gates_is_stable():
    """log alpha = -30: every exponent the decomposition forms is <= 0, outputs stay finite and equal
    <q_t,k_t> v_t (+ e^-30 corrections)."""
    rng = np.random.default_rng(1)
    T, K, V = 32, 4, 3
    q, k, v = (rng.standard_normal((T, d)) for d in (K, K, V))
    g = np.full((T, K), -30.0)
    o, _ = chunk_fwd(q, k, v, g, 16, 4)
    assert np.all(np.isfinite(o))
    diag = np.sum(q * k, axis=1)[:, None] * v
    assert nerr(o, diag) < 1e-11


@pytest.mark.parametrize("C,tau", [(16, 16.0), (8, 1.0), (32, 2.0)])
def test_chunk_backward_equals_oracle(C, tau):
    rng = np.random.default_rng(C)
    T, K, V = 64, 5, 4
    q, k, v, do = (rng.standard_normal((T, d)) for d in (K, K, V, V))
    g = -np.log1p(np.exp(-rng.standard_normal((T, K)))) / tau
    h0, dfin = rng.standard_normal((K, V)), rng.standard_normal((K, V))
    got = chunk_bwd(q, k, v, g, do, C, h0, dfin)
    ref = oracle.bwd(q[None, None], k[None, None], v[None, None], g[None, None], do[None, None],
                     h0=h0[None, None], d_final=dfin[None, None])
    for name, a, b in zip(("dq", "dk", "dv", "dg", "dh0"), got, ref):
        assert nerr(a, b[0, 0]) < 1e-11, name
