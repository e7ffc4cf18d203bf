"""Pins for the fp64 oracle (CPU only).  Each test checks the oracle against something OTHER than
itself: a different form of the same operator from the paper, a textbook special case, a hand-
evaluated example, finite differences, or a closed-form invariant.  A dropped term, a wrong sign,
an off-by-one in the gate index or a transposed operand in oracle/gla_oracle.c fails at least one.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "hand_examples.json")


def rnd(shape, rng, scale=1.0):
    return rng.standard_normal(shape) * scale


def gates(shape, rng, tau=16.0):
    z = rng.standard_normal(shape)
    return -np.log1p(np.exp(-z)) / tau          # logsigmoid(z)/tau


def semiring_form(q, k, v, g, h0=None):
    """Quadratic log-space parallel form, App. Eqs. genbmm_1/genbmm_2 with beta == 1:
    O_t = sum_{s<=t} (sum_m exp(LA_tm - LA_sm) q_tm k_sm) v_s   [+ (q_t * exp(LA_t)) h0]."""
    LA = np.cumsum(g, axis=-2)                    # A_t = prod_{j<=t} alpha_j, in log space
    T = q.shape[-2]
    out = np.zeros(q.shape[:-1] + (v.shape[-1],))
    for t in range(T):
        for s in range(t + 1):
            w = np.sum(np.exp(LA[..., t, :] - LA[..., s, :]) * q[..., t, :] * k[..., s, :], axis=-1)
            out[..., t, :] += w[..., None] * v[..., s, :]
    if h0 is not None:
        out += np.einsum("...tk,...kv->...tv", q * np.exp(LA), h0)
    return out


def parallel_form(q, k, v, g):
    """Eq. gla_QKV2: Q~ = Q*A, K~ = K/A, O = (Q~K~^T (.) M)V (beta == 1).  In range only."""
    A = np.exp(np.cumsum(g, axis=-2))
    T = q.shape[-2]
    M = np.tril(np.ones((T, T)))
    return np.einsum("...ts,...sv->...tv", np.einsum("...tk,...sk->...ts", q * A, k / A) * M, v)


def final_state_closed_form(k, v, g, h0=None):
    """S_T = sum_s (k_s * exp(LA_T - LA_s))^T v_s + exp(LA_T) (.) h0   (unfolded P:188)."""
    LA = np.cumsum(g, axis=-2)
    w = np.exp(LA[..., -1:, :] - LA) * k
    S = np.einsum("...tk,...tv->...kv", w, v)
    if h0 is not None:
        S += np.exp(LA[..., -1, :])[..., :, None] * h0
    return S


def nerr(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fwd_matches_semiring_and_parallel_forms(seed):
    rng = np.random.default_rng(seed)
    B, H, T, K, V = 2, 2, 24, 5, 7
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng, tau=2.0)
    o, fs = oracle.fwd(q, k, v, g)
    assert nerr(o, semiring_form(q, k, v, g)) < 1e-12
    assert nerr(o, parallel_form(q, k, v, g)) < 1e-10
    assert nerr(fs, final_state_closed_form(k, v, g)) < 1e-12


def test_fwd_with_initial_state():
    rng = np.random.default_rng(5)
    B, H, T, K, V = 1, 3, 16, 4, 6
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng, tau=1.0)
    h0 = rnd((B, H, K, V), rng)
    o, fs = oracle.fwd(q, k, v, g, h0=h0)
    assert nerr(o, semiring_form(q, k, v, g, h0)) < 1e-12
    assert nerr(fs, final_state_closed_form(k, v, g, h0)) < 1e-12


def test_alpha_one_is_linear_attention():
    """alpha == 1 -> unnormalised linear attention (QK^T (.) M)V."""
    rng = np.random.default_rng(7)
    B, H, T, K, V = 1, 2, 20, 6, 5
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    o, fs = oracle.fwd(q, k, v, np.zeros((B, H, T, K)))
    M = np.tril(np.ones((T, T)))
    ref = np.einsum("...ts,...sv->...tv", np.einsum("...tk,...sk->...ts", q, k) * M, v)
    assert nerr(o, ref) < 1e-13
    assert nerr(fs, np.einsum("...tk,...tv->...kv", k, v)) < 1e-13


@pytest.mark.parametrize("gamma", [0.5, 0.9, 0.99])
def test_constant_alpha_is_retnet(gamma):
    """alpha == gamma -> RetNet O = (QK^T (.) D)V, D_nm = gamma^(n-m)."""
    rng = np.random.default_rng(11)
    B, H, T, K, V = 1, 1, 18, 4, 3
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    o, _ = oracle.fwd(q, k, v, np.full((B, H, T, K), np.log(gamma)))
    n = np.arange(T)
    D = np.where(n[:, None] >= n[None, :], gamma ** (n[:, None] - n[None, :]).astype(float), 0.0)
    ref = np.einsum("...ts,...sv->...tv", np.einsum("...tk,...sk->...ts", q, k) * D, v)
    assert nerr(o, ref) < 1e-12


def test_length_one():
    """L = 1: O_1 = <q_1, k_1> v_1 (S_0 = 0)."""
    rng = np.random.default_rng(3)
    q, k, v = rnd((1, 1, 1, 8), rng), rnd((1, 1, 1, 8), rng), rnd((1, 1, 1, 5), rng)
    o, _ = oracle.fwd(q, k, v, gates((1, 1, 1, 8), rng))
    np.testing.assert_allclose(o[0, 0, 0], np.dot(q[0, 0, 0], k[0, 0, 0]) * v[0, 0, 0], rtol=1e-14)


def test_hand_examples():
    gold = json.load(open(GOLD))
    for c in gold["cases"]:
        shp = lambda x: np.asarray(x, float).reshape(1, 1, 2, 1)
        q, k, v, g = shp(c["q"]), shp(c["k"]), shp(c["v"]), shp(c["log_alpha"])
        if "o" in c:
            o, fs = oracle.fwd(q, k, v, g)
            np.testing.assert_allclose(o.ravel(), c["o"], rtol=1e-14)
            np.testing.assert_allclose(fs.ravel(), [c["final_state"]], rtol=1e-14)
        if "dq" in c:
            dq, dk, dv, dg, dh0 = oracle.bwd(q, k, v, g, shp(c["d_out"]))
            for name, val in (("dq", dq), ("dk", dk), ("dv", dv), ("dlog_alpha", dg)):
                np.testing.assert_allclose(val.ravel(), c[name], rtol=1e-14, atol=1e-15, err_msg=name)
            np.testing.assert_allclose(dh0.ravel(), [c["dh0"]], rtol=1e-14)
    ge = gold["gate_example"]
    assert abs(-np.log1p(np.exp(-ge["z"])) / 16.0 - ge["log_alpha"]) < 1e-16


def test_causality():
    """Perturbing inputs at t > t0 leaves outputs at t <= t0 bit-identical."""
    rng = np.random.default_rng(13)
    B, H, T, K, V = 1, 2, 16, 4, 4
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng)
    o1, _ = oracle.fwd(q, k, v, g)
    q2, k2, v2, g2 = q.copy(), k.copy(), v.copy(), g.copy()
    for a in (q2, k2, v2, g2):
        a[..., 9:, :] += 1.0
    o2, _ = oracle.fwd(q2, k2, v2, g2)
    assert np.array_equal(o1[..., :9, :], o2[..., :9, :])
    assert not np.array_equal(o1[..., 9:, :], o2[..., 9:, :])


def _loss(q, k, v, g, h0, do, dfin):
    o, fs = oracle.fwd(q, k, v, g, h0=h0)
    return float(np.sum(o * do) + np.sum(fs * dfin))


def test_bwd_matches_central_finite_differences():
    """Hand backward vs central differences, h = 1e-6."""
    rng = np.random.default_rng(17)
    B, H, T, K, V = 1, 1, 70, 3, 4   # T > 64 crosses an oracle checkpoint boundary
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng, tau=4.0)
    h0, do, dfin = rnd((B, H, K, V), rng), rnd((B, H, T, V), rng), rnd((B, H, K, V), rng)
    grads = oracle.bwd(q, k, v, g, do, h0=h0, d_final=dfin)
    names = ("q", "k", "v", "g", "h0")
    arrs = [q, k, v, g, h0]
    h = 1e-6
    pick = np.random.default_rng(0)
    for name, arr, grad in zip(names, arrs, grads):
        idx = [tuple(pick.integers(0, s) for s in arr.shape) for _ in range(12)]
        for ix in idx:
            arr[ix] += h
            lp = _loss(*arrs[:4], arrs[4], do, dfin)
            arr[ix] -= 2 * h
            lm = _loss(*arrs[:4], arrs[4], do, dfin)
            arr[ix] += h
            fd = (lp - lm) / (2 * h)
            tol = 1e-4 if name == "g" else 1e-5
            assert abs(fd - grad[ix]) <= tol * max(abs(fd), abs(grad[ix]), 1.0), (name, ix, fd, grad[ix])


def test_bwd_invariants():
    """Closed-form invariants of the gradients:
    (1) with h0 = 0, d log alpha_1 == 0 exactly (alpha_1 only scales S_0 = 0);
    (2) with h0 = 0 and d_final = 0, per channel sum_t q*dq == sum_t k*dk (o is invariant under
        q -> q*c, k -> k/c per channel);
    (3) d log alpha_t == sum_{s>=t} (q*dq - k*dk)_s + [t == T] * rowsum(S_T (.) dS_T)."""
    rng = np.random.default_rng(19)
    B, H, T, K, V = 2, 1, 40, 5, 3
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng, tau=2.0)
    do = rnd((B, H, T, V), rng)
    dq, dk, dv, dg, dh0 = oracle.bwd(q, k, v, g, do)
    assert np.all(dg[..., 0, :] == 0.0)
    lhs, rhs = np.sum(q * dq, axis=-2), np.sum(k * dk, axis=-2)
    assert nerr(lhs, rhs) < 1e-12
    dfin = rnd((B, H, K, V), rng)
    h0 = rnd((B, H, K, V), rng)
    dq, dk, dv, dg, dh0 = oracle.bwd(q, k, v, g, do, h0=h0, d_final=dfin)
    _, fs = oracle.fwd(q, k, v, g, h0=h0)
    x = q * dq - k * dk
    rc = np.flip(np.cumsum(np.flip(x, -2), -2), -2)
    rc = rc + np.sum(fs * dfin, axis=-1)[..., None, :]   # S_T = e^{LA_T} (.) (...): final-state term
    assert nerr(dg, rc) < 1e-11


def test_step_matches_fwd():
    """T decode steps == one fwd call (output and final state)."""
    rng = np.random.default_rng(23)
    B, H, T, K, V = 2, 2, 9, 4, 6
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng)
    o, fs = oracle.fwd(q, k, v, g)
    st = np.zeros((B, H, K, V))
    for t in range(T):
        ot, st = oracle.step(q[:, :, t], k[:, :, t], v[:, :, t], g[:, :, t], st)
        assert nerr(ot, o[:, :, t]) < 1e-13
    assert nerr(st, fs) < 1e-13


def test_threading_is_deterministic():
    rng = np.random.default_rng(29)
    B, H, T, K, V = 3, 2, 33, 4, 5
    q, k, v = rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng)
    g = gates((B, H, T, K), rng)
    do = rnd((B, H, T, V), rng)
    a = oracle.bwd(q, k, v, g, do, nthreads=1)
    b = oracle.bwd(q, k, v, g, do, nthreads=4)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
