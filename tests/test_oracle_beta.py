"""Pins for the general-gate fp64 oracle (oracle/gla_beta_oracle.c, G_t = alpha_t^T beta_t).
CPU only.  Each test checks it against something other than itself:
  * beta == 1 reduces it to the alpha-only oracle, itself pinned in tests/test_oracle.py;
  * the paper's parallel form with both gates, Eq. gla_QKV2 (Q~ = Q A, K~ = K/A, V~ = V/B,
    O = ((Q~ K~^T) (.) M) V~ (.) B), evaluated by brute force on tiny inputs;
  * the transposed recurrence: with alpha == 1, S^T follows the alpha-only recurrence with k and v swapped and
    log beta as the gate, so the final state is the alpha-only oracle's on (v, k, log beta), transposed;
  * beta == gamma (constant per value channel), alpha == 1: the value-side RetNet mask, closed form;
  * central finite differences for every gradient (dq, dk, dv, d log alpha, d log beta, dh0);
  * the d log beta identity: o depends on (v, log beta) only through v (.) e^{-LB} and the e^{LB} output factor,
    so d log beta_t = sum_{s >= t} (o_s (.) do_s - v_s (.) dv_s) + colsum(S_T (.) dS_T) at t = T.
A dropped gate, a gate on the wrong side, a wrong sign or a transposed operand fails at least one."""
import numpy as np
import pytest

import oracle


def rnd(shape, rng, scale=1.0):
    return rng.standard_normal(shape) * scale


def gates(shape, rng, tau=16.0):
    z = rng.standard_normal(shape)
    return -np.log1p(np.exp(-z)) / tau          # logsigmoid(z)/tau


def nerr(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def parallel_form_beta(q, k, v, ga, gb):
    """Eq. gla_QKV2 with both gates: A = prod alpha, B = prod beta."""
    A = np.exp(np.cumsum(ga, axis=-2))
    Bc = np.exp(np.cumsum(gb, axis=-2))
    T = q.shape[-2]
    M = np.tril(np.ones((T, T)))
    P = np.einsum("...tk,...sk->...ts", q * A, k / A) * M
    return np.einsum("...ts,...sv->...tv", P, v / Bc) * Bc


def problem(rng, B=1, H=2, T=24, K=5, V=6, tau=4.0):
    return (rnd((B, H, T, K), rng), rnd((B, H, T, K), rng), rnd((B, H, T, V), rng),
            gates((B, H, T, K), rng, tau), gates((B, H, T, V), rng, tau))


def test_beta_one_is_alpha_only_oracle():
    rng = np.random.default_rng(0)
    q, k, v, ga, _ = problem(rng)
    h0 = rnd((1, 2, 5, 6), rng)
    o1, f1 = oracle.fwd(q, k, v, ga, h0)
    o2, f2 = oracle.fwd_beta(q, k, v, ga, np.zeros_like(v), h0)
    assert nerr(o2, o1) < 1e-14 and nerr(f2, f1) < 1e-14
    do, df = rnd(v.shape, rng), rnd(h0.shape, rng)
    g1 = oracle.bwd(q, k, v, ga, do, h0, df)
    g2 = oracle.bwd_beta(q, k, v, ga, np.zeros_like(v), do, h0, df)
    for a, b in zip((g2[0], g2[1], g2[2], g2[3], g2[5]), g1):
        assert nerr(a, b) < 1e-13


def test_parallel_form_both_gates():
    rng = np.random.default_rng(1)
    q, k, v, ga, gb = problem(rng, T=20)
    o, _ = oracle.fwd_beta(q, k, v, ga, gb)
    assert nerr(o, parallel_form_beta(q, k, v, ga, gb)) < 1e-11


def test_transposed_recurrence_final_state():
    """alpha == 1: S_t^T = diag(beta_t) S_{t-1}^T + v_t^T k_t -- the alpha-only recurrence on (v, k, log beta)."""
    rng = np.random.default_rng(2)
    q, k, v, _, gb = problem(rng, T=30)
    _, fs = oracle.fwd_beta(q, k, v, np.zeros_like(q), gb)
    _, fsT = oracle.fwd(np.zeros_like(v), v, k, gb)      # state [V, K]
    assert nerr(fs, np.swapaxes(fsT, -1, -2)) < 1e-13


@pytest.mark.parametrize("gamma", [0.5, 0.9, 0.99])
def test_value_side_retnet_closed_form(gamma):
    """alpha == 1, beta_t[j] == gamma_j: o_t[j] = sum_{s<=t} gamma_j^{t-s} <q_t, k_s> v_s[j]."""
    rng = np.random.default_rng(3)
    q, k, v, _, _ = problem(rng, T=16, V=4)
    gam = gamma ** np.array([1.0, 0.5, 2.0, 1.5])
    gb = np.broadcast_to(np.log(gam), v.shape).copy()
    o, _ = oracle.fwd_beta(q, k, v, np.zeros_like(q), gb)
    T = q.shape[-2]
    ref = np.zeros_like(v)
    for t in range(T):
        for s in range(t + 1):
            ref[..., t, :] += np.sum(q[..., t, :] * k[..., s, :], axis=-1)[..., None] * gam ** (t - s) * v[..., s, :]
    assert nerr(o, ref) < 1e-13


def test_finite_differences_all_gradients():
    rng = np.random.default_rng(4)
    q, k, v, ga, gb = problem(rng, B=1, H=1, T=70, K=3, V=4, tau=2.0)   # crosses the 64-step checkpoint
    h0, df = rnd((1, 1, 3, 4), rng), rnd((1, 1, 3, 4), rng)
    do = rnd(v.shape, rng)

    def loss(q_, k_, v_, ga_, gb_, h0_):
        o, fs = oracle.fwd_beta(q_, k_, v_, ga_, gb_, h0_)
        return np.sum(o * do) + np.sum(fs * df)

    grads = oracle.bwd_beta(q, k, v, ga, gb, do, h0, df)
    args = [q, k, v, ga, gb, h0]
    h = 1e-6
    for gi, (ai, name) in enumerate(zip((0, 1, 2, 3, 4, 5), ("q", "k", "v", "la", "lb", "h0"))):
        x = args[ai]
        idx = [tuple(rng.integers(0, n) for n in x.shape) for _ in range(6)]
        for ix in idx:
            xp, xm = x.copy(), x.copy()
            xp[ix] += h
            xm[ix] -= h
            ap, am = list(args), list(args)
            ap[ai], am[ai] = xp, xm
            fd = (loss(*ap) - loss(*am)) / (2 * h)
            g = grads[gi][ix]
            assert abs(fd - g) <= 1e-5 * max(1.0, abs(fd)), (name, ix, fd, g)


def test_dlog_beta_identity():
    rng = np.random.default_rng(5)
    q, k, v, ga, gb = problem(rng, T=40)
    h0, df = rnd((1, 2, 5, 6), rng), rnd((1, 2, 5, 6), rng)
    do = rnd(v.shape, rng)
    o, fs = oracle.fwd_beta(q, k, v, ga, gb, h0)
    dq, dk, dv, dga, dgb, dh0 = oracle.bwd_beta(q, k, v, ga, gb, do, h0, df)
    dLB = o * do - v * dv
    dLB[..., -1, :] += np.sum(fs * df, axis=-2)
    ref = np.flip(np.cumsum(np.flip(dLB, -2), -2), -2)
    assert nerr(dgb, ref) < 1e-10
    # and the alpha-side identity still holds with beta present (q (.) e^{LA}, k (.) e^{-LA})
    dLA = q * dq - k * dk
    dLA[..., -1, :] += np.sum(fs * df, axis=-1)
    assert nerr(dga, np.flip(np.cumsum(np.flip(dLA, -2), -2), -2)) < 1e-10


def test_step_beta_matches_forward():
    rng = np.random.default_rng(6)
    q, k, v, ga, gb = problem(rng, T=9)
    o, fs = oracle.fwd_beta(q, k, v, ga, gb)
    st = np.zeros((1, 2, 5, 6))
    for t in range(9):
        ot, st = oracle.step_beta(q[:, :, t], k[:, :, t], v[:, :, t], ga[:, :, t], gb[:, :, t], st)
        assert nerr(ot, o[:, :, t]) < 1e-14
    assert nerr(st, fs) < 1e-14
