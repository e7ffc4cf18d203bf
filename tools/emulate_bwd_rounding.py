"""Emulates the tensor-core backward's rounding points in numpy (fp32 compute, bf16 roundings where the
kernels round) to attribute the d log alpha error.  python tools/emulate_bwd_rounding.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402


def bf(x):
    return torch.from_numpy(np.asarray(x, np.float32)).bfloat16().float().numpy().astype(np.float64)


def run(q, k, v, g, do, C, R, excl=False):
    """R: set of names rounded to bf16: 'qk' (Q~,K~ operands), 'sb' (state copies), 'dp' (dP, P), 'part' (partials)."""
    T, K = q.shape
    V = v.shape[1]
    NC = T // C
    r_ = lambda name, x: bf(x) if name in R else x
    H = np.zeros((K, V)); Hs = [H]
    bs = []
    for i in range(NC):
        sl = slice(i * C, (i + 1) * C)
        b = np.cumsum(g[sl], 0); bs.append(b)
        rr = b[C // 2 - 1]
        Kt = r_('qk', k[sl] * np.exp(rr - b))
        H = np.exp(b[-1] - rr)[:, None] * (np.exp(rr)[:, None] * H + Kt.T @ v[sl])
        Hs.append(H)
    dq = np.zeros((T, K)); dk = np.zeros((T, K)); dH = np.zeros((K, V))
    xq = np.zeros((T, K)); xk = np.zeros((T, K))
    M = np.tril(np.ones((C, C)))
    for i in reversed(range(NC)):
        sl = slice(i * C, (i + 1) * C)
        b = bs[i]; rr = b[C // 2 - 1]; G = b[-1]
        Qt = r_('qk', q[sl] * np.exp(b - rr)); Kt = r_('qk', k[sl] * np.exp(rr - b))
        SB = r_('sb', (np.exp(rr)[:, None] * Hs[i]).T)          # [V][K]
        dHt = np.exp(G - rr)[:, None] * dH
        dSB = r_('sb', dHt.T)
        dPf = (do[sl] @ v[sl].T) * M
        dP = r_('dp', dPf * (np.tril(np.ones((C, C)), -1) if excl else 1.0))
        dPd = np.diag(dPf)
        dqp = r_('part', do[sl] @ SB + dP @ Kt)
        dkp = r_('part', v[sl] @ dSB + dP.T @ Qt)
        dq[sl] = np.exp(b - rr) * dqp
        dk[sl] = np.exp(rr - b) * dkp
        if excl:
            xq[sl] = dq[sl].copy(); xk[sl] = dk[sl].copy()
            dq[sl] += dPd[:, None] * k[sl]
            dk[sl] += dPd[:, None] * q[sl]
        dH = np.exp(rr)[:, None] * (dHt + Qt.T @ do[sl])
    x = (q * xq - k * xk) if excl else (q * dq - k * dk)
    dg = np.flip(np.cumsum(np.flip(x, 0), 0), 0)
    return dq, dk, dg


def nerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


T, K, V, C = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 64, 128, 64
p = synth.problem(1, 1, T, K, V, seed=1)
f = {n: p[n][0, 0].double().numpy() for n in p}
rdq, rdk, rdv, rdg, _ = oracle.bwd(*(p[n].double().numpy() for n in ("q", "k", "v", "g", "do")))
rdq, rdk, rdg = rdq[0, 0], rdk[0, 0], rdg[0, 0]
for excl in (False, True):
    for R in [{"qk"}, {"part"}, {"qk", "sb", "dp", "part"}, {"qk", "sb", "dp"}]:
        dq, dk, dg = run(f["q"], f["k"], f["v"], f["g"], f["do"], C, R, excl)
        print(f"T={T} excl_diag={excl} bf16 at {sorted(R)!s:36s} dq {nerr(dq, rdq):.2e} dk {nerr(dk, rdk):.2e} "
              f"dlogalpha {nerr(dg, rdg):.2e}")
