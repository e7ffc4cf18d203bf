"""fp64 numpy transcription of the chunk-wise two-level decomposition the CUDA kernels implement
(SURVEY App. A.1, A.2, A.5).  Test-only: it pins the
*readings* of the paper (chunk-local inclusive cumsum, state passing order, per-pair sub-chunk
normalisers, the backward and the d log alpha carry) against the recurrent oracle, before and
independently of any GPU code.  Per (b,h) unit, 0-based t, chunk i = rows [iC, iC+C).
"""
import numpy as np


def chunk_fwd(q, k, v, g, C, c, h0=None):
    T, K = q.shape
    V = v.shape[1]
    H = np.zeros((K, V)) if h0 is None else h0.copy()
    o = np.zeros((T, V))
    for i in range(T // C):
        sl = slice(i * C, (i + 1) * C)
        qi, ki, vi, gi = q[sl], k[sl], v[sl], g[sl]
        b = np.cumsum(gi, axis=0)                 # (a1) chunk-local inclusive log cumsum
        Gam = b[-1]                               # chunk total log decay
        # (a2) cross-chunk output with the state entering the chunk (P:257 first term)
        o[sl] = (qi * np.exp(b)) @ H
        # (a3) intra-chunk two-level: sub-chunk pairs
        P = np.zeros((C, C))
        n = C // c
        for x in range(n):
            tx = slice(x * c, (x + 1) * c)
            for y in range(x):
                ty = slice(y * c, (y + 1) * c)
                e_y = b[(y + 1) * c - 1]          # normaliser: b at the end of key sub-chunk y
                P[tx, ty] = (qi[tx] * np.exp(b[tx] - e_y)) @ (ki[ty] * np.exp(e_y - b[ty])).T
            for t in range(x * c, (x + 1) * c):   # diagonal block: per-element log space, s <= t
                for s in range(x * c, t + 1):
                    P[t, s] = np.sum(qi[t] * ki[s] * np.exp(b[t] - b[s]))
        o[sl] += P @ vi
        # (a2) state passing: H_{i+1} = e^Gam (.) H_i + (K (.) e^{Gam - b})^T V
        H = np.exp(Gam)[:, None] * H + (ki * np.exp(Gam - b)).T @ vi
    return o, H


def chunk_bwd(q, k, v, g, do, C, h0=None, dfin=None):
    """A.5: reverse state pass; dq/dk/dv inter + intra; d log alpha by the local carry
    rowsum(H_{i+1} (.) dH_{i+1}); returns (dq, dk, dv, dg, dh0)."""
    T, K = q.shape
    V = v.shape[1]
    NC = T // C
    Hs = [np.zeros((K, V)) if h0 is None else h0.copy()]
    bs = []
    for i in range(NC):
        sl = slice(i * C, (i + 1) * C)
        b = np.cumsum(g[sl], axis=0)
        bs.append(b)
        Hs.append(np.exp(b[-1])[:, None] * Hs[-1] + (k[sl] * np.exp(b[-1] - b)).T @ v[sl])
    dH = np.zeros((K, V)) if dfin is None else dfin.copy()
    dq, dk, dg = np.zeros((T, K)), np.zeros((T, K)), np.zeros((T, K))
    dv = np.zeros((T, V))
    M = np.tril(np.ones((C, C)))
    for i in reversed(range(NC)):
        sl = slice(i * C, (i + 1) * C)
        qi, ki, vi, doi, b = q[sl], k[sl], v[sl], do[sl], bs[i]
        Gam = b[-1]
        E = np.exp(b[:, None, :] - b[None, :, :]) * M[:, :, None]    # E[t,s,m] = e^{b_t - b_s}, s <= t
        P = np.einsum("tm,sm,tsm->ts", qi, ki, E)
        dP = (doi @ vi.T) * M
        dq[sl] = (doi @ Hs[i].T) * np.exp(b) + np.einsum("ts,sm,tsm->tm", dP, ki, E)
        dk[sl] = (vi @ dH.T) * np.exp(Gam - b) + np.einsum("ts,tm,tsm->sm", dP, qi, E)
        dv[sl] = P.T @ doi + (ki * np.exp(Gam - b)) @ dH
        x = qi * dq[sl] - ki * dk[sl]
        carry = np.sum(Hs[i + 1] * dH, axis=1)                     # rowsum(H_{i+1} (.) dH_{i+1})
        dg[sl] = np.flip(np.cumsum(np.flip(x, 0), 0), 0) + carry
        dH = np.exp(Gam)[:, None] * dH + (qi * np.exp(b)).T @ doi  # dH_i
    return dq, dk, dv, dg, dH
