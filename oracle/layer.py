"""fp64 CPU oracle of the full multi-head GLA layer.  TEST INFRASTRUCTURE ONLY (same rules as
``oracle/__init__.py``: only tests/, smoke() and bench.py's baseline legs may use it).

Written step by step from the paper, beta == 1:
    P:298-301  per head h:  S^h_t = G^h_t (.) S^h_{t-1} + K^h_t^T V^h_t,  O^h_t = Q^h_t S^h_t   -> ``oracle.fwd``
    P:302      O'_t = concat(LN(O^1_t), ..., LN(O^H_t))           (LayerNorm per head, RetNet-style; a per-channel
                                                                  affine ln_w, ln_b -- reading L1 in DESIGN.md)
    P:304      R_t = Swish(X_t W_r + b_r)
    P:305      Y_t = (R_t (.) O'_t) W_O
    P:322-325  alpha = sigma(X W_a1 W_a2 + b_a)^{1/tau}, i.e. log alpha = logsigmoid(X W_a1 W_a2 + b_a) / tau
               (the log-space temperature of P:177's footnote; reading L2), rank 16
    P:325      d_k = d/2, d_v = d, full-rank W_Q, W_K, W_V, W_O, W_r
The backward is the chain rule of these steps written out by hand (the core's part is ``oracle.bwd``); it is
pinned against central finite differences in tests/test_layer.py.
"""
from __future__ import annotations

import numpy as np

from . import bwd as core_bwd
from . import fwd as core_fwd


def _logsigmoid(z):
    return np.minimum(z, 0.0) - np.log1p(np.exp(-np.abs(z)))


def _sigmoid(z):
    return 1.0 / (1.0 + np.exp(-z))


def _heads(x, H):          # [B, T, H*D] -> [B, H, T, D]
    B, T, HD = x.shape
    return x.reshape(B, T, H, HD // H).transpose(0, 2, 1, 3)


def _unheads(x):           # [B, H, T, D] -> [B, T, H*D]
    B, H, T, D = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B, T, H * D)


def layer_fwd(x, W_qkvr, W_a1, W_a2, b_alpha, b_r, ln_w, ln_b, W_o, H, tau=16.0, eps=1e-5):
    """y [B,T,d] and a cache for layer_bwd.  All arrays fp64; W_qkvr = [W_Q | W_K | W_V | W_r]."""
    dk, dv = W_a2.shape[1], W_o.shape[0]
    P = x @ W_qkvr
    q, k, v, r = P[..., :dk], P[..., dk:2 * dk], P[..., 2 * dk:2 * dk + dv], P[..., 2 * dk + dv:]
    lr = x @ W_a1
    z = lr @ W_a2 + b_alpha
    g = _logsigmoid(z) / tau                                   # P:322-325 with P:177
    qh, kh, vh, gh = _heads(q, H), _heads(k, H), _heads(v, H), _heads(g, H)
    O, _ = core_fwd(qh, kh, vh, gh)
    mu = O.mean(-1, keepdims=True)
    var = ((O - mu) ** 2).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    n = (O - mu) * rstd                                        # LN per head
    a = _unheads(n) * ln_w + ln_b
    rr = r + b_r
    sw = rr * _sigmoid(rr)                                     # Swish
    Zo = a * sw
    y = Zo @ W_o
    cache = dict(x=x, P=P, qh=qh, kh=kh, vh=vh, gh=gh, z=z, lr=lr, n=n, rstd=rstd, a=a, rr=rr, sw=sw, Zo=Zo,
                 H=H, tau=tau, dk=dk, dv=dv)
    return y, cache


def layer_bwd(dy, cache, W_qkvr, W_a1, W_a2, b_alpha, b_r, ln_w, ln_b, W_o):
    """Gradients of <y, dy> w.r.t. (x, W_qkvr, W_a1, W_a2, b_alpha, b_r, ln_w, ln_b, W_o), fp64."""
    c = cache
    H, tau, dk, dv = c["H"], c["tau"], c["dk"], c["dv"]
    x, Zo = c["x"], c["Zo"]
    B, T, d = x.shape
    flat = lambda a: a.reshape(B * T, -1)                     # noqa: E731
    dW_o = flat(Zo).T @ flat(dy)
    dZ = dy @ W_o.T
    rr, sw, a = c["rr"], c["sw"], c["a"]
    sg = _sigmoid(rr)
    da = dZ * sw
    drr = dZ * a * sg * (1.0 + rr * (1.0 - sg))               # d Swish(r) / dr
    d_b_r = drr.sum((0, 1))
    n = c["n"]
    nf = _unheads(n)
    d_ln_w = (da * nf).sum((0, 1))
    d_ln_b = da.sum((0, 1))
    dn = _heads(da * ln_w, H)
    dO = c["rstd"] * (dn - dn.mean(-1, keepdims=True) - n * (dn * n).mean(-1, keepdims=True))
    dq, dk_, dv_, dg, _ = core_bwd(c["qh"], c["kh"], c["vh"], c["gh"], dO)
    dz = _unheads(dg) * _sigmoid(-c["z"]) / tau               # d logsigmoid(z) / dz = sigmoid(-z)
    d_b_alpha = dz.sum((0, 1))
    dW_a2 = flat(c["lr"]).T @ flat(dz)
    dlr = dz @ W_a2.T
    dW_a1 = flat(x).T @ flat(dlr)
    dP = np.concatenate([_unheads(dq), _unheads(dk_), _unheads(dv_), drr], axis=-1)
    dW_qkvr = flat(x).T @ flat(dP)
    dx = dP @ W_qkvr.T + dlr @ W_a1.T
    return dict(x=dx, W_qkvr=dW_qkvr, W_a1=dW_a1, W_a2=dW_a2, b_alpha=d_b_alpha, b_r=d_b_r, ln_w=d_ln_w,
                ln_b=d_ln_b, W_o=dW_o, b_alpha_abs=np.abs(dz).sum((0, 1)))
