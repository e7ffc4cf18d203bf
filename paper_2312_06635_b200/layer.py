"""A full multi-head GLA layer around the chunk-wise core.

P:298-307 (multi-head GLA layer) and P:321-326 (parameter allocation), beta == 1:
    Q = x W_Q, K = x W_K, V = x W_V                       (d -> d_k, d_k, d_v; d_k = d/2, d_v = d)
    log alpha = logsigmoid(x W_a1 W_a2 + b_a) / tau        (low-rank, rank 16; tau = 16, P:177 footnote)
    O^h = GLA(Q^h, K^h, V^h, alpha^h)                       (the tensor-core core, gla_chunk_fwd / _bwd_saved)
    O'  = concat_h LN(O^h)                                  (LayerNorm per head; per-channel affine)
    R   = Swish(x W_r + b_r);   y = (R (.) O') W_O
The projections are plain GEMMs (cuBLAS through torch.matmul, bf16); x W_Q | x W_K | x W_V | x W_r is one GEMM
against the concatenated weight.  Everything between the GEMMs runs in the library's kernels: the transpose
into the core's [B,H,T,D] layout fused with the gate's logsigmoid (gla_layer_prep), the core, and the per-head
LayerNorm fused with the Swish gate and the transpose back (gla_layer_out), and their backward kernels.
"""
from __future__ import annotations

import math

import torch

from . import binding as G


class _LayerCore(torch.autograd.Function):
    """(P, z_alpha, b_alpha, b_r, ln_w, ln_b) -> Z = (LN(GLA(...)) * ln_w + ln_b) (.) Swish(r + b_r)."""

    @staticmethod
    def forward(ctx, P, Za, b_alpha, b_r, ln_w, ln_b, cfg):
        H, K, V, tau, eps, chunk, subchunk, path = cfg
        q, k, v, g = G.layer_prep(P, Za, b_alpha, H, K, V, tau)
        ws = G.fwd_workspace(q, v, g, chunk, subchunk, path)
        O, _ = G.chunk_fwd(q, k, v, g, chunk, subchunk, None, False, path, workspace=ws)
        r_off = 2 * H * K + H * V
        Z, mean, rstd = G.layer_out(O, P, r_off, b_r, ln_w, ln_b, eps)
        ctx.save_for_backward(P, Za, b_alpha, b_r, ln_w, ln_b, q, k, v, g, O, mean, rstd)
        ctx.ws, ctx.cfg = ws, cfg
        return Z

    @staticmethod
    def backward(ctx, dZ):
        P, Za, b_alpha, b_r, ln_w, ln_b, q, k, v, g, O, mean, rstd = ctx.saved_tensors
        H, K, V, tau, eps, chunk, subchunk, path = ctx.cfg
        B, T = P.shape[:2]
        r_off = 2 * H * K + H * V
        dP = torch.zeros_like(P) if P.shape[-1] > 2 * H * K + 2 * H * V else torch.empty_like(P)
        wsb = G.layer_bwd_workspace(B, T, H, K, V, P.device)
        dO, d_ln_w, d_ln_b, d_b_r = G.layer_out_bwd(dZ.contiguous(), O, P, r_off, b_r, ln_w, ln_b, mean, rstd, dP, wsb)
        dq, dk, dv, dg, _ = G.chunk_bwd(q, k, v, g, dO, chunk, subchunk, path=path, fwd_workspace=ctx.ws)
        ctx.ws = None
        dZa, d_b_alpha = G.layer_prep_bwd(dq, dk, dv, dg, Za, b_alpha, dP, tau, wsb)
        return dP, dZa, d_b_alpha, d_b_r, d_ln_w, d_ln_b, None


class GLALayer(torch.nn.Module):
    """Multi-head GLA layer (beta == 1) with the paper's parameter allocation: d_k = d/2, d_v = d, rank-16 gate."""

    def __init__(self, d_model: int, n_heads: int = 4, d_k: int | None = None, d_v: int | None = None,
                 tau: float = 16.0, rank: int = 16, eps: float = 1e-5, chunk: int = 64, subchunk: int = 16,
                 path: str = "auto", device=None, dtype=torch.bfloat16, seed: int = 0):
        super().__init__()
        d = d_model
        self.H = n_heads
        self.dk = d_k if d_k is not None else d // 2
        self.dv = d_v if d_v is not None else d
        assert self.dk % n_heads == 0 and self.dv % n_heads == 0
        self.K, self.V = self.dk // n_heads, self.dv // n_heads
        self.tau, self.eps, self.chunk, self.subchunk, self.path = tau, eps, chunk, subchunk, path
        gen = torch.Generator(device="cpu").manual_seed(seed)

        def w(shape, fan_in):
            return torch.nn.Parameter((torch.randn(shape, generator=gen) / math.sqrt(fan_in)).to(device=device,
                                                                                                  dtype=dtype))

        def vec(n, fill):
            return torch.nn.Parameter(torch.full((n,), float(fill), device=device, dtype=torch.float32))

        self.W_qkvr = w((d, 2 * self.dk + 2 * self.dv), d)      # [W_Q | W_K | W_V | W_r]
        self.W_a1 = w((d, rank), d)
        self.W_a2 = w((rank, self.dk), rank)
        self.b_alpha = vec(self.dk, 0.0)
        self.b_r = vec(self.dv, 0.0)
        self.ln_w = vec(self.dv, 1.0)
        self.ln_b = vec(self.dv, 0.0)
        self.W_o = w((self.dv, d), self.dv)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        """x [B, T, d] bf16 -> y [B, T, d] bf16."""
        P = x @ self.W_qkvr
        Za = (x @ self.W_a1) @ self.W_a2
        cfg = (self.H, self.K, self.V, self.tau, self.eps, self.chunk, self.subchunk, self.path)
        Z = _LayerCore.apply(P.contiguous(), Za.contiguous(), self.b_alpha, self.b_r, self.ln_w, self.ln_b, cfg)
        return Z @ self.W_o
