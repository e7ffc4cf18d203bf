"""Seeded synthetic inputs shared by the oracle and the CUDA path (tests, smoke, bench).

This module holds NO arithmetic of the method: it only draws random numbers with the shapes and
value distributions of the paper's workloads.  Both sides receive the
exact same values: q, k, v, d_out are drawn in fp32 by a seeded ``torch.Generator`` on the CPU and
rounded once to the compute dtype; the oracle upcasts those rounded values exactly to fp64.

Gate distributions (log alpha, always <= 0):
  std      log alpha = logsigmoid(z) / 16, z ~ N(0,1)    (P:177 footnote: temperature 16 in log space)
  lowrank  log alpha = logsigmoid(x W1 W2 + b) / 16, rank 16
  strong   logsigmoid(z)  (tau = 1)
  near1    -1e-4           (state grows ~T)
  mixed    half the channels -5, half -1e-3
  ones     0               (alpha == 1: plain linear attention)
  const    log gamma, gamma = 0.9 (RetNet fixed decay)
  extreme  -30             (every cross-token weight underflows)
"""
from __future__ import annotations

import math

import torch

GATES = ("std", "lowrank", "strong", "near1", "mixed", "ones", "const", "extreme")


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def gates(kind: str, B: int, H: int, T: int, K: int, seed: int = 0, gamma: float = 0.9) -> torch.Tensor:
    """log alpha [B,H,T,K] fp32 on CPU."""
    shape = (B, H, T, K)
    g = _gen(seed * 7919 + 17)
    if kind == "std":
        z = torch.randn(shape, generator=g)
        return torch.nn.functional.logsigmoid(z) / 16.0
    if kind == "lowrank":
        d = 64
        x = torch.randn((B, T, d), generator=g)
        w1 = torch.randn((d, 16), generator=g) / math.sqrt(d)
        w2 = torch.randn((16, H * K), generator=g) / 4.0
        b = torch.randn((H * K,), generator=g) * 0.5 + 2.0
        z = (x @ w1 @ w2 + b).reshape(B, T, H, K).permute(0, 2, 1, 3).contiguous()
        return torch.nn.functional.logsigmoid(z) / 16.0
    if kind == "strong":
        return torch.nn.functional.logsigmoid(torch.randn(shape, generator=g))
    if kind == "near1":
        return torch.full(shape, -1e-4)
    if kind == "mixed":
        out = torch.full(shape, -1e-3)
        out[..., : K // 2] = -5.0
        return out
    if kind == "ones":
        return torch.zeros(shape)
    if kind == "const":
        return torch.full(shape, math.log(gamma))
    if kind == "extreme":
        return torch.full(shape, -30.0)
    raise ValueError(f"unknown gate distribution {kind!r}")


def qkv(B: int, H: int, T: int, K: int, V: int, seed: int = 0, dtype=torch.bfloat16):
    """q, k [B,H,T,K]; v [B,H,T,V]; unit normal, rounded once to ``dtype``, on CPU."""
    g = _gen(seed)
    q = torch.randn((B, H, T, K), generator=g).to(dtype)
    k = torch.randn((B, H, T, K), generator=g).to(dtype)
    v = torch.randn((B, H, T, V), generator=g).to(dtype)
    return q, k, v


def d_out(B: int, H: int, T: int, V: int, seed: int = 0, dtype=torch.bfloat16) -> torch.Tensor:
    g = _gen(seed * 104729 + 3)
    return torch.randn((B, H, T, V), generator=g).to(dtype)


def state(B: int, H: int, K: int, V: int, seed: int = 0, scale: float = 1.0) -> torch.Tensor:
    """A random fp32 [B,H,K,V] state (initial_state / d_final_state tests)."""
    g = _gen(seed * 31337 + 5)
    return torch.randn((B, H, K, V), generator=g) * scale


def problem(B, H, T, K, V, seed=0, gate="std", dtype=torch.bfloat16, gate_dtype=torch.float32):
    """Convenience bundle: dict of CPU tensors q, k, v, g, do."""
    q, k, v = qkv(B, H, T, K, V, seed, dtype)
    g = gates(gate, B, H, T, K, seed).to(gate_dtype)
    do = d_out(B, H, T, V, seed, dtype)
    return {"q": q, "k": k, "v": v, "g": g, "do": do}
