"""Multi-GPU plumbing for the GLA core: batch x head sharding and sequence-parallel state passing.

* B x H sharding: the (b,h) units are independent recurrences.  `shard_bh` gives each rank a
  contiguous slice of the batch; there is no collective on the data path.
* Sequence parallelism (T >= 16K): rank r of R owns tokens [r T/R, (r+1) T/R).  The chunk-level recurrence is
  a two-stage scan ("needs only a single pass"):
      forward : (S_loc_r, D_r) = state_summary(segment r)           -- all ranks in parallel
                H_r = recv(r-1);  H_{r+1} = e^{D_r} (.) H_r + S_loc_r; send(r+1)   -- linear chain of K x V states
                o_r = chunk_fwd(segment r, initial_state = H_r)      -- all ranks in parallel
      backward: dh_loc_r = dstate_summary(segment r)                 -- all ranks in parallel
                dF_r = recv(r+1) (d_final_state for the last rank);  dF_{r-1} = e^{D_r} (.) dF_r + dh_loc_r; send(r-1)
                grads_r = chunk_bwd(segment r, initial_state = H_r, d_final_state = dF_r)
  The exchanged message is one fp32 [B,H,K,V] state per hop (torch.distributed send/recv: NCCL on GPUs,
  gloo in the CPU tests).  `ops` defaults to the CUDA library; tests may inject other local operators to
  check the scan algebra and the communication pattern on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


@dataclass
class LocalOps:
    state_summary: Callable      # (k, v, g) -> (S_loc [B,H,K,V] fp32, log_decay [B,H,K] fp32)
    dstate_summary: Callable     # (q, do, g) -> dh0_loc [B,H,K,V] fp32
    state_combine: Callable      # (H_in, log_decay, S_loc) -> H_out
    chunk_fwd: Callable          # (q, k, v, g, h0) -> (o, final_state)
    chunk_bwd: Callable          # (q, k, v, g, do, h0, dfinal) -> (dq, dk, dv, dg, dh0)


def cuda_ops(chunk: int = 64, subchunk: int = 16, path: str = "auto") -> LocalOps:
    from . import binding as G
    return LocalOps(
        state_summary=lambda k, v, g: G.state_summary(k, v, g, chunk, subchunk),
        dstate_summary=lambda q, do, g: G.dstate_summary(q, do, g, chunk, subchunk),
        state_combine=lambda h, d, s: G.state_combine(h.contiguous(), d.contiguous(), s.contiguous()),
        chunk_fwd=lambda q, k, v, g, h0: G.chunk_fwd(q, k, v, g, chunk, subchunk, h0, True, path),
        chunk_bwd=lambda q, k, v, g, do, h0, dfin: G.chunk_bwd(q, k, v, g, do, chunk, subchunk, h0, dfin, True, path),
    )


def shard_bh(B: int, rank: int, world: int):
    """Contiguous batch slice [b0, b1) of rank `rank` (B x H sharding along B)."""
    per = (B + world - 1) // world
    b0 = min(B, rank * per)
    return b0, min(B, b0 + per)


@dataclass
class SPContext:
    H_in: torch.Tensor           # state entering this rank's segment
    log_decay: torch.Tensor      # D_r = sum of log alpha over the segment


def sp_forward(q, k, v, g, ops: LocalOps, group=None, initial_state: Optional[torch.Tensor] = None):
    """Sequence-parallel forward of this rank's segment.  Returns (o_local, final_state, ctx); final_state is
    the state after this rank's segment (the global final state on the last rank)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    S_loc, D = ops.state_summary(k, v, g)
    if rank == 0:
        H_in = initial_state if initial_state is not None else torch.zeros_like(S_loc)
    else:
        H_in = torch.empty_like(S_loc)
        dist.recv(H_in, src=_global(rank - 1, group), group=group)
    if rank + 1 < world:
        H_out = ops.state_combine(H_in, D, S_loc)
        dist.send(H_out.contiguous(), dst=_global(rank + 1, group), group=group)
    o, fs = ops.chunk_fwd(q, k, v, g, H_in)
    return o, fs, SPContext(H_in=H_in, log_decay=D)


def sp_backward(q, k, v, g, do, ctx: SPContext, ops: LocalOps, group=None,
                d_final_state: Optional[torch.Tensor] = None):
    """Sequence-parallel backward of this rank's segment: (dq, dk, dv, dlog_alpha, d_initial_state_of_segment)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dh_loc = ops.dstate_summary(q, do, g)
    if rank == world - 1:
        dF = d_final_state if d_final_state is not None else torch.zeros_like(dh_loc)
    else:
        dF = torch.empty_like(dh_loc)
        dist.recv(dF, src=_global(rank + 1, group), group=group)
    if rank > 0:
        dF_prev = ops.state_combine(dF, ctx.log_decay, dh_loc)
        dist.send(dF_prev.contiguous(), dst=_global(rank - 1, group), group=group)
    return ops.chunk_bwd(q, k, v, g, do, ctx.H_in, dF)


def _global(r: int, group) -> int:
    return r if group is None else dist.get_global_rank(group, r)
