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

Three exchange schedules for the middle stage:
  "chain"      the linear chain above: R-1 sequential hops of the whole [B,H,K,V] state per direction;
  "pipelined"  the same chain split into one message per (b,h) unit: rank r forwards unit u as soon as it has
               combined it, so the hops of later units overlap the earlier units' transfers (latency
               R-1 + U-1 message times instead of (R-1) U);
  "allgather"  one all_gather of every rank's (S_loc, D) (or (dh_loc, D)); each rank then folds the earlier
               (later) ranks' summaries locally with state_combine: one collective, O(R) local combines.
All three give the same H_r / dF_r up to the order of fp32 additions (identical for chain / pipelined).

When the process group's backend is gloo (CPU tests; ranks sharing one GPU), CUDA tensors are staged through
host memory for the exchange; with NCCL they go device to device over NVLink.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist

SCHEDULES = ("chain", "pipelined", "allgather")


@dataclass
class LocalOps:
    state_summary: Callable      # (k, v, g) -> (S_loc [B,H,K,V] fp32, log_decay [B,H,K] fp32)
    dstate_summary: Callable     # (q, do, g) -> dh0_loc [B,H,K,V] fp32
    state_combine: Callable      # (H_in, log_decay, S_loc) -> H_out
    chunk_fwd: Callable          # (q, k, v, g, h0) -> (o, final_state)
    chunk_bwd: Callable          # (q, k, v, g, do, h0, dfinal) -> (dq, dk, dv, dg, dh0)


def cuda_ops(chunk: int = 64, subchunk: int = 16, path: str = "auto", saved: bool = True) -> LocalOps:
    """The library's operators.  With ``saved`` the forward's workspace (per-chunk operands, segment states) is
    kept between chunk_fwd and chunk_bwd of the same segment, as in a training step (gla_chunk_bwd_saved)."""
    from . import binding as G
    ws = {}

    def fwd(q, k, v, g, h0):
        w = G.fwd_workspace(q, v, g, chunk, subchunk, path)
        if saved:
            ws["f"] = (w, q.data_ptr())
        return G.chunk_fwd(q, k, v, g, chunk, subchunk, h0, True, path, workspace=w)

    def bwd(q, k, v, g, do, h0, dfin):
        w = ws.get("f")
        fw = w[0] if (w is not None and w[1] == q.data_ptr()) else None
        return G.chunk_bwd(q, k, v, g, do, chunk, subchunk, h0, dfin, True, path, fwd_workspace=fw)

    return LocalOps(
        state_summary=lambda k, v, g: G.state_summary(k, v, g, chunk, subchunk, path),
        dstate_summary=lambda q, do, g: G.dstate_summary(q, do, g, chunk, subchunk, path),
        state_combine=lambda h, d, s: G.state_combine(h.contiguous(), d.contiguous(), s.contiguous()),
        chunk_fwd=fwd,
        chunk_bwd=bwd,
    )


def shard_bh(B: int, rank: int, world: int):
    """Contiguous batch slice [b0, b1) of rank `rank` (B x H sharding along B)."""
    per = (B + world - 1) // world
    b0 = min(B, rank * per)
    return b0, min(B, b0 + per)


def shard_seq(T: int, rank: int, world: int, chunk: int = 64):
    """Token slice [t0, t1) of rank `rank` for sequence parallelism (whole chunks per rank)."""
    if T % (world * chunk) != 0:
        raise ValueError(f"T={T} must split into {world} ranks of whole {chunk}-token chunks")
    per = T // world
    return rank * per, (rank + 1) * per


# ---- point-to-point with host staging on gloo ---------------------------------------------------------------
def _staged(group) -> bool:
    return dist.get_backend(group) == "gloo"


def _send(t: torch.Tensor, dst: int, group):
    if _staged(group) and t.is_cuda:
        t = t.cpu()
    dist.send(t.contiguous(), dst=dst, group=group)


def _recv(like: torch.Tensor, src: int, group) -> torch.Tensor:
    if _staged(group) and like.is_cuda:
        buf = torch.empty(like.shape, dtype=like.dtype)
        dist.recv(buf, src=src, group=group)
        return buf.to(like.device)
    buf = torch.empty_like(like)
    dist.recv(buf, src=src, group=group)
    return buf


def _all_gather(t: torch.Tensor, group):
    world = dist.get_world_size(group)
    src = t.cpu() if (_staged(group) and t.is_cuda) else t.contiguous()
    out = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(out, src, group=group)
    return [x.to(t.device) for x in out]


def _global(r: int, group) -> int:
    return r if group is None else dist.get_global_rank(group, r)


# ---- the middle stage: prefix (forward) / suffix (backward) of the chunk-state scan ---------------------------
def _flat(x):   # [B,H,...] -> [B*H,...] view (units)
    return x.reshape(x.shape[0] * x.shape[1], *x.shape[2:])


def scan_forward(S_loc, D, ops: LocalOps, group=None, initial_state=None, schedule: str = "chain"):
    """H_r (state entering this rank's segment) and H_{r+1} (leaving it), for every schedule."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    zero = torch.zeros_like(S_loc)
    h0 = initial_state if initial_state is not None else zero
    if schedule == "allgather":
        Ss, Ds = _all_gather(S_loc, group), _all_gather(D, group)
        h0s = _all_gather(h0, group)           # rank 0's initial state reaches everyone
        H = h0s[0]
        for j in range(rank):
            H = ops.state_combine(H, Ds[j], Ss[j])
        return H, ops.state_combine(H, D, S_loc)
    if schedule == "chain":
        H_in = h0 if rank == 0 else _recv(S_loc, _global(rank - 1, group), group)
        H_out = ops.state_combine(H_in, D, S_loc)
        if rank + 1 < world:
            _send(H_out, _global(rank + 1, group), group)
        return H_in, H_out
    if schedule == "pipelined":
        B, H = S_loc.shape[:2]
        Sf, Df, hf = _flat(S_loc), _flat(D), _flat(h0)
        H_in = torch.empty_like(Sf)
        H_out = torch.empty_like(Sf)
        for u in range(B * H):                 # one message per (b,h) unit, forwarded as soon as it is combined
            hin = hf[u:u + 1] if rank == 0 else _recv(Sf[u:u + 1], _global(rank - 1, group), group)
            H_in[u:u + 1] = hin
            H_out[u:u + 1] = ops.state_combine(hin[None], Df[u:u + 1][None], Sf[u:u + 1][None])[0]
            if rank + 1 < world:
                _send(H_out[u:u + 1], _global(rank + 1, group), group)
        return H_in.reshape(S_loc.shape), H_out.reshape(S_loc.shape)
    raise ValueError(f"unknown schedule {schedule!r} (one of {SCHEDULES})")


def scan_backward(dh_loc, D, ops: LocalOps, group=None, d_final_state=None, schedule: str = "chain"):
    """dF_r: the d_final_state of this rank's segment (= the d_initial_state of rank r+1's)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    zero = torch.zeros_like(dh_loc)
    dfin = d_final_state if d_final_state is not None else zero
    if schedule == "allgather":
        hs, Ds = _all_gather(dh_loc, group), _all_gather(D, group)
        dfs = _all_gather(dfin, group)         # the last rank's d_final_state reaches everyone
        dF = dfs[world - 1]
        for j in range(world - 1, rank, -1):
            dF = ops.state_combine(dF, Ds[j], hs[j])
        return dF
    if schedule == "chain":
        dF = dfin if rank == world - 1 else _recv(dh_loc, _global(rank + 1, group), group)
        if rank > 0:
            _send(ops.state_combine(dF, D, dh_loc), _global(rank - 1, group), group)
        return dF
    if schedule == "pipelined":
        hf, Df, ff = _flat(dh_loc), _flat(D), _flat(dfin)
        dF = torch.empty_like(hf)
        for u in range(hf.shape[0]):
            x = ff[u:u + 1] if rank == world - 1 else _recv(hf[u:u + 1], _global(rank + 1, group), group)
            dF[u:u + 1] = x
            if rank > 0:
                _send(ops.state_combine(x[None], Df[u:u + 1][None], hf[u:u + 1][None])[0],
                      _global(rank - 1, group), group)
        return dF.reshape(dh_loc.shape)
    raise ValueError(f"unknown schedule {schedule!r} (one of {SCHEDULES})")


@dataclass
class SPContext:
    H_in: torch.Tensor           # state entering this rank's segment
    log_decay: torch.Tensor      # D_r = sum of log alpha over the segment


def sp_forward(q, k, v, g, ops: LocalOps, group=None, initial_state: Optional[torch.Tensor] = None,
               schedule: str = "chain"):
    """Sequence-parallel forward of this rank's segment.  Returns (o_local, final_state, ctx); final_state is
    the state after this rank's segment (the global final state on the last rank)."""
    S_loc, D = ops.state_summary(k, v, g)
    H_in, _ = scan_forward(S_loc, D, ops, group, initial_state, schedule)
    o, fs = ops.chunk_fwd(q, k, v, g, H_in)
    return o, fs, SPContext(H_in=H_in, log_decay=D)


def sp_backward(q, k, v, g, do, ctx: SPContext, ops: LocalOps, group=None,
                d_final_state: Optional[torch.Tensor] = None, schedule: str = "chain"):
    """Sequence-parallel backward of this rank's segment: (dq, dk, dv, dlog_alpha, d_initial_state_of_segment)."""
    dh_loc = ops.dstate_summary(q, do, g)
    dF = scan_backward(dh_loc, ctx.log_decay, ops, group, d_final_state, schedule)
    return ops.chunk_bwd(q, k, v, g, do, ctx.H_in, dF)
