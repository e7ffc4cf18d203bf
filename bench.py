#!/usr/bin/env python
"""bench.py -- GLA layer (core op) forward+backward throughput at the paper's 1.3B shapes on B200.

Metric (BASELINE.json): "GLA layer fwd+bwd tokens/s at 1.3B shapes, T=2K-16K; % of bf16 tensor peak".
One step = gla_chunk_fwd + gla_chunk_bwd over one synthetic batch (all four parts of the method).
Default workload (N=1): BASELINE.json configs[2] -- B=16, H=4, T=2048, per-head K=256, V=512 (d_model 2048,
d_k = d/2, d_v = d), chunk 64, sub-chunk 16, bf16 q/k/v/d_out, fp32 log alpha = logsigmoid(z)/16.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 1p3b|340m|long4k|...|sp32k]
                  [--scaling weak|strong] [--schedule chain|pipelined|allgather]

Multi-GPU: `--gpus N` without a torchrun environment re-launches itself under torch.distributed.run with N
ranks (127.0.0.1); under torchrun WORLD_SIZE must equal N.  One process per GPU; ranks beyond the visible
GPU count share devices round-robin (then the control collectives run on gloo; the timing is still per rank
on the device, max over ranks).
  * B x H configs: batch x head sharding with no collective on the data path.
      --scaling weak   (default) every rank runs the full per-GPU workload (global batch = N x B);
      --scaling strong the global batch B is fixed and split across ranks (parallel.shard_bh).
  * sp32k (BASELINE.json configs[4]): B=1, H=4, T=32768 at 1.3B shapes, sequence-parallel across the N ranks:
    state summaries -> chunk-state scan over send/recv (NCCL; host-staged on gloo) -> local fwd from the
    received state; the backward mirrors it.  Total work fixed ("scaling": "strong").
Time = max over ranks (all_reduce MAX) of CUDA-event time on each rank's stream, with barriers around.
--impl reference: the fp64 CPU oracle (the only reference that exists for this paper), timed on the host
cores on a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

CONFIGS = {
    # name: (B, H, T, K, V)
    "1p3b": (16, 4, 2048, 256, 512),
    "340m": (8, 4, 2048, 128, 256),
    "long4k": (8, 4, 4096, 256, 512),
    "long8k": (4, 4, 8192, 256, 512),
    "long16k": (2, 4, 16384, 256, 512),
    "sp32k": (1, 4, 32768, 256, 512),
    "tiny": (1, 1, 64, 16, 32),
}
SP_CONFIGS = ("sp32k",)
METRIC = "GLA layer fwd+bwd tokens/s at 1.3B shapes, T=2K-16K; % of bf16 tensor peak"
L2_BYTES = 126 * 2**20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return {"hbm": d["hbm_gbs"], "tf_burst": d["bf16_tflops"],
                "tf_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    except Exception:   # B200_PROFILING.md fallback figures
        return {"hbm": 6650.0, "tf_burst": 1590.0, "tf_sustained": 1400.0, "source": "fallback"}


# ---- algorithmic work ------------------------------------------
def flops_per_token_head(K, V, C, c):
    """Method FLOPs per token per head, recompute excluded."""
    fwd = 4 * K * V + (C + 1) * K + (C + c) * V
    bwd = 8 * K * V + 2 * (C + 1) * K + 2 * (C + c) * V
    return fwd, bwd


def bytes_per_token_head(K, V, g=4, e=2):
    """Algorithmic HBM bytes per token per head: each input read once, each output written once (§8(d))."""
    fwd = e * K + e * K + e * V + g * K + e * V                       # q, k, v, log alpha in; o out
    bwd = (2 * e * K + e * V + g * K + e * V) + (2 * e * K + e * V + g * K)   # q,k,v,g,dO in; dq,dk,dv,dg out
    return fwd, bwd


def kernel_algo(name, K, V, C, c, g=4, e=2):
    """(method FLOPs, algorithmic bytes) per token-head assigned to one kernel.  Every term of §8(d) is assigned
    to exactly one kernel -- the one that computes it, or, for a tensor of the method's I/O, the first kernel of
    the step that reads it / the kernel that writes it -- so the per-kernel figures sum to the step's.  Design
    intermediates (Q~, K~, P, dP, statistics, V-tile partials, anchors) are NOT algorithmic: they show up only in
    `traffic` (ncu DRAM bytes) and the step's traffic_ratio."""
    table = {
        # forward: a1 + a3's scores in prep; a2 + a3's P V in the state walk
        "tc::fwd_prep": ((C + 1) * K, 2 * e * K + g * K),                       # reads q, k, log alpha
        "tc::fwd_state": (4 * K * V + (C + c) * V, e * V + e * V),              # reads v, writes o
        # backward (saved forward operands)
        "tc::bwd_dp": ((C + c) * V, e * V + e * V),                             # dP = dO V^T; reads dO, v
        "tc::bwd_prep": ((C + c) * V, e * V + e * V),
        "tc::bwd_dq": (2 * K * V + (C + 1) * K, 0),                             # dq inter + intra
        "tc::bwd_dk": (2 * K * V + (C + 1) * K, 0),                             # dk inter + intra (K-tiled walk)
        "tc::bwd_dv": (4 * K * V + (C + c) * V, e * V),                         # dH update, dv inter + intra; writes dv
        "tc::bwd_dkv": (6 * K * V + (C + 1) * K + (C + c) * V, e * V),          # dk, dv inter + intra, dH; writes dv
        "tc::bwd_reduce": (0, 2 * e * K + g * K + 2 * e * K + g * K),           # reads q, k, g; writes dq, dk, dg
    }
    for key, val in table.items():
        if name == key or name.endswith(key):
            return val
    return None


# ---- clocks sampler -------------------------------------------------------------------------------------------
class Clocks:
    """Samples SM clock and throttle reasons via NVML every ~2 ms during the timed region (the same fields as
    the recipe's nvidia-smi clocks line: clocks.sm, clocks.max.sm, hw/sw slowdown, sw_power_cap)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.sm, self.reasons, self.max = [], set(), None
        self.stop = threading.Event()
        self.t = None

    def _run(self):
        import pynvml as N
        N.nvmlInit()
        h = N.nvmlDeviceGetHandleByIndex(self.idx)
        self.max = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
        while not self.stop.is_set():
            self.sm.append(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM))
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.reasons |= {n for bit, n in self.REASONS.items() if r & bit}
            time.sleep(0.002)

    def __enter__(self):
        try:
            import pynvml  # noqa: F401
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.sm and time.time() - t0 < 5.0:   # NVML initialised and sampling before timing starts
                time.sleep(0.002)
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.sm), "sm_max_mhz": self.max, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


# ---- CPU oracle baseline -------------------------------------------------------------------------------------
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_oracle_sample(cfg, seed=0, n_slices=None, T_sample=None):
    """Time the fp64 oracle fwd+bwd on a bounded sample of (b,h) slices of the workload on the host cores."""
    import oracle
    import synth
    B, H, T, K, V = cfg
    cores = host_cores()
    n = n_slices or max(1, 2 * min(cores, 32))
    Ts = T_sample or T
    p = synth.problem(1, n, Ts, K, V, seed=seed)
    f = {k: v.double().numpy() for k, v in p.items()}
    t0 = time.perf_counter()
    oracle.fwd(f["q"], f["k"], f["v"], f["g"], nthreads=n)
    oracle.bwd(f["q"], f["k"], f["v"], f["g"], f["do"], nthreads=n)
    dt = time.perf_counter() - t0
    tokens = n * Ts / H          # a token of the layer = H head-slices
    return {"value": tokens / dt, "unit": "tokens/s", "cores": min(n, cores), "kind": "oracle",
            "sample": f"{n} (b,h) slices x T={Ts} of B={B},H={H},T={T},K={K},V={V} fwd+bwd in fp64 "
                      f"({dt:.2f} s; tokens = slices*T/H)", "seconds": dt}


# ---- launch ---------------------------------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="1p3b")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--schedule", choices=["chain", "pipelined", "allgather"], default="chain")
    ap.add_argument("--path", choices=["auto", "simt", "tc"], default="auto")
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--subchunk", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    return ap.parse_args()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch_under_torchrun(args):
    """`--gpus N` from a plain shell: re-exec this script as N ranks (one process per GPU)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")            # the driver can see nranks in NCCL's init lines
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    return subprocess.call(cmd, env=env)


def config_dict(args, cfg, world, per_rank):
    B, H, T, K, V = cfg
    sp = args.config in SP_CONFIGS
    if sp:
        par = f"sequence-parallel x{world} ({args.schedule} chunk-state scan over send/recv)" if world > 1 \
            else "single GPU (intra-GPU segment split)"
    else:
        par = f"bh-shard x{world} (no data-path collective)"
    d = {"workload": f"GLA core fwd+bwd, BASELINE.json configs[{4 if sp else 2}] shapes ({args.config})",
         "model": "gla-1.3b-layer" if K == 256 else "gla-340m-layer",
         "global_batch": B * world if (args.scaling == "weak" and not sp) else B,
         "per_gpu_batch": per_rank[0], "heads": H, "seq_len": T, "per_gpu_seq_len": per_rank[2],
         "d_k_head": K, "d_v_head": V, "chunk": args.chunk, "subchunk": args.subchunk, "parallelism": par,
         "gates": "logsigmoid(N(0,1))/16 fp32",
         "l2": "inputs > L2 (no flush)" if input_bytes(per_rank) > 2 * L2_BYTES else "L2 flushed between steps"}
    return d


def input_bytes(cfg):
    B, H, T, K, V = cfg
    return B * H * T * (2 * K * 2 + 2 * V * 2 + 4 * K)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    B, H, T, K, V = cfg
    vals = []
    base = None
    T_s = min(T, 2048)
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(cfg, seed=i, n_slices=None, T_sample=T_s)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    v = statistics.mean(vals)
    ms = (B * T) / v * 1e3
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_step_note": "extrapolated: each timed step is a bounded sample (see cpu_baseline.sample); "
                                "ms_per_step = workload tokens / measured tokens per second",
            "higher_is_better": True, "scaling": "strong" if args.config in SP_CONFIGS else args.scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, cfg, 1, cfg),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": base["cores"], "kind": "oracle",
                             "sample": base["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---- the workload -------------------------------------------------------------------------------------------
class Workload:
    """One rank's part of a step: tensors resident on the device, and `step(inputs)` through the public API."""

    def __init__(self, args, cfg, rank, world, dev, group):
        import synth
        from paper_2312_06635_b200 import binding as G
        from paper_2312_06635_b200 import parallel as P
        self.G, self.P = G, P
        self.args, self.dev, self.group = args, dev, group
        B, H, T, K, V = cfg
        self.sp = args.config in SP_CONFIGS
        C, c = args.chunk, args.subchunk
        if self.sp:
            t0, t1 = P.shard_seq(T, rank, world, C)
            p = synth.problem(B, H, T, K, V, seed=1)           # one global sequence; each rank takes its tokens
            p = {n: x[:, :, t0:t1].contiguous() for n, x in p.items()}
            self.per_rank = (B, H, t1 - t0, K, V)
            self.tokens_global = B * T
        else:
            if args.scaling == "strong":
                b0, b1 = P.shard_bh(B, rank, world)
                p = synth.problem(B, H, T, K, V, seed=1)
                p = {n: x[b0:b1].contiguous() for n, x in p.items()}
                self.per_rank = (b1 - b0, H, T, K, V)
                self.tokens_global = B * T
            else:
                p = synth.problem(B, H, T, K, V, seed=1000 * rank + 1)
                self.per_rank = (B, H, T, K, V)
                self.tokens_global = B * T * world
        self.inputs = [p[n].to(dev) for n in ("q", "k", "v", "g", "do")]
        q, k, v, g, do = self.inputs
        self.path = G.resolve_path(q, v, g, C, c, args.path)
        self.wf = G.fwd_workspace(q, v, g, C, c, args.path)
        self.wb = G.bwd_workspace(q, v, g, C, c, args.path)
        self.ops = P.cuda_ops(C, c, args.path) if self.sp else None
        self.group_size = world
        self.chain_ms = []

    def outputs_like(self):
        q, k, v, g, do = self.inputs
        return [torch.empty_like(v), torch.empty_like(q), torch.empty_like(k), torch.empty_like(v),
                torch.empty(q.shape, dtype=torch.float32, device=self.dev)]

    def step(self, x, outs, stream, time_chain=False):
        """Forward + backward of this rank's part.  x = (q, k, v, g, dO); outs = (o, dq, dk, dv, dg)."""
        G, args = self.G, self.args
        C, c = args.chunk, args.subchunk
        q, k, v, g, do = x
        if not self.sp:
            G.chunk_fwd(q, k, v, g, C, c, None, False, args.path, out=outs[0], workspace=self.wf)
            G.chunk_bwd(q, k, v, g, do, C, c, None, None, False, args.path, grads=(*outs[1:], None),
                        workspace=self.wb, fwd_workspace=self.wf)
            return
        P = self.P
        if self.group_size == 1:   # one GPU: the whole sequence locally (intra-GPU segment split)
            G.chunk_fwd(q, k, v, g, C, c, None, False, args.path, out=outs[0], workspace=self.wf)
            G.chunk_bwd(q, k, v, g, do, C, c, None, None, False, args.path, grads=(*outs[1:], None),
                        workspace=self.wb, fwd_workspace=self.wf)
            return
        S_loc, D = G.state_summary(k, v, g, C, c, args.path, workspace=self.wf)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if time_chain else None
        if e:
            e[0].record(stream)
        H_in, _ = P.scan_forward(S_loc, D, self.ops, self.group, None, args.schedule)
        if e:
            e[1].record(stream)
        G.chunk_fwd(q, k, v, g, C, c, H_in, False, args.path, out=outs[0], workspace=self.wf)
        dh = G.dstate_summary(q, do, g, C, c, args.path, workspace=self.wb_sum())
        if e:
            e[2].record(stream)
        dF = P.scan_backward(dh, D, self.ops, self.group, None, args.schedule)
        if e:
            e[3].record(stream)
        G.chunk_bwd(q, k, v, g, do, C, c, H_in, dF, False, args.path, grads=(*outs[1:], None), workspace=self.wb,
                    fwd_workspace=self.wf)
        if e:
            self.chain_ms.append(e)

    def wb_sum(self):
        # the adjoint summary must not overwrite the forward's workspace (the saved backward reuses it)
        if not hasattr(self, "_wsum"):
            q, k, v, g, do = self.inputs
            self._wsum = self.G.fwd_workspace(q, do, g, self.args.chunk, self.args.subchunk, self.args.path)
        return self._wsum


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        return run_reference(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    ndev = torch.cuda.device_count()
    sharing = world > ndev
    torch.cuda.set_device(local % ndev)
    dev = torch.device("cuda", local % ndev)
    dist = None
    group = None
    if world > 1:
        import torch.distributed as dist
        if sharing:   # NCCL needs one device per rank: ranks sharing a GPU use gloo (host-staged exchange)
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    W = Workload(args, cfg, rank, world, dev, group)
    outs = W.outputs_like()
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) \
        if input_bytes(W.per_rank) <= 2 * L2_BYTES else None
    stream = torch.cuda.current_stream(dev)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if sharing else dev)
        if dist:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        W.step(W.inputs, outs, stream)
    barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(dev.index) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            evs[i][0].record(stream)
            W.step(W.inputs, outs, stream, time_chain=W.sp and world > 1)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    total_ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs))
    ms_step = total_ms / args.steps
    value = W.tokens_global / (ms_step / 1e3)
    chain = None
    if W.chain_ms:
        f = statistics.median(e[0].elapsed_time(e[1]) for e in W.chain_ms)
        b = statistics.median(e[2].elapsed_time(e[3]) for e in W.chain_ms)
        chain = {"fwd_scan_ms": max_over_ranks(f), "bwd_scan_ms": max_over_ranks(b), "hops": world - 1,
                 "schedule": args.schedule, "message_bytes": 4 * W.per_rank[0] * W.per_rank[1] * cfg[3] * cfg[4],
                 "note": "per-rank CUDA-event time of the exchange stage (includes waiting for the upstream ranks), "
                         "median over steps, max over ranks"}

    # per-kernel live times: a separate pass with the library's launch tracer on (it brackets every launch with
    # events on its stream and runs the two backward walks one after the other so each launch's time is its own)
    prof, launches = {}, None
    if not args.no_profile:
        W.G.profile(True)
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            W.step(W.inputs, outs, stream)
        torch.cuda.synchronize()
        W.G.lib().gla_profile_enable(0)
        prof = W.G.profile_read()
        launches = W.G.lib().gla_profile_count()
    barrier()

    # e2e through the public API with pinned host buffers: every step copies its inputs host -> device and all of
    # its results device -> host.  The copies are pipelined against the compute the way a training input / output
    # pipeline would run them (H2D of step n+1 and D2H of step n-1 on their own streams while step n computes;
    # inputs and outputs double-buffered on the device), so the step time is bounded by PCIe, not by the sum.
    e2e = None
    if not args.no_e2e:
        host_in = [x.cpu().pin_memory() for x in W.inputs]
        host_out = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
        n_e2e = max(2, min(args.steps, 20))
        h2d = sum(x.numel() * x.element_size() for x in host_in)
        d2h = sum(x.numel() * x.element_size() for x in host_out)
        dd = [[torch.empty_like(x) for x in W.inputs] for _ in range(2)]
        oo = [W.outputs_like() for _ in range(2)]
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = {k_: [torch.cuda.Event() for _ in range(2)] for k_ in ("in_ready", "in_free", "out_ready", "out_free")}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        s_h2d.wait_stream(stream)
        s_d2h.wait_stream(stream)
        for n in range(n_e2e):
            bb = n & 1
            with torch.cuda.stream(s_h2d):
                if n >= 2:
                    s_h2d.wait_event(ev["in_free"][bb])
                for dst, src in zip(dd[bb], host_in):
                    dst.copy_(src, non_blocking=True)
                ev["in_ready"][bb].record(s_h2d)
            stream.wait_event(ev["in_ready"][bb])
            if n >= 2:
                stream.wait_event(ev["out_free"][bb])
            W.step(dd[bb], oo[bb], stream)
            ev["in_free"][bb].record(stream)
            ev["out_ready"][bb].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev["out_ready"][bb])
                for dst, src in zip(host_out, oo[bb]):
                    dst.copy_(src, non_blocking=True)
                ev["out_free"][bb].record(s_d2h)
        stream.wait_stream(s_d2h)
        e1.record(stream)
        torch.cuda.synchronize()
        et = max_over_ranks(e0.elapsed_time(e1) / n_e2e)
        e2e = {"value": W.tokens_global / (et / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": et, "steps": n_e2e,
               "overlap": "H2D(n+1) and D2H(n-1) overlap compute(n); pipeline fill and drain included",
               "bytes_note": "per rank" if world > 1 else None}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    line = report(args, cfg, W, world, ms_step, value, prof, launches, clk, e2e, chain, sharing)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def report(args, cfg, W, world, ms_step, value, prof, launches, clk, e2e, chain, sharing):
    pk = load_peaks()
    Bp, H, Tp, K, V = W.per_rank
    C, c = args.chunk, args.subchunk
    u_rank = Bp * H * Tp                              # token-heads per rank per step
    ff, fb = flops_per_token_head(K, V, C, c)
    bf, bb = bytes_per_token_head(K, V)
    # step level (per rank; every rank runs the same amount of work)
    algo_flops, algo_bytes = u_rank * (ff + fb), u_rank * (bf + bb)
    step_s = ms_step / 1e3
    ncu = {}
    try:   # per-launch DRAM bytes of each kernel from the committed `ncu --set full` capture (profiles/)
        ncu = json.load(open(os.path.join(ROOT, "profiles", "ncu_summary_latest.json")))
    except Exception:
        pass
    # which kernel of the capture each traced name is (the K-tiled dq / dk walks are one template, REV = 0 / 1;
    # the dv walk is k_bwd_dkv3<K, 2>)
    ncu_keys = {"tc::fwd_prep": [f"k_fwd_prep<{K},"], "tc::fwd_state": [f"k_fwd_state<{K}>"],
                "tc::bwd_dp": ["k_bwd_dp"], "tc::bwd_prep": [f"k_bwd_prep<{K},"],
                "tc::bwd_dq": [f"k_bwd_kwalk<{K}, 0,", f"k_bwd_kwalk<{K}, false", f"k_bwd_dq3<{K}>"],
                "tc::bwd_dk": [f"k_bwd_kwalk<{K}, 1,", f"k_bwd_kwalk<{K}, true"],
                "tc::bwd_dv": [f"k_bwd_dkv3<{K}, 2>"], "tc::bwd_dkv": [f"k_bwd_dkv3<{K}, 1>"],
                "tc::bwd_reduce": [f"k_bwd_reduce_tma<{K},"], "simt::bwd_gate": ["k_bwd_gate"]}

    def traffic_of(name):
        for key in ncu_keys.get(name, []):
            for n, v in ncu.items():
                if key in n:
                    return v.get("traffic_bytes")
        return None

    kernels = {}
    roof = None
    if prof:
        prof_ms = sum(v_[0] for v_ in prof.values()) / args.steps
        for n, (tot, nl) in prof.items():
            per_s = tot / nl / 1e3
            a = kernel_algo(n, K, V, C, c)
            ent = {"ms_total": tot, "launches": nl, "ms_per_launch": per_s * 1e3,
                   "share_of_step": tot / args.steps / prof_ms if prof_ms else None}
            if a and W.path == "tc":
                fl, by = a[0] * u_rank, a[1] * u_rank
                ent.update({"method_tflops": fl / per_s / 1e12, "tensor_frac": fl / per_s / 1e12 / pk["tf_sustained"],
                            "algo_gbs": by / per_s / 1e9, "hbm_frac": by / per_s / 1e9 / pk["hbm"],
                            "traffic": traffic_of(n)})
            kernels[n] = ent
        top = max(prof, key=lambda n: prof[n][0])
        ent = kernels[top]
        a = kernel_algo(top, K, V, C, c)
        if a and W.path == "tc":
            fl, by = a[0] * u_rank, a[1] * u_rank
            t_flop, t_hbm = fl / (pk["tf_sustained"] * 1e12), by / (pk["hbm"] * 1e9)
            per_s = ent["ms_per_launch"] / 1e3
            tensor = t_flop >= t_hbm
            roof = {"kernel": top, "bound": "tensor" if tensor else "hbm",
                    "achieved": fl / per_s / 1e12 if tensor else by / per_s / 1e9,
                    "peak": pk["tf_sustained"] if tensor else pk["hbm"], "unit": "TFLOP/s" if tensor else "GB/s",
                    "frac": (fl / per_s / 1e12 / pk["tf_sustained"]) if tensor else (by / per_s / 1e9 / pk["hbm"]),
                    "traffic": ent.get("traffic"),
                    "algo_flops_per_launch": fl, "algo_bytes_per_launch": by, "ms_per_launch": ent["ms_per_launch"],
                    "share_of_step": ent["share_of_step"],
                    "peak_source": f"{pk['source']} ({'bf16 sustained' if tensor else 'HBM copy'}, MEASURED_PEAKS.json)",
                    "accounting": "achieved = SURVEY §8(d) method FLOPs (or algorithmic bytes) assigned to this "
                                  "kernel per token-head x token-heads per launch / its CUDA-event launch time"}
    traffic_total = None
    if ncu and prof:
        tt = [traffic_of(n) for n in prof]
        if all(t is not None for t in tt):
            traffic_total = sum(tt)
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if (W.sp or args.scaling == "strong") else "weak",
            "vs_baseline": None, "dtype": "bf16" if W.inputs[0].dtype == torch.bfloat16 else "f32",
            "data": "synthetic", "config": config_dict(args, cfg, world, W.per_rank), "path": W.path,
            "algo": {"flops_per_step_per_gpu": algo_flops, "bytes_per_step_per_gpu": algo_bytes,
                     "tflops": algo_flops / step_s / 1e12,
                     "frac_of_bf16_peak_burst": algo_flops / step_s / 1e12 / pk["tf_burst"],
                     "frac_of_bf16_peak_sustained": algo_flops / step_s / 1e12 / pk["tf_sustained"],
                     "hbm_gbs": algo_bytes / step_s / 1e9, "frac_of_hbm": algo_bytes / step_s / 1e9 / pk["hbm"],
                     "ncu_traffic_bytes_per_step": traffic_total,
                     "traffic_ratio": traffic_total / algo_bytes if traffic_total else None,
                     "accounting": "SURVEY §8(d): FLOPs fwd 4KV+(C+1)K+(C+c)V, bwd 8KV+2(C+1)K+2(C+c)V; bytes "
                                   "fwd 4K+4V+4K(g), bwd 8K+6V+8K(g) per token-head; recompute and design "
                                   "intermediates excluded (they appear in traffic_ratio)"},
            "roofline": roof, "kernels": kernels, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e}
    if chain:
        line["sp_exchange"] = chain
    if sharing:
        line["device_sharing"] = f"{world} ranks on {torch.cuda.device_count()} GPU(s): timing valid per rank, " \
                                 "not a scaling number"
    if world == 1 and not args.no_cpu_baseline:
        # ~10 s of oracle work on the host cores (5 slices per core): the contract's bounded 10-30 s sample
        n_cpu = 5 * min(host_cores(), 32)
        line["cpu_baseline"] = {k_: v_ for k_, v_ in cpu_oracle_sample(cfg, n_slices=n_cpu,
                                                                        T_sample=min(cfg[2], 2048)).items()
                                if k_ != "seconds"}
    return line


if __name__ == "__main__":
    main()
