#!/usr/bin/env python
"""bench.py -- GLA layer (core op) forward+backward throughput at the paper's 1.3B shapes on B200.

Metric (BASELINE.json): "GLA layer fwd+bwd tokens/s at 1.3B shapes, T=2K-16K; % of bf16 tensor peak".
One step = gla_chunk_fwd + gla_chunk_bwd over one synthetic batch (all four parts of the method).
Default workload (N=1): BASELINE.json configs[2] -- B=16, H=4, T=2048, per-head K=256, V=512 (d_model 2048,
d_k = d/2, d_v = d), chunk 64, sub-chunk 16, bf16 q/k/v/d_out, fp32 log alpha = logsigmoid(z)/16.

  python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference] [--config 1p3b|340m|long4k|...]

Multi-GPU (torchrun): batch x head sharding with no communication on the data path ("scaling": "weak":
every rank runs the full per-GPU workload on its own seed); time = max over ranks (all_reduce MAX).
--impl reference: the fp64 CPU oracle (the only reference that exists for this paper), timed on the host
cores on a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
    "tiny": (1, 1, 64, 16, 32),
}
METRIC = "GLA layer fwd+bwd tokens/s at 1.3B shapes, T=2K-16K; % of bf16 tensor peak"
L2_BYTES = 126 * 2**20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d.get("bf16_tflops_sustained", d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---- algorithmic work ------------------------------------------------------
def flops_per_token_head(K, V, C, c):
    fwd = 4 * K * V + (C + 1) * K + (C + c) * V
    bwd = 8 * K * V + 2 * (C + 1) * K + 2 * (C + c) * V
    return fwd, bwd


def kernel_algo(name, B, H, T, K, V, C, c, g_bytes=4, e=2):
    """(algorithmic HBM bytes per launch, algorithmic FLOPs per launch) for one kernel launch.
    Bytes = the unique tensors the kernel must read once + write once;
    for the V-tiled backward kernels the per-V-tile dq/dk partials they exchange are counted as outputs/inputs.
    FLOPs = the algorithmic FLOPs of the method assigned to that kernel (recompute excluded)."""
    u = B * H * T          # token-heads per launch
    nvt = max(1, V // 128)
    fwd_f, bwd_f = flops_per_token_head(K, V, C, c)
    P = 2 * C                   # one bf16 row of the C x C score matrix per token
    st = 2 * 4 * K // C         # per-chunk (r, Gamma) statistics per token
    table = {
        # split forward: prep reads q, k, log alpha and writes Q~hi, K~hi, P, stats; state reads those + v, writes o
        "tc::fwd_prep": (u * (2 * e * K + g_bytes * K + 2 * e * K + P + st), u * 2 * (C + 1) * K),
        "tc::fwd_state": (u * (2 * e * K + e * V + P + st + e * V), u * (4 * K * V + (C + c) * V)),
        # split backward
        "tc::bwd_dp": (u * (2 * e * V + P), u * 2 * C * V),
        "tc::bwd_prep": (u * (2 * e * K + g_bytes * K + 2 * e * V + 2 * e * K + 2 * P + st),
                         u * (2 * (C + 1) * K + 2 * (C + 1) * V)),
        "tc::bwd_dq": (u * (e * K + 2 * e * V + P + st + nvt * e * K), u * (2 * K * V + (C + 1) * K)),
        "tc::bwd_dkv": (u * (2 * e * K + 2 * e * V + 2 * P + st + e * V + nvt * e * K),
                        u * (6 * K * V + (C + 1) * K + (C + c) * V)),
        "tc::bwd_reduce": (u * (2 * nvt * e * K + 2 * e * K + g_bytes * K + 2 * e * K + 4 * K), 0),
        # fp32 CUDA-core kernels
        "simt::k_fwd_state": (u * (2 * e * K + e * V + g_bytes * K + e * V + 4 * C), u * 4 * K * V + u * (C + 1) * V),
        "simt::k_intra_P": (u * (2 * e * K + g_bytes * K + 4 * C), u * (C + 1) * K),
        "simt::k_intra_dP": (u * (2 * e * V + 4 * C), u * (C + 1) * V),
        "simt::k_bwd_dq": (u * (e * K + e * V + g_bytes * K + e * V + 4 * C + e * K + 4 * K), u * 4 * K * V),
        "simt::k_bwd_dk": (u * (2 * e * K + e * V + g_bytes * K + e * V + 4 * C + 4 * K + e * K + 4 * K), u * 4 * K * V),
        "simt::k_bwd_dv": (u * (2 * e * K + g_bytes * K + e * V + 4 * C + e * V), u * 4 * K * V),
    }
    for key, val in table.items():
        if name.endswith(key) or name == key:
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
def cpu_oracle_sample(cfg, seed=0, n_slices=None, T_sample=None):
    """Time the fp64 oracle fwd+bwd on a bounded sample of (b,h) slices of the workload on the host cores."""
    import oracle
    import synth
    B, H, T, K, V = cfg
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:
        cores = os.cpu_count() or 1
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


# ---- main ---------------------------------------------------------------------------------------------------
def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="1p3b")
    ap.add_argument("--path", choices=["auto", "simt", "tc"], default="auto")
    ap.add_argument("--chunk", type=int, default=64)
    ap.add_argument("--subchunk", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def config_dict(args, cfg, n):
    B, H, T, K, V = cfg
    return {"workload": f"GLA core fwd+bwd, BASELINE.json configs[2] shapes ({args.config})", "model": "gla-1.3b-layer"
            if args.config == "1p3b" else f"gla-{args.config}", "global_batch": B * n, "per_gpu_batch": B, "heads": H,
            "seq_len": T, "d_k_head": K, "d_v_head": V, "chunk": args.chunk, "subchunk": args.subchunk,
            "parallelism": f"bh-shard x{n} (no data-path collective)", "gates": "logsigmoid(N(0,1))/16 fp32",
            "l2": "inputs > L2 (no flush)" if input_bytes(cfg) > 2 * L2_BYTES else "L2 flushed between steps"}


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
    for i in range(args.warmup + args.steps):
        r = cpu_oracle_sample(cfg, seed=i, n_slices=None, T_sample=T)
        if i >= args.warmup:
            vals.append(r["value"])
            base = r
    v = statistics.mean(vals)
    ms = (B * T) / v * 1e3
    line = {"metric": METRIC, "value": v, "unit": "tokens/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(args, cfg, 1),
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": base["cores"], "kind": "oracle",
                             "sample": base["sample"]},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import synth
    from paper_2312_06635_b200 import binding as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    cfg = CONFIGS[args.config]
    B, H, T, K, V = cfg
    C, c = args.chunk, args.subchunk
    p = synth.problem(B, H, T, K, V, seed=1000 * rank + 1)
    q, k, v, g, do = (p[n].to(dev) for n in ("q", "k", "v", "g", "do"))
    path = G.resolve_path(q, v, g, C, c, args.path)
    wf = G.fwd_workspace(q, v, g, C, c, args.path)
    wb = G.bwd_workspace(q, v, g, C, c, args.path)
    o = torch.empty((B, H, T, V), dtype=q.dtype, device=dev)
    grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v),
             torch.empty(q.shape, dtype=torch.float32, device=dev), None)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev) if input_bytes(cfg) <= 2 * L2_BYTES \
        else None
    stream = torch.cuda.current_stream(dev)

    def step():
        G.chunk_fwd(q, k, v, g, C, c, None, False, args.path, out=o, workspace=wf)
        G.chunk_bwd(q, k, v, g, do, C, c, None, None, False, args.path, grads=grads, workspace=wb,
                    fwd_workspace=wf)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with Clocks(local) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # per-kernel live times: a separate pass with the library's launch tracer on (it brackets every launch with
    # events and runs the two backward walks one after the other so each launch's time is its own)
    G.profile(True)
    for i in range(args.steps):
        if flush is not None:
            flush.zero_()
        step()
    torch.cuda.synchronize()
    G.lib().gla_profile_enable(0)
    prof = G.profile_read()
    launches = G.lib().gla_profile_count()
    prof_ms = sum(v_[0] for v_ in prof.values()) / args.steps
    total_ms = sum(a.elapsed_time(b) for a, b in evs)
    t = torch.tensor([total_ms], device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_step = total_ms / args.steps
    tokens = B * T * world
    value = tokens / (ms_step / 1e3)

    # e2e through the public API with pinned host buffers: every step copies its inputs host -> device and all of
    # its results device -> host.  The copies are pipelined against the compute the way a training input / output
    # pipeline would run them (H2D of step n+1 and D2H of step n-1 on their own streams while step n computes;
    # inputs and outputs double-buffered on the device), so the step time is bounded by PCIe, not by the sum.
    e2e = None
    if not args.no_e2e:
        hq, hk, hv, hg, hdo = (x.cpu().pin_memory() for x in (q, k, v, g, do))
        ho = torch.empty(o.shape, dtype=o.dtype).pin_memory()
        hgr = [torch.empty(x.shape, dtype=x.dtype).pin_memory() for x in grads[:4]]
        n_e2e = max(2, min(args.steps, 10))
        h2d = sum(x.numel() * x.element_size() for x in (hq, hk, hv, hg, hdo))
        d2h = ho.numel() * ho.element_size() + sum(x.numel() * x.element_size() for x in hgr)
        dd = [[torch.empty_like(x) for x in (q, k, v, g, do)] for _ in range(2)]
        outs = [[torch.empty_like(o)] + [torch.empty_like(x) for x in grads[:4]] for _ in range(2)]
        s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev = {k_: [torch.cuda.Event() for _ in range(2)] for k_ in ("in_ready", "in_free", "out_ready", "out_free")}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        s_h2d.wait_stream(stream)
        s_d2h.wait_stream(stream)
        for n in range(n_e2e):
            bb = n & 1
            with torch.cuda.stream(s_h2d):
                if n >= 2:
                    s_h2d.wait_event(ev["in_free"][bb])
                for dst, src in zip(dd[bb], (hq, hk, hv, hg, hdo)):
                    dst.copy_(src, non_blocking=True)
                ev["in_ready"][bb].record(s_h2d)
            stream.wait_event(ev["in_ready"][bb])
            if n >= 2:
                stream.wait_event(ev["out_free"][bb])
            x = dd[bb]
            ob = outs[bb]
            G.chunk_fwd(x[0], x[1], x[2], x[3], C, c, None, False, args.path, out=ob[0], workspace=wf)
            G.chunk_bwd(x[0], x[1], x[2], x[3], x[4], C, c, None, None, False, args.path,
                        grads=(ob[1], ob[2], ob[3], ob[4], None), workspace=wb, fwd_workspace=wf)
            ev["in_free"][bb].record(stream)
            ev["out_ready"][bb].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev["out_ready"][bb])
                for dst, src in zip([ho] + hgr, ob):
                    dst.copy_(src, non_blocking=True)
                ev["out_free"][bb].record(s_d2h)
        stream.wait_stream(s_d2h)
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1) / n_e2e], device=dev)
        if dist:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": tokens / (float(et.item()) / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": float(et.item()), "steps": n_e2e,
               "overlap": "H2D(n+1) and D2H(n-1) overlap compute(n); pipeline fill and drain included"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    hbm, tf_burst, tf_sus, peak_src = load_peaks()
    ncu = {}
    try:   # per-launch DRAM bytes of each kernel from the committed `ncu --set full` capture (profiles/)
        ncu = json.load(open(os.path.join(ROOT, "profiles", "r1_ncu_summary.json")))
    except Exception:
        pass

    def traffic_of(name):
        key = {"tc::fwd_prep": "k_fwd_prep<", "tc::fwd_state": "k_fwd_state<",
               "tc::bwd_prep": "k_bwd_prep<", "tc::bwd_dq": "k_bwd_dq3<", "tc::bwd_dkv": "k_bwd_dkv3<",
               "tc::bwd_reduce": "k_bwd_reduce_tma<", "tc::bwd_dp": "k_bwd_dp"}.get(name)
        for n, v in ncu.items():
            if key and key in n.split("::")[-1] and (f"<{K}," in n or f"<{K}>" in n):
                return v.get("traffic_bytes")
        return None
    roof = None
    if prof:
        top = max(prof, key=lambda n: prof[n][0])
        tot, nl = prof[top]
        per_launch_s = tot / nl / 1e3
        algo = kernel_algo(top, B, H, T, K, V, C, c)
        if algo:
            by, fl = algo
            roof = {"kernel": top, "bound": "hbm", "achieved": by / per_launch_s / 1e9, "peak": hbm, "unit": "GB/s",
                    "frac": by / per_launch_s / 1e9 / hbm, "traffic": traffic_of(top), "peak_source": peak_src,
                    "algo_bytes_per_launch": by, "algo_flops_per_launch": fl,
                    "tensor_tflops": fl / per_launch_s / 1e12,
                    "share_of_step": tot / (prof_ms * args.steps) if prof_ms else None,
                    "ms_per_launch": per_launch_s * 1e3}
    fwd_f, bwd_f = flops_per_token_head(K, V, C, c)
    layer_tflops = B * H * T * (fwd_f + bwd_f) / (ms_step / 1e3) / 1e12
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16" if q.dtype == torch.bfloat16 else "f32", "data": "synthetic",
            "config": config_dict(args, cfg, world), "path": path,
            "algorithmic_tflops": layer_tflops, "frac_of_bf16_peak": layer_tflops * 1e12 / (tf_burst * 1e12),
            "roofline": roof, "kernels": {n: {"ms_total": v_[0], "launches": v_[1]} for n, v_ in prof.items()},
            "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e}
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = {k_: v_ for k_, v_ in cpu_oracle_sample(cfg, T_sample=T).items()
                                if k_ != "seconds"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
