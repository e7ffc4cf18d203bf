"""One-GPU sweep for DESIGN.md / profiles: fwd+bwd tokens/s at the BASELINE.json configs (340M, 1.3B, long
sequences at fixed tokens per batch) and gla_recurrent_step decode throughput.  Device time with CUDA events,
inputs > L2 (or L2 flushed), warm-up first.  python tools/sweep.py > profiles/r1_sweep.md"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
HBM = PEAKS["hbm_gbs"]
TF = PEAKS["bf16_tflops"]
DEC = bool(os.environ.get("SWEEP_DECODE_ONLY"))   # decode table only
flush = torch.empty(256 * 2**20 // 4, device="cuda")


def timeit(fn, n=10, warm=3, do_flush=False):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(n):
        if do_flush:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return sorted(x.elapsed_time(y) for x, y in evs)[n // 2]


print("# One-GPU sweep (B200, tools/sweep.py)\n")
print("## fwd + bwd (gla_chunk_fwd + gla_chunk_bwd_saved), C = 64\n")
print("| config | B, H, T, K, V | ms / step | M tokens/s | algorithmic TFLOP/s (% of bf16 peak) |")
print("|---|---|---|---|---|")
for name, (B, H, T, K, V) in [] if DEC else [("340M (configs[1])", (8, 4, 2048, 128, 256)), ("1.3B (configs[2])", (16, 4, 2048, 256, 512)),
                              ("1.3B T=4K (configs[3])", (8, 4, 4096, 256, 512)),
                              ("1.3B T=8K (configs[3])", (4, 4, 8192, 256, 512)),
                              ("1.3B T=16K (configs[3])", (2, 4, 16384, 256, 512)),
                              ("1.3B T=32K, one GPU (configs[4] shapes)", (1, 4, 32768, 256, 512))]:
    p = synth.problem(B, H, T, K, V, seed=1)
    q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
    wf, wb = G.fwd_workspace(q, v, g), G.bwd_workspace(q, v, g)
    o = torch.empty(B, H, T, V, dtype=q.dtype, device="cuda")
    gr = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty(q.shape, device="cuda"), None)
    small = B * H * T * (4 * K + 4 * V + 4 * K) < 2 * 126 * 2**20

    def step():
        G.chunk_fwd(q, k, v, g, out=o, workspace=wf)
        G.chunk_bwd(q, k, v, g, do, grads=gr, workspace=wb, fwd_workspace=wf)
    ms = timeit(step, do_flush=small)
    C, c = 64, 16
    fl = B * H * T * ((4 * K * V + (C + 1) * K + (C + c) * V) + (8 * K * V + 2 * (C + 1) * K + 2 * (C + c) * V))
    print(f"| {name} | {B}, {H}, {T}, {K}, {V} | {ms:.3f} | {B * T / ms / 1e3:.1f} | "
          f"{fl / ms / 1e9:.0f} ({100 * fl / ms / 1e9 / TF:.1f} %) |")
    del q, k, v, g, do, wf, wb, o, gr
    torch.cuda.empty_cache()

print("\n## Guard cliff: the same 1.3B step with `mixed` gates (half the channels log alpha = -5: every chunk fails "
      "the factorisation guard, DESIGN.md R9)\n")
print("| gates | ms / step | M tokens/s |")
print("|---|---|---|")
for gate in (() if DEC else ("std", "mixed")):
    B, H, T, K, V = 16, 4, 2048, 256, 512
    p = synth.problem(B, H, T, K, V, seed=1, gate=gate)
    q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
    wf, wb = G.fwd_workspace(q, v, g), G.bwd_workspace(q, v, g)
    o = torch.empty(B, H, T, V, dtype=q.dtype, device="cuda")
    gr = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty(q.shape, device="cuda"), None)

    def step():
        G.chunk_fwd(q, k, v, g, out=o, workspace=wf)
        G.chunk_bwd(q, k, v, g, do, grads=gr, workspace=wb, fwd_workspace=wf)
    ms = timeit(step, n=3, warm=1)
    print(f"| {gate} | {ms:.3f} | {B * T / ms / 1e3:.1f} |")
    del q, k, v, g, do, wf, wb, o, gr
    torch.cuda.empty_cache()

print("\n## Decode: gla_recurrent_step (fp32 state read + written once per step), H = 4, K = 256, V = 512; "
      "20 steps per CUDA graph replay, each step on a different state buffer of a >= 512 MB pool (so every "
      "step's state comes from HBM, not from the 126 MB L2)\n")
print("| B | us / step | M head-steps/s | state GB/s | % of HBM copy peak |")
print("|---|---|---|---|---|")
for B in (1, 16, 64, 256):
    H, K, V = 4, 256, 512
    qt = torch.randn(B, H, K, device="cuda").bfloat16()
    kt = torch.randn(B, H, K, device="cuda").bfloat16()
    vt = torch.randn(B, H, V, device="cuda").bfloat16()
    gt = torch.nn.functional.logsigmoid(torch.randn(B, H, K, device="cuda")) / 16
    nst = max(20, -(-512 * 2**20 // (B * H * K * V * 4)))
    sts = [torch.zeros(B, H, K, V, device="cuda") for _ in range(nst)]
    out = torch.empty(B, H, V, device="cuda", dtype=torch.bfloat16)
    # 20 steps captured in a CUDA graph and replayed: device time per step without host launch overhead
    s_ = torch.cuda.Stream()
    s_.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s_):
        for i in range(3):
            G.recurrent_step(qt, kt, vt, gt, sts[i], out)
    torch.cuda.current_stream().wait_stream(s_)
    graphs = []
    for r in range(nst // 20):
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(20):
                G.recurrent_step(qt, kt, vt, gt, sts[20 * r + i], out)
        graphs.append(graph)
    it = [0]

    def replay():
        graphs[it[0] % len(graphs)].replay()
        it[0] += 1
    ms = timeit(replay, n=20, warm=3) / 20
    by = B * H * K * V * 8
    print(f"| {B} | {ms * 1e3:.1f} | {B * H / ms / 1e3:.2f} | {by / ms / 1e6:.0f} | {100 * by / ms / 1e6 / HBM:.1f} |")
