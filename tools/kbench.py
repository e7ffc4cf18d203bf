"""Quick per-direction timing of the TC path (CUDA events, inputs > L2): python tools/kbench.py [config]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

if os.environ.get("GLA_LIB"):   # A/B timing against another build of the library
    G.LIB_PATH = os.environ["GLA_LIB"]

CFG = {"1p3b": (16, 4, 2048, 256, 512), "340m": (8, 4, 2048, 128, 256), "long16k": (2, 4, 16384, 256, 512), "t4k": (8, 4, 4096, 256, 512),
       "t8k": (4, 4, 8192, 256, 512), "long32k": (1, 4, 32768, 256, 512)}
name = sys.argv[1] if len(sys.argv) > 1 else "1p3b"
B, H, T, K, V = CFG[name]
p = synth.problem(B, H, T, K, V, seed=1)
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
wf, wb = G.fwd_workspace(q, v, g), G.bwd_workspace(q, v, g)
o = torch.empty(B, H, T, V, dtype=q.dtype, device="cuda")
gr = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v), torch.empty(q.shape, device="cuda"), None)
for _ in range(3):
    G.chunk_fwd(q, k, v, g, out=o, workspace=wf)
    G.chunk_bwd(q, k, v, g, do, grads=gr, workspace=wb, fwd_workspace=wf)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    G.chunk_fwd(q, k, v, g, out=o, workspace=wf)
    G.chunk_bwd(q, k, v, g, do, grads=gr, workspace=wb, fwd_workspace=wf)
e1.record()
torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / 10
G.profile(True)
for _ in range(10):
    G.chunk_fwd(q, k, v, g, out=o, workspace=wf)
    G.chunk_bwd(q, k, v, g, do, grads=gr, workspace=wb, fwd_workspace=wf)
torch.cuda.synchronize()
res = G.profile_read()
tot = 0.0
for n, (ms, c) in sorted(res.items(), key=lambda x: -x[1][0]):
    print(f"{n:24s} {ms / c * 1e3:9.1f} us/launch")
    tot += ms / 10
print(f"{'sum of kernels':24s} {tot * 1e3:9.1f} us (concurrent kernels overlap)")
print(f"{'step (wall, no tracing)':24s} {wall * 1e3:9.1f} us   -> {B * T / (wall / 1e3) / 1e6:.2f} M tokens/s")
