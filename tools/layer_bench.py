"""Full GLA layer (`paper_2312_06635_b200.layer.GLALayer`) forward + backward at the paper's
layer shapes (d_k = d/2, d_v = d, 4 heads, rank-16 gate): tokens/s of the whole layer and the share
of its time spent in the chunk-wise core (the library's kernels, traced) vs the projection GEMMs (cuBLAS).
Device time, CUDA events, warm.  python tools/layer_bench.py [d_model batch seq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_06635_b200 import binding as G

if os.environ.get("GLA_LIB"):   # another build of the library (variants/)
    G.LIB_PATH = os.environ["GLA_LIB"]
from paper_2312_06635_b200.layer import GLALayer

d = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
T = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
layer = GLALayer(d, 4, device="cuda")
x = torch.randn(B, T, d, device="cuda", dtype=torch.bfloat16, requires_grad=True)
dy = torch.randn(B, T, d, device="cuda", dtype=torch.bfloat16)


def step():
    y = layer(x)
    y.backward(dy)


for _ in range(3):
    step()
torch.cuda.synchronize()
n = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
G.profile(True)
step()
torch.cuda.synchronize()
prof = G.profile_read()
G.profile(False)
lib_ms = sum(v[0] for v in prof.values())
core = {k: v[0] for k, v in prof.items() if k.startswith("tc::") or k.startswith("simt::")}
print(f"GLA layer d={d} H=4 B={B} T={T}: {ms:.3f} ms per fwd+bwd step, {B * T / ms / 1e3:.1f} M tokens/s")
print(f"  library kernels (traced, serialised): {lib_ms:.3f} ms, of which the core {sum(core.values()):.3f} ms")
for k, v in sorted(prof.items(), key=lambda x: -x[1][0]):
    print(f"    {k:28s} {v[0] * 1e3:8.1f} us")
