"""Per-kernel device time of the fp32 CUDA-core (SIMT) path at the 1.3B shape -- the exact fallback behind the
guard (R9) and the fp32 debug build.  python tools/simt_breakdown.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

B, H, T, K, V = 16, 4, 2048, 256, 512
p = synth.problem(B, H, T, K, V, seed=1, gate="mixed")
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
G.chunk_fwd(q, k, v, g, 64, 16, path="simt")
G.chunk_bwd(q, k, v, g, do, 64, 16, path="simt")
torch.cuda.synchronize()
G.profile(True)
G.chunk_fwd(q, k, v, g, 64, 16, path="simt")
G.chunk_bwd(q, k, v, g, do, 64, 16, path="simt")
torch.cuda.synchronize()
for n, (ms, c) in sorted(G.profile_read().items(), key=lambda x: -x[1][0]):
    print(f"{n:30s} {ms:9.3f} ms ({c})")
