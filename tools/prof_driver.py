"""Driver for ncu captures: python tools/prof_driver.py [fwd|bwd] [config]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

what = sys.argv[1] if len(sys.argv) > 1 else "fwd"
CFG = {"1p3b": (16, 4, 2048, 256, 512), "340m": (8, 4, 2048, 128, 256)}
B, H, T, K, V = CFG[sys.argv[2] if len(sys.argv) > 2 else "1p3b"]
p = synth.problem(B, H, T, K, V, seed=1)
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
for _ in range(3):
    if what in ("fwd", "all"):
        G.chunk_fwd(q, k, v, g, 64, 16)
    if what in ("bwd", "all"):
        G.chunk_bwd(q, k, v, g, do, 64, 16)
torch.cuda.synchronize()
