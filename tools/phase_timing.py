"""Runs the forward and backward once with the -DGLA_PHASE_TIMING build (libgla_timing.so): the walk kernels
print per-chunk event traces (clock64 cycles) of CTA (0,0)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_06635_b200 import binding as G

G.LIB_PATH = os.path.join(os.path.dirname(G.LIB_PATH), "libgla_timing.so")
import torch  # noqa: E402

import synth  # noqa: E402

CFG = {"1p3b": (16, 4, 2048, 256, 512), "340m": (8, 4, 2048, 128, 256)}
B, H, T, K, V = CFG[sys.argv[1] if len(sys.argv) > 1 else "1p3b"]
p = synth.problem(B, H, T, K, V, seed=1)
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
G.chunk_fwd(q, k, v, g, 64, 16)
torch.cuda.synchronize()
if "--bwd" in sys.argv:
    G.chunk_bwd(q, k, v, g, do, 64, 16)
    torch.cuda.synchronize()
