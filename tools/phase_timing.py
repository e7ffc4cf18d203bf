"""Runs the forward once with the -DGLA_PHASE_TIMING build (libgla_timing.so) to print per-phase cycles."""
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
q, k, v, g = (p[n].cuda() for n in ("q", "k", "v", "g"))
G.chunk_fwd(q, k, v, g, 64, 16)
torch.cuda.synchronize()
