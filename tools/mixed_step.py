"""One warm fwd+bwd step of the 1.3B configuration with `mixed` gates (every chunk on the exact path) -- the
workload for ncu captures of the exact-path kernels.  python tools/mixed_step.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

B, H, T, K, V = 16, 4, 2048, 256, 512
p = synth.problem(B, H, T, K, V, seed=1, gate=os.environ.get("GATE", "mixed"))
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
wf = G.fwd_workspace(q, v, g)
for _ in range(2):
    G.chunk_fwd(q, k, v, g, workspace=wf)
    G.chunk_bwd(q, k, v, g, do, fwd_workspace=wf)
torch.cuda.synchronize()
