import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2312_06635_b200 import binding as G
G.LIB_PATH = os.path.join(os.path.dirname(G.LIB_PATH), "libgla_timing.so")
import torch, synth
B, H, T, K, V = 16, 4, 2048, 256, 512
p = synth.problem(B, H, T, K, V, seed=1)
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
G.chunk_bwd(q, k, v, g, do, 64, 16)
torch.cuda.synchronize()
