import sys, os
sys.path.insert(0, os.getcwd())
import torch, synth
from paper_2312_06635_b200 import binding as G
B, H, T, K, V = 16, 4, 2048, 256, 512
p = synth.problem(B, H, T, K, V, seed=1, gate="mixed")
q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
wf = G.fwd_workspace(q, v, g)
for _ in range(2):
    G.chunk_fwd(q, k, v, g, workspace=wf); G.chunk_bwd(q, k, v, g, do, fwd_workspace=wf)
torch.cuda.synchronize()
G.profile(True)
G.chunk_fwd(q, k, v, g, workspace=wf); G.chunk_bwd(q, k, v, g, do, fwd_workspace=wf)
torch.cuda.synchronize()
for n, (ms, c) in sorted(G.profile_read().items(), key=lambda x: -x[1][0]):
    print(f"{n:30s} {ms:9.3f} ms ({c})")
