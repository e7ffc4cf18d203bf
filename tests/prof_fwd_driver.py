import sys, torch
sys.path.insert(0, '.')
import synth
from paper_2312_06635_b200 import binding as G
B,H,T,K,V = 16,4,2048,256,512
p = synth.problem(B,H,T,K,V,seed=1)
pc = {n: t.cuda() for n,t in p.items()}
for _ in range(3):
    o, fs = G.chunk_fwd(pc["q"], pc["k"], pc["v"], pc["g"], 64, 16, None, False, "tc")
torch.cuda.synchronize()
