"""Strict normwise errors (max |x - y| / max |y| per (b,h) slice, worst slice) of every gradient of the product
path -- forward with saved operands + gla_chunk_bwd_saved (K-tiled walks, reduce) -- against the fp64 oracle at the
BASELINE.json lengths, and of the recomputing backward for comparison.  python tools/dlog_err.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import synth
from paper_2312_06635_b200 import binding as G

if os.environ.get("GLA_LIB"):   # another build of the library (variants/)
    G.LIB_PATH = os.environ["GLA_LIB"]


def nerr(x, y):
    x = x.float().cpu().double().numpy()
    return max(float(np.max(np.abs(x[b, h] - y[b, h])) / np.max(np.abs(y[b, h])))
               for b in range(y.shape[0]) for h in range(y.shape[1]))


print("| T | path | dq | dk | dv | d log alpha |")
print("|---|---|---|---|---|---|")
for T in (2048, 4096, 16384):
    B, H, K, V = 1, 2, 256, 512
    p = synth.problem(B, H, T, K, V, seed=3)
    pc = {n: t.cuda() for n, t in p.items()}
    f = {n: p[n].double().numpy() for n in ("q", "k", "v", "g", "do")}
    ref = oracle.bwd(f["q"], f["k"], f["v"], f["g"], f["do"])
    wf = G.fwd_workspace(pc["q"], pc["v"], pc["g"])
    G.chunk_fwd(pc["q"], pc["k"], pc["v"], pc["g"], workspace=wf)
    saved = G.chunk_bwd(pc["q"], pc["k"], pc["v"], pc["g"], pc["do"], fwd_workspace=wf)
    recomp = G.chunk_bwd(pc["q"], pc["k"], pc["v"], pc["g"], pc["do"], 64, 16, path="tc")
    torch.cuda.synchronize()
    for name, got in (("saved (bench)", saved), ("recomputing", recomp)):
        e = [nerr(x, y) for x, y in zip(got[:4], ref[:4])]
        print(f"| {T} | {name} | " + " | ".join(f"{v:.2e}" for v in e) + " |")
