"""Guard cliff: the 1.3B step (configs[2] shapes) with gates that fail the factorisation guard on
every chunk (`mixed`: half the channels at log alpha = -5), per-kernel device times (library tracer) and the
untraced step time beside the std-gate step.  python tools/cliff_breakdown.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

B, H, T, K, V = 16, 4, 2048, 256, 512
for gate in ("std", "mixed"):
    p = synth.problem(B, H, T, K, V, seed=1, gate=gate)
    q, k, v, g, do = (p[n].cuda() for n in ("q", "k", "v", "g", "do"))
    wf = G.fwd_workspace(q, v, g)

    def step():
        G.chunk_fwd(q, k, v, g, workspace=wf)
        G.chunk_bwd(q, k, v, g, do, fwd_workspace=wf)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    print(f"{gate}: {e0.elapsed_time(e1) / 10:.3f} ms per fwd+bwd step")
    G.profile(True)
    step()
    torch.cuda.synchronize()
    for n, (ms, c) in sorted(G.profile_read().items(), key=lambda x: -x[1][0]):
        print(f"    {n:30s} {ms * 1e3:9.1f} us ({c})")
    G.profile(False)
