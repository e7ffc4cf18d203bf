"""Small-shape run of every kernel family under compute-sanitizer (memcheck / racecheck / synccheck):
TC forward + saved backward (K-tiled dq / dk walks, dv walk, reduce), recomputing TC backward, SIMT forward +
backward, TC segment summaries, the exact path (mixed gates), decode step, the two-gate (beta) path.  python tools/sanitize_small.py  (run under compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

torch.cuda.set_device(0)
if os.environ.get("GLA_SERIAL"):   # the launch tracer runs every kernel on the caller's stream, one at a time
    G.profile(True)
for (B, H, T, K, V, gate) in [(1, 2, 256, 256, 512, "std"), (1, 1, 192, 128, 256, "std"),
                              (1, 1, 256, 256, 512, "mixed")]:   # mixed: every chunk on the exact path (R9)
    p = {n: t.cuda() for n, t in synth.problem(B, H, T, K, V, seed=0, gate=gate).items()}
    h0 = synth.state(B, H, K, V, 1).cuda()
    df = synth.state(B, H, K, V, 2).cuda()
    wf = G.fwd_workspace(p["q"], p["v"], p["g"], 64, 16, "tc")
    G.chunk_fwd(p["q"], p["k"], p["v"], p["g"], 64, 16, h0, True, "tc", workspace=wf)
    G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 64, 16, h0, df, True, "tc", fwd_workspace=wf)
    G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 64, 16, h0, df, True, "tc")
    G.state_summary(p["k"], p["v"], p["g"])
    G.dstate_summary(p["q"], p["do"], p["g"])
    torch.cuda.synchronize()
p = {n: t.cuda() for n, t in synth.problem(1, 2, 128, 64, 128, seed=0, dtype=torch.float32).items()}
G.chunk_fwd(p["q"], p["k"], p["v"], p["g"], 32, 8, None, True, "simt")
G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 32, 8, path="simt")
st = torch.zeros(1, 2, 64, 128, device="cuda")
G.recurrent_step(p["q"][:, :, 0].contiguous(), p["k"][:, :, 0].contiguous(), p["v"][:, :, 0].contiguous(),
                 p["g"][:, :, 0].contiguous(), st)
lb = synth.gates("std", 1, 2, 128, 128, seed=5).cuda()
G.chunk_fwd_beta(p["q"], p["k"], p["v"], p["g"], lb, 32, 8, None, True)
G.chunk_bwd_beta(p["q"], p["k"], p["v"], p["g"], lb, p["do"], 32, 8)
G.recurrent_step_beta(p["q"][:, :, 0].contiguous(), p["k"][:, :, 0].contiguous(), p["v"][:, :, 0].contiguous(),
                      p["g"][:, :, 0].contiguous(), lb[:, :, 0].contiguous(), st)
torch.cuda.synchronize()
print("sanitize_small: done")
