"""Chunk-size sweep (the paper's Fig. 2 right): per chunk size C, the device time of
the forward's intra-chunk part (the score blocks P, `simt::k_intra_P`), of the inter-chunk state passing alone
(`gla_state_summary` on the SIMT path = `k_fwd_state` without outputs), of the whole forward walk
(`k_fwd_state`: state passing + cross-chunk output + P V) and of the whole backward, on the fp32 CUDA-core
kernels (the only path with a free C; the tensor-core path is built for C = 64 and is timed beside it).

python tools/chunk_sweep.py [--out profiles/r2_chunk_sweep.md]   (one B200)
"""
import argparse
import os
import sys

# the SIMT kernels' register-tiled loops exist only for C = 64: compare the plans on the same (scalar) code
os.environ.setdefault("GLA_SIMT_NOTILE", "1")

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2312_06635_b200 import binding as G

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()

B, H, T, K, V = 4, 4, 2048, 128, 128     # 32K tokens; C = 128 tiles fit the SIMT kernels' shared memory at K, V <= 128
p = {n: t.cuda() for n, t in synth.problem(B, H, T, K, V, seed=0).items()}


def timed(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    G.profile(True)                      # per-kernel times from a second, traced pass
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    per = {n: ms / c * 1e3 for n, (ms, c) in G.profile_read().items()}
    G.profile(False)
    return e0.elapsed_time(e1) / reps * 1e3, per


rows = []
for C in (8, 16, 32, 64, 128):
    c = min(16, C)
    fwd_us, fk = timed(lambda: G.chunk_fwd(p["q"], p["k"], p["v"], p["g"], C, c, None, False, "simt"), args.reps)
    st_us, sk = timed(lambda: G.state_summary(p["k"], p["v"], p["g"], C, c, path="simt"), args.reps)
    bwd_us, bk = timed(lambda: G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], C, c, path="simt"), args.reps)
    rows.append((f"simt C={C} c={c}", fk.get("simt::k_intra_P", 0.0), sk.get("simt::k_fwd_state", st_us),
                 fk.get("simt::k_fwd_state", 0.0), fwd_us, bwd_us))
    print(rows[-1], flush=True)
wf = G.fwd_workspace(p["q"], p["v"], p["g"])
tc_fwd, tk = timed(lambda: G.chunk_fwd(p["q"], p["k"], p["v"], p["g"], 64, 16, None, False, "tc", workspace=wf),
                   args.reps)
tc_bwd, tb = timed(lambda: G.chunk_bwd(p["q"], p["k"], p["v"], p["g"], p["do"], 64, 16, path="tc",
                                       fwd_workspace=wf), args.reps)
rows.append(("tc C=64 (bf16 tensor cores)", tk.get("tc::fwd_prep", 0.0), float("nan"), tk.get("tc::fwd_state", 0.0),
             tc_fwd, tc_bwd))

lines = [f"# Chunk-size sweep (f4; P:471-490 Fig. 2 right) -- B={B}, H={H}, T={T}, K={K}, V={V}, bf16 inputs, "
         f"{torch.cuda.get_device_name()}", "",
         "Device time in us per call (CUDA events of the library tracer, warm, mean of the repetitions).  "
         "`intra scores` = the intra-chunk score blocks P (k_intra_P; on the TC row the prep kernel, which also "
         "forms Q~, K~); `state passing` = the inter-chunk recurrence alone (gla_state_summary, no outputs); "
         "`forward walk` = state passing + cross-chunk output + P V.  The SIMT backward is the fp32 debug "
         "path (one CTA per (b,h) and 32-channel tile): its totals show the trend, not a tuned kernel.  "
         "The SIMT rows run the scalar loops for every C (GLA_SIMT_NOTILE=1; the register-tiled loops exist "
         "only for C = 64).", "",
         "| path / plan | intra scores | state passing | forward walk | forward total | backward total |",
         "|---|---|---|---|---|---|"]
for r in rows:
    lines.append(f"| {r[0]} | " + " | ".join("-" if x != x else f"{x:.1f}" for x in r[1:]) + " |")
txt = "\n".join(lines) + "\n"
print(txt)
if args.out:
    with open(args.out, "w") as f:
        f.write(txt)
