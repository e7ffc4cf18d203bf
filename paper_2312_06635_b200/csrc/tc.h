// tc.h -- host-side interface of the tensor-core (tcgen05/TMEM/TMA, sm_100a) kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>

#include "simt.h"

namespace gla {
namespace tc {
bool supported(int B, int H, int T, int K, int V, int C, int c, int qkv_dtype, int gate_dtype);
cudaError_t fwd(const Problem& p, cudaStream_t st);
cudaError_t bwd(const BwdProblem& p, cudaStream_t st);
size_t fwd_ws(int B, int H, int T, int K, int V, int C);
size_t bwd_ws(int B, int H, int T, int K, int V, int C);
// 2-D bf16 TMA map over a [rows][cols] row-major tensor, box {64 cols, 64 rows}, optional 128B swizzle.
// d log alpha carry re-anchored from exact states every ANCH chunks (R12).
#ifndef GLA_ANCH
#define GLA_ANCH 8
#endif
constexpr int ANCH = GLA_ANCH;
// The per-chunk operands a TC forward (tc_fwd2.cu) leaves in its workspace, reused by the backward.
struct FwdSaved {
    const void *Qt, *Kt, *Pm;     // Q~hi, K~hi [B*H*T, K] bf16; P [B*H*T, 64] bf16
    const float* stats;           // (r, Gamma) per (b,h, chunk) [B*H, T/64, 2, K] fp32
    const int* flags;             // per-chunk exact-path flags [B*H, T/64]
    const void* anch;             // bf16(H_i e^{r_i}) at chunks i = ANCH, 2 ANCH, ...: [(T/64-1)/ANCH, B*H, V, K]
    const float* h0v;             // segment-entry states [B*H*S, K, V] fp32 (S > 1 only)
    int S;                        // intra-GPU segments the forward used (fwd_segments)
};
// Intra-GPU segment split of long sequences: the walks run over B*H*S virtual units of T/S
// tokens each -- the same [B*H*T, D] rows, since unit (b,h) segment s starts at row (b*H + h)*T + s*T/S.
// Used when the unsplit walks fill at most a quarter of the SMs (S doubles while the split walks still fit in one
// wave and every segment keeps >= 8 chunks; S >= 4, else 1), or at most half of them with segments of >= 32
// chunks (S = 2).  GLA_SEGMENTS=1 disables it.
int fwd_segments(int BH, int V, int NC);
// With S > 1 segments, each segment's summary contraction is split over seg_parts() token ranges (partial sums
// added in a fixed order by the chains), so the summary kernels fill the SMs (1 when S == 1).
int seg_parts(int BH, int K, int V, int NC, int S);
// Sequential state chains over the segments of every (b,h): forward H_{s+1} = e^{D_s} H_s + S_loc_s
// (writes H_s for every s; H_0 = h0 or 0), backward dF_{s-1} = e^{D_s} dF_s + dh_loc_s (dF_{S-1} = dfinal or 0).
// D_s = sum of the chunk totals Gamma over segment s, read from the prep statistics.
// Segment summaries as one tensor-core contraction per (128 channels, 256 values, segment) (tc_fwd2.cu):
// adj = false: out = each segment's end state from a zero start (mA = K~hi map, mB = v map);
// adj = true: out = each segment's d_initial_state with a zero d_final_state (mA = Q~hi map, mB = dO map).
bool seg_summary_ok(int K, int V);
// The K-tiled walks (tc_kwalk.cu): channels on the TMEM lanes, value halves of 256 per CTA (a 2-CTA cluster at
// V = 512 that sums the halves through distributed shared memory).  Each writes the unscaled fp32 rows
// [units*T][K] summed over all values (dq: forward walk, with dfinal also the final-state row sums
// stdot [V/256][units][K]; dk: reverse walk).  The reduce kernel applies e^{+-(b - r)} and forms d log alpha.
bool kwalk_ok(int K, int V);
cudaError_t dq_kwalk(int K, int V, const CUtensorMap& mK, const CUtensorMap& mDP, const CUtensorMap& mV,
                     const CUtensorMap& mD, const float* stats, const float* h0, const float* dfinal, float* dq32,
                     float* stdot, const int* flag, const int* cflags, int T, int units, cudaStream_t st);
cudaError_t dk_kwalk(int K, int V, const CUtensorMap& mQ, const CUtensorMap& mDP, const CUtensorMap& mD,
                     const CUtensorMap& mV, const float* stats, const float* dfinal, float* dk32, const int* flag,
                     const int* cflags, int T, int units, cudaStream_t st);
// skip_edge (segment split only): the last segment's summary (adj = false) / the first one's (adj = true) is not
// computed -- the chains never read it.
cudaError_t seg_summary(const CUtensorMap& mB, const CUtensorMap& mA, const float* stats, const int* flags, float* out,
                        int K, int V, int Tv, int S, int units, bool adj, cudaStream_t st, bool skip_edge = false,
                        int parts = 1, float* dec = nullptr);
cudaError_t seg_chain_fwd(const float* stats, const float* h0, const float* S_loc, float* Hv, int BH, int S, int NC,
                          int K, int V, cudaStream_t st, int parts = 1, const float* dec = nullptr);
cudaError_t seg_chain_bwd(const float* stats, const float* dfinal, const float* dh_loc, float* dFv, int BH, int S,
                          int NC, int K, int V, cudaStream_t st, int parts = 1, const float* dec = nullptr);
// TC segment summaries of a whole [B,H,T] call (gla_state_summary / gla_dstate_summary): p.q, p.k, p.g as in the
// forward (adj: p.k may alias p.q), B_op = v (adj = false) or d_out (adj = true); workspace p.ws of fwd_ws size.
bool summary_tc_ok(int K, int V);
cudaError_t summary_tc(const Problem& p, const void* B_op, float* out, float* log_decay, bool adj, cudaStream_t st);
FwdSaved fwd2_saved(const void* ws, int B, int H, int T, int K, int V);
bool fwd_is_split();              // the forward leaves its per-chunk operands in the workspace (always)
bool saved_anchors();             // false when GLA_SERIAL_WALKS=1: the forward saves no anchor states and the
                                  // backward walks run one after the other (A/B measurements)

// Number of SMs of the current device (cached; persistent kernels size their grids with it).
int num_sms();
cudaError_t make_map_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, bool swizzle);
// General 2-D map: bf16 (elem_bytes 2) or fp32 (4) [rows][cols] row-major, box {box_cols, box_rows}.
cudaError_t make_map_2d_ex(CUtensorMap* map, const void* base, int elem_bytes, uint64_t rows, uint64_t cols,
                           uint32_t box_cols, uint32_t box_rows, bool swizzle);
}  // namespace tc
}  // namespace gla
