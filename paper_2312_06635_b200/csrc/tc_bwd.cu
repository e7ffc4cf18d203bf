// tc_bwd.cu -- chunk-wise GLA backward on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// The paper gives no backward; the equations are DESIGN.md "Backward".
// Per chunk i with b = chunk-local cumsum, r = b at the middle row, Gamma = b at the last row,
// Q~ = q e^{b-r}, K~ = k e^{r-b}, E_q = e^{b-r}, E_k = e^{r-b} (per channel), dP = (dO V^T) (.) M:
//   dq = E_q (.) [ dO (H_i e^r)^T + dP K~ ]                                   (inter + intra)
//   dk = E_k (.) [ V (e^{Gamma-r} dH_{i+1})^T + dP^T Q~ ]
//   dv = P^T dO + K~ (e^{Gamma-r} dH_{i+1})        P = (Q~ K~^T) (.) M
//   dH_i = e^{r} (.) [ e^{Gamma-r} dH_{i+1} + Q~^T dO ]                      (reverse state pass)
//   d log alpha_t = sum_{s>=t} (q dq - k dk)_s + rowsum(S_T (.) dS_T)
// The d_k x d_v states are V-tiled (128 value columns per CTA, TMEM-resident), so the contractions over V
// (dO H^T, V dH^T) are computed per V tile; dq and dk are linear in them, so each CTA emits its per-tile
// partial (bf16) and the reduce kernel sums the V/128 partials in a fixed order (deterministic).
//   k_bwd_prep / k_bwd_dp : chunk-parallel operands (Q~hi, K~hi, P, dP, statistics; or only dP when the
//                           forward's operands are reused, gla_chunk_bwd_saved)
//   k_bwd_dq3  : forward walk, recomputes H in TMEM          -> dq partials, S_T . dS_T partials, anchors
//   k_bwd_dkv3 : reverse walk, dH in TMEM                    -> dv (final), dk partials, anchor carries, dh0
//   k_bwd_reduce_tma : per (b,h, 64 channels, segment)       -> dq, dk, d log alpha (carry across chunks)
// If any chunk's half-chunk log decay exceeds the factorisation guard the prep (or the forward) raises a device
// flag; the TC kernels that follow then do nothing and a gate kernel tail-launches the exact fp32 CUDA-core
// backward (simt.cu), which produces every gradient instead (no host synchronisation).
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <cuda.h>
#include <cuda_bf16.h>

#include "common.cuh"
#include "prof.h"
#include "tc.h"
#include "tc_build.cuh"
#include "tc_common.cuh"

namespace gla {
namespace tc {

namespace {
constexpr int CH = 64;
constexpr int VT = 128;
constexpr int NTH = 256;
constexpr float L2E = 1.4426950408889634f;
constexpr float GUARD = 60.f;
}  // namespace

// ---------------------------------------------------------------------------------------------------------------
// Shared pieces: the TMEM state pass and the accumulator epilogues.
// M=64 accumulator [64 t x 64 s] in TMEM -> causal-masked bf16 rows [t][s] (SW128) in smem.
// M=64 layout: row t lives in TMEM lane 32*(t/16) + t%16 (lanes 0-15 of each quarter; probe-tested).
__device__ __forceinline__ void m64_epilogue(uint32_t tcol, uint32_t lane_base, int lq, int lane, uint8_t* dst) {
    uint32_t a[32], b[32];
    tmem_ld32(tcol + lane_base, a);
    tmem_ld32(tcol + lane_base + 32, b);
    tmem_wait_ld();
    if (lane < 16) {
        const int t = 16 * lq + lane;
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 64; j += 2) {
            const float x0 = __uint_as_float(j < 32 ? a[j] : b[j - 32]);
            const float x1 = __uint_as_float(j + 1 < 32 ? a[j + 1] : b[j + 1 - 32]);
            pk[j / 2] = pack_bf16(j <= t ? x0 : 0.f, j + 1 <= t ? x1 : 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
            *reinterpret_cast<uint4*>(dst + sw128_off(t, 8 * u)) =
                make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
    }
}

// k_bwd_reduce_tma: the same computation as k_bwd_reduce, with every input tile of a chunk -- the NVT dq and dk
// partials, q, k, log alpha ([64 rows x 64 channels] each) -- staged in shared memory by TMA (SWIZZLE_128B) two
// chunks ahead, so the HBM latency of the partials overlaps the scans of the chunks in between (the register-
// prefetched version waited on its loads: ncu long-scoreboard stalls at the first use of every partial).
// NQ32 > 0: dq and dk arrive as NQ32 unscaled fp32 partials each (one per 256-value half, the K-tiled walks in
// tc_kwalk.cu), a [64 t][64 k] fp32 tile (two [64][32] SW128 boxes); NQ32 = 0: NVT bf16 V-tile partials each.
template <int NVT, typename TG, int NQ32 = 0>
struct RedCfg {
    static constexpr int NQ = NQ32 ? NQ32 : NVT;                         // dq (and dk) partial tiles per chunk
    static constexpr uint32_t TILE = 8192;                               // [64 rows][64 bf16] or [64][32 fp32]
    static constexpr uint32_t QT = NQ32 ? 2 * TILE : TILE;               // bytes of one partial tile
    static constexpr uint32_t OFF_DK = NQ * QT;                          // dk partials, then q, k, log alpha
    static constexpr uint32_t OFF_Q = 2 * NQ * QT;
    static constexpr uint32_t GT = 64 * 64 * sizeof(TG);                 // log alpha tile bytes
    static constexpr uint32_t STAGE = OFF_Q + 2 * TILE + GT;
    static constexpr uint32_t EX = NQ32 ? 3 * 64 * 68 * 4 : 0;   // exact chunks: alpha, dP, dP^T ([64][68] fp32 each)
    static constexpr int NS = 2 * STAGE + EX + 2 * 4 * 64 * 4 + 1024 <= 232448 ? 2 : 1;
    static constexpr uint32_t OFF_EX = NS * STAGE;
    static constexpr uint32_t SMEM = NS * STAGE + EX + 1024;
};

// The exact intra-chunk terms of k_bwd_reduce_tma for one flagged chunk (see there), by the reduce's 256 compute
// threads: thread (rows 4 (tid / 16) + [0, 4), channels 4 (tid % 16) + [0, 4)) runs both sums for its 4 x 4 block,
// so each step's shared loads (alpha and k or q of one row: 4 channels each; dP of 4 rows: one float4) feed 16
// terms.  In: the staged q / k tiles (SW128 bf16 [64][64]), al = alpha, dp = dP, dpT = dP^T (fp32 [64][68]).
// Out (after a barrier, so every read of al / dp is done): al <- the dq terms, dp <- the dk terms, [t][channel].
// Not inlined: its registers stay out of the reduce's common path.
__device__ __noinline__ void exact_intra(const uint8_t* qt, const uint8_t* kt, float (*al)[68], float (*dp)[68],
                                         const float (*dpT)[68]) {
    const int tid = threadIdx.x, t0 = 4 * (tid >> 4), c0 = 4 * (tid & 15);
    auto ld4 = [&](const uint8_t* tile, int u) {   // 4 bf16 channels [c0, c0 + 4) of row u of a SW128 tile
        const uint2 x = *reinterpret_cast<const uint2*>(tile + u * 128 + ((((c0 >> 3) ^ (u & 7))) << 4) + (c0 & 7) * 2);
        return make_float4(bf16lo(x.x), bf16hi(x.x), bf16lo(x.y), bf16hi(x.y));
    };
    auto ld_al = [&](int u) { return *reinterpret_cast<const float4*>(&al[u][c0]); };
    float2 w[4][2], aq[4][2], ak[4][2];   // [row][channel pair]
    auto step = [&](float4 xv, float4 d4, float4 a4, bool upd, float2 (&acc)[4][2]) {   // all 4 rows active
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (upd) { w[r][0] = mul2(w[r][0], make_float2(a4.x, a4.y)); w[r][1] = mul2(w[r][1], make_float2(a4.z, a4.w)); }
            const float2 p2 = make_float2(dv[r], dv[r]);
            acc[r][0] = fma2(mul2(p2, make_float2(xv.x, xv.y)), w[r][0], acc[r][0]);
            acc[r][1] = fma2(mul2(p2, make_float2(xv.z, xv.w)), w[r][1], acc[r][1]);
        }
    };
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) { w[r][h] = make_float2(1.f, 1.f); aq[r][h] = make_float2(0.f, 0.f); }
    // dq_t = sum_{s <= t} dP[t][s] k_s e^{b_t - b_s}: s from t0 + 3 down; row t joins at s = t with w = 1, and
    // w_t <- w_t alpha_{s+1} for s < t.  The ragged head (s >= t0: rows joining) first, then the rest.
#pragma unroll
    for (int j = 3; j >= 0; --j) {
        const int s2 = t0 + j;
        const float4 kv = ld4(kt, s2), d4 = *reinterpret_cast<const float4*>(&dpT[s2][t0]);
        const float4 a4 = j < 3 ? ld_al(s2 + 1) : make_float4(1.f, 1.f, 1.f, 1.f);
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r < j) continue;
            if (r > j) { w[r][0] = mul2(w[r][0], make_float2(a4.x, a4.y)); w[r][1] = mul2(w[r][1], make_float2(a4.z, a4.w)); }
            const float2 p2 = make_float2(dv[r], dv[r]);
            aq[r][0] = fma2(mul2(p2, make_float2(kv.x, kv.y)), w[r][0], aq[r][0]);
            aq[r][1] = fma2(mul2(p2, make_float2(kv.z, kv.w)), w[r][1], aq[r][1]);
        }
    }
#pragma unroll 1
    for (int s2 = t0 - 1; s2 >= 0; --s2)
        step(ld4(kt, s2), *reinterpret_cast<const float4*>(&dpT[s2][t0]), ld_al(s2 + 1), true, aq);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int h = 0; h < 2; ++h) { w[r][h] = make_float2(1.f, 1.f); ak[r][h] = make_float2(0.f, 0.f); }
    // dk_t = sum_{u >= t} dP[u][t] q_u e^{b_u - b_t}: u from t0 up; row t joins at u = t, w_t <- w_t alpha_u for u > t
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const int u2 = t0 + j;
        const float4 qv = ld4(qt, u2), d4 = *reinterpret_cast<const float4*>(&dp[u2][t0]);
        const float4 a4 = j > 0 ? ld_al(u2) : make_float4(1.f, 1.f, 1.f, 1.f);
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r > j) continue;
            if (r < j) { w[r][0] = mul2(w[r][0], make_float2(a4.x, a4.y)); w[r][1] = mul2(w[r][1], make_float2(a4.z, a4.w)); }
            const float2 p2 = make_float2(dv[r], dv[r]);
            ak[r][0] = fma2(mul2(p2, make_float2(qv.x, qv.y)), w[r][0], ak[r][0]);
            ak[r][1] = fma2(mul2(p2, make_float2(qv.z, qv.w)), w[r][1], ak[r][1]);
        }
    }
    {   // u = t0 + 3: row t0 + 3 joins (w = 1), the others decay
        const int u2 = t0 + 3;
        const float4 qv = ld4(qt, u2), d4 = *reinterpret_cast<const float4*>(&dp[u2][t0]), a4 = ld_al(u2);
        const float dv[4] = {d4.x, d4.y, d4.z, d4.w};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (r < 3) { w[r][0] = mul2(w[r][0], make_float2(a4.x, a4.y)); w[r][1] = mul2(w[r][1], make_float2(a4.z, a4.w)); }
            const float2 p2 = make_float2(dv[r], dv[r]);
            ak[r][0] = fma2(mul2(p2, make_float2(qv.x, qv.y)), w[r][0], ak[r][0]);
            ak[r][1] = fma2(mul2(p2, make_float2(qv.z, qv.w)), w[r][1], ak[r][1]);
        }
    }
#pragma unroll 1
    for (int u2 = t0 + 4; u2 < 64; ++u2)
        step(ld4(qt, u2), *reinterpret_cast<const float4*>(&dp[u2][t0]), ld_al(u2), true, ak);
    named_bar_sync(1, 256);   // every read of al / dp done
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        *reinterpret_cast<float4*>(&al[t0 + r][c0]) = make_float4(aq[r][0].x, aq[r][0].y, aq[r][1].x, aq[r][1].y);
        *reinterpret_cast<float4*>(&dp[t0 + r][c0]) = make_float4(ak[r][0].x, ak[r][0].y, ak[r][1].x, ak[r][1].y);
    }
    named_bar_sync(1, 256);
}

template <int K, int NVT, typename TG, int NQ32>
__global__ void __launch_bounds__(288, 1)
k_bwd_reduce_tma(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmG, const __grid_constant__ CUtensorMap tmDQP,
                 const __grid_constant__ CUtensorMap tmDKP, const float* __restrict__ stdot, int n_stdot,
                 __nv_bfloat16* __restrict__ dq, __nv_bfloat16* __restrict__ dk, float* __restrict__ dg,
                 const float* __restrict__ cpart, const int* __restrict__ flag, int T, int BH,
                 const int* __restrict__ cflags, const __nv_bfloat16* __restrict__ dPm) {
    // cflags / dPm (NQ32 only, else NULL): the forward's per-chunk exact-path flags and dP = (dO V^T) (.) M.  On a
    // flagged chunk the walks delivered the inter terms in the r = 0 frame (dq = e^{b} (.) X_q, dk = e^{Gamma - b}
    // (.) X_k) and no intra term; the intra terms are formed here in fp32 with decay factors <= 1 built as running
    // products of alpha (no exponent of a difference of cumsums, no overflow whatever the gates):
    //     dq_t += sum_{s <= t} dP[t][s] k_s e^{b_t - b_s},   dk_t += sum_{u >= t} dP[u][t] q_u e^{b_u - b_t}.
    using RC = RedCfg<NVT, TG, NQ32>;
    constexpr int NQ = RC::NQ;
    constexpr uint32_t ODK = RC::OFF_DK, OQ = RC::OFF_Q;
    if (*flag) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    __shared__ float gt_s[4][64], xt_s[4][64];   // per row group: totals of g and of q (.) dq - k (.) dk
    float (*al)[68] = reinterpret_cast<float (*)[68]>(sm + RC::OFF_EX);                    // exact chunks: alpha
    float (*sdp)[68] = reinterpret_cast<float (*)[68]>(sm + RC::OFF_EX + 64 * 68 * 4);     // exact chunks: dP
    float (*sdpT)[68] = reinterpret_cast<float (*)[68]>(sm + RC::OFF_EX + 2 * 64 * 68 * 4);   // and dP^T
    __shared__ uint64_t bar[2], empty[2];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.x * 64, bh = blockIdx.y;
    const int NC = T / CH;
    // Segment blockIdx.z: chunks [i_lo, i_hi].  The exact carries at every ANCH-th chunk boundary (cpart) make the
    // segments independent, so they run as separate CTAs (more, shorter CTAs: better wave balance).
    const int i_lo = blockIdx.z * ANCH, i_hi = min(NC, i_lo + ANCH) - 1;
    const size_t head_row = (size_t)bh * T;
    auto issue = [&](int i) {         // all input tiles of chunk i into stage i % NS
        uint8_t* st = sm + (i % RC::NS) * RC::STAGE;
        uint64_t* b = &bar[i % RC::NS];
        const int row = (int)(head_row + (size_t)i * CH);
        mbar_expect_tx(b, RC::STAGE);
        for (int j = 0; j < NQ; ++j) {
            tma_load_2d(st + j * RC::QT, &tmDQP, b, m0, row + j * BH * T);
            if (NQ32) tma_load_2d(st + j * RC::QT + RC::TILE, &tmDQP, b, m0 + 32, row + j * BH * T);
        }
        for (int j = 0; j < NQ; ++j) {
            tma_load_2d(st + ODK + j * RC::QT, &tmDKP, b, m0, row + j * BH * T);
            if (NQ32) tma_load_2d(st + ODK + j * RC::QT + RC::TILE, &tmDKP, b, m0 + 32, row + j * BH * T);
        }
        tma_load_2d(st + OQ, &tmQ, b, m0, row);
        tma_load_2d(st + OQ + RC::TILE, &tmK, b, m0, row);
        if (sizeof(TG) == 4) {
            tma_load_2d(st + OQ + 2 * RC::TILE, &tmG, b, m0, row);
            tma_load_2d(st + OQ + 2 * RC::TILE + 8192, &tmG, b, m0 + 32, row);
        } else {
            tma_load_2d(st + OQ + 2 * RC::TILE, &tmG, b, m0, row);
        }
    };
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        mbar_init(&empty[0], 1);
        mbar_init(&empty[1], 1);
        fence_mbar_init();
        prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmG); prefetch_tmap(&tmDQP); prefetch_tmap(&tmDKP);
    }
    __syncthreads();
    if (tid >= 256) {                          // producer warp: keeps the ring of stages full (one lane issues)
        if (tid == 256) {
            uint32_t n = 0;
            for (int c = i_hi; c >= i_lo; --c, ++n) {
                const int slot = c % RC::NS;
                if (n >= (uint32_t)RC::NS) mbar_wait(&empty[slot], ((n / RC::NS) - 1) & 1);
                issue(c);
            }
        }
        return;
    }
    // Thread layout of the scans: channel ch = tid % 64 of the CTA's 64, rows [16 rg, 16 rg + 16) of the chunk with
    // rg = tid / 64.  Both scans (the chunk-local cumsum b, the reverse cumsum of q (.) dq - k (.) dk) run in
    // registers over the thread's 16 rows; the four row groups of a channel combine their totals through shared
    // memory (one barrier per scan).  The carry of later chunks lives in every thread's registers.
    const int ch = tid & 63, rg = tid >> 6, t0 = 16 * rg;
    float carry = 0.f;    // d log alpha carry entering the current chunk from above, channel m0 + ch
    if (i_hi == NC - 1) {
        if (stdot)
            for (int j = 0; j < n_stdot; ++j) carry += stdot[((size_t)j * BH + bh) * K + m0 + ch];
    } else {
        const size_t a2 = (i_hi + 1) / ANCH - 1;
        for (int j = 0; j < NVT; ++j) carry += cpart[((a2 * NVT + j) * BH + bh) * K + m0 + ch];
    }
    __shared__ int slow_s[ANCH];      // exact-path flags of this segment's chunks
    if (NQ32 && tid < ANCH)
        slow_s[tid] = (cflags && i_lo + tid <= i_hi) ? cflags[(size_t)bh * NC + i_lo + tid] : 0;
    named_bar_sync(1, 256);
    uint32_t slow_bits = 0u;
    if (NQ32)
#pragma unroll
        for (int c = 0; c < ANCH; ++c) slow_bits |= (slow_s[c] ? 1u : 0u) << c;
    uint32_t uses[2] = {0u, 0u};
    // byte offset of element (row u, channel ch) in a SW128 [64][64] bf16 tile / in a pair of [64][32] fp32 boxes
    auto bf_at = [&](int u) { return (uint32_t)(u * 128 + ((((ch >> 3) ^ (u & 7))) << 4) + (ch & 7) * 2); };
    auto f32_at = [&](int u) {
        return (uint32_t)((ch >> 5) * RC::TILE + u * 128 + (((((ch & 31) >> 2) ^ (u & 7))) << 4) + (ch & 3) * 4);
    };
    auto ldbf = [](const uint8_t* p) { return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p)); };
    for (int i = i_hi; i >= i_lo; --i) {
        const int sidx = i % RC::NS;
        const uint8_t* st = sm + sidx * RC::STAGE;
        if (i + 1 < NC && (i + 1) % ANCH == 0) {   // exact carry rowsum(H_{i+1} (.) dH_{i+1})
            const size_t a = (i + 1) / ANCH - 1;
            carry = 0.f;
            for (int j = 0; j < NVT; ++j) carry += cpart[((a * NVT + j) * BH + bh) * K + m0 + ch];
        }
        mbar_wait(&bar[sidx], (uses[sidx]++) & 1);
        const bool slow = NQ32 && ((slow_bits >> (i - i_lo)) & 1u);
        // (a1) chunk-local cumsum over the thread's rows, then the offset of the earlier row groups
        float b[16];
        {
            const uint8_t* gt = st + OQ + 2 * RC::TILE;
            float run = 0.f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const float gv = sizeof(TG) == 4 ? *reinterpret_cast<const float*>(gt + f32_at(t0 + j))
                                                 : ldbf(gt + bf_at(t0 + j));
                if (NQ32 && slow) al[t0 + j][ch] = ex2f(gv * L2E);
                run += gv;
                b[j] = run;
            }
            gt_s[rg][ch] = run;
            if (NQ32 && slow) {   // dP rows [t0, t0 + 16), key column ch (dP is token x token)
                const __nv_bfloat16* dr = dPm + (head_row + (size_t)i * CH + t0) * 64 + ch;
#pragma unroll 4
                for (int j = 0; j < 16; ++j) sdp[t0 + j][ch] = sdpT[ch][t0 + j] = __bfloat162float(dr[(size_t)j * 64]);
            }
        }
        named_bar_sync(1, 256);
        float pre = 0.f;
#pragma unroll
        for (int g2 = 0; g2 < 3; ++g2) pre += g2 < rg ? gt_s[g2][ch] : 0.f;
        const float r = gt_s[0][ch] + gt_s[1][ch];            // b at row CH / 2 - 1
        const float gam = r + gt_s[2][ch] + gt_s[3][ch];      // b at row CH - 1
#pragma unroll
        for (int j = 0; j < 16; ++j) b[j] += pre;
        // exact-path chunk: the r = 0 frame for dq, r = Gamma for dk, plus the exact intra terms
        const float rq = slow ? 0.f : r, rk = slow ? gam : r;
        if (NQ32 && slow) exact_intra(st + OQ, st + OQ + RC::TILE, al, sdp, sdpT);   // (all 256 threads)
        float x[16];
        const size_t ix0 = (head_row + (size_t)i * CH + t0) * K + m0 + ch;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int u = t0 + j;
            float sq = 0.f, sk = 0.f;
#pragma unroll
            for (int p = 0; p < NQ; ++p) {
                if (NQ32) {
                    sq += *reinterpret_cast<const float*>(st + p * RC::QT + f32_at(u));
                    sk += *reinterpret_cast<const float*>(st + ODK + p * RC::QT + f32_at(u));
                } else {
                    sq += ldbf(st + p * RC::TILE + bf_at(u));
                    sk += ldbf(st + ODK + p * RC::TILE + bf_at(u));
                }
            }
            float dqv = sq * ex2f((b[j] - rq) * L2E), dkv = sk * ex2f((rk - b[j]) * L2E);
            if (NQ32 && slow) { dqv += al[u][ch]; dkv += sdp[u][ch]; }
            x[j] = ldbf(st + OQ + bf_at(u)) * dqv - ldbf(st + OQ + RC::TILE + bf_at(u)) * dkv;
            dq[ix0 + (size_t)j * K] = __float2bfloat16_rn(dqv);
            dk[ix0 + (size_t)j * K] = __float2bfloat16_rn(dkv);
        }
        // reverse cumsum of x over the thread's rows; the later row groups' totals and the carry come next
        float run = 0.f;
#pragma unroll
        for (int j = 15; j >= 0; --j) { run += x[j]; x[j] = run; }
        xt_s[rg][ch] = run;
        named_bar_sync(1, 256);            // every read of the stage (and of al / sdp) is done, xt_s complete
        if (tid == 0) mbar_arrive(&empty[sidx]);   // the producer may refill this stage
        float post = carry;
#pragma unroll
        for (int g2 = 1; g2 < 4; ++g2) post += g2 > rg ? xt_s[g2][ch] : 0.f;
        carry += (xt_s[0][ch] + xt_s[1][ch]) + (xt_s[2][ch] + xt_s[3][ch]);
#pragma unroll
        for (int j = 0; j < 16; ++j) dg[ix0 + (size_t)j * K] = x[j] + post;
    }
}

// ===============================================================================================================
// Split backward (default): k_bwd_prep (chunk-parallel) computes, once per (b,h, chunk), the chunk-local cumsum
// statistics, Q~hi, K~hi, P = (Q~ K~^T) (.) M (stacked hi/lo MMA) and dP = (dO V^T) (.) M over the full V
// (TMA-streamed in 256-wide rounds); the two V-tiled walks are then fed entirely by TMA, and the intra-chunk terms
// K~^T dP^T and Q~^T dP are added by the V tile 0 CTA only (dq, dk are sums over V tiles).
template <int K>
struct BPrepCfg {
    using Tl = Tile<K>;
    static constexpr int KB = K / 64;
    static constexpr uint32_t OP = KB * 16384;            // [KB][128 rows: hi | lo][128 B]
    static constexpr uint32_t OFF_Q = 0, OFF_K = OP;
    static constexpr uint32_t OFF_D = 2 * OP;             // dO round: [4][64 t][128 B]
    static constexpr uint32_t OFF_V = OFF_D + 32768;      // V round:  [4][64 t][128 B]
    static constexpr uint32_t OFF_P = OFF_V + 32768;      // P  [64 t][128 B]
    static constexpr uint32_t OFF_DP = OFF_P + 8192;      // dP [64 t][128 B]
    static constexpr uint32_t OFF_X = OFF_DP + 8192;      // fp32 exchange [64][64] / cumsum exchange
    static constexpr uint32_t SMEM = OFF_X + 16384 + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
};

// Persistent like k_fwd_prep: CTA c processes work items (b,h, chunk) c, c + gridDim.x, ...; the next item's
// q / k / log alpha go into the dead operand registers after the build, and its first dO / V round is loaded
// by TMA while this item's epilogue runs.
template <int K, typename TG>
__global__ void __launch_bounds__(NTH, 1)
k_bwd_prep(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmDP,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmD,
           const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, const TG* __restrict__ g,
           float* __restrict__ stats, int* __restrict__ flag, int T, int V, int NC, int nitems) {
    using Cfg = BPrepCfg<K>;
    using Tl = typename Cfg::Tl;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sQ = sm + Cfg::OFF_Q;
    uint8_t* sK = sm + Cfg::OFF_K;
    uint8_t* sD = sm + Cfg::OFF_D;
    uint8_t* sV = sm + Cfg::OFF_V;
    uint8_t* sP = sm + Cfg::OFF_P;
    uint8_t* sdP = sm + Cfg::OFF_DP;
    float* exch = reinterpret_cast<float*>(sm + Cfg::OFF_X);
    __shared__ uint64_t bar_in, bar_m, bar_done;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int oc = tid % Tl::NOCT, rg = tid / Tl::NOCT;
    const int ch0 = 8 * oc, row0 = rg * Tl::RPG;
    const int VR = V < 256 ? V : 256, NR = V / VR, NBX = VR / 64;   // V rounds of VR columns (NBX boxes)
    auto crow_of = [&](int it) { return (size_t)(it / NC) * T + (size_t)(it % NC) * CH; };
    auto load_round = [&](int it, int rd) {
        const int row = (int)crow_of(it);
        mbar_expect_tx(&bar_in, 2 * NBX * 8192);
        for (int b = 0; b < NBX; ++b) {
            tma_load_2d(sD + b * 8192, &tmD, &bar_in, rd * VR + 64 * b, row);
            tma_load_2d(sV + b * 8192, &tmV, &bar_in, rd * VR + 64 * b, row);
        }
    };

    if (warp == 0) tmem_alloc(&tmem_base, 256);
    int item = blockIdx.x;
    if (tid == 0) {
        mbar_init(&bar_in, 1);
        mbar_init(&bar_m, 1);
        mbar_init(&bar_done, 1);
        fence_mbar_init();
        if (item < nitems) load_round(item, 0);
    }
    ChunkRegs<K> R;
    if (item < nitems) load_chunk<K, TG, true, true>(R, q, k, g, crow_of(item), row0, ch0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tP = tmem_base, tdP = tmem_base + 128;
    uint32_t in_cnt = 0, m_cnt = 0, done_ph = 0;
    for (; item < nitems; item += gridDim.x, done_ph ^= 1) {
        const int chunk = item % NC, bh = item / NC;
        const size_t crow = crow_of(item);
        if (tid == 0) tma_store_wait_read();    // the previous item's stores have read their smem
        float2 off[4], rr[4], Gm[4];
        chunk_cumsum<K>(R, exch, rg, ch0, off, rr, Gm);
        bool bad = false;
        if (rg == 0)
#pragma unroll
            for (int p = 0; p < 4; ++p)
                bad |= (-rr[p].x > GUARD) | (-rr[p].y > GUARD) | (rr[p].x - Gm[p].x > GUARD) | (rr[p].y - Gm[p].y > GUARD);
        if (__syncthreads_or(bad) && tid == 0) atomicOr(flag, 1);   // whole call -> exact CUDA-core kernels
        if (rg == 0) {
            float* st = stats + ((size_t)bh * NC + chunk) * 2 * K + ch0;
            reinterpret_cast<float4*>(st)[0] = make_float4(rr[0].x, rr[0].y, rr[1].x, rr[1].y);
            reinterpret_cast<float4*>(st)[1] = make_float4(rr[2].x, rr[2].y, rr[3].x, rr[3].y);
            reinterpret_cast<float4*>(st + K)[0] = make_float4(Gm[0].x, Gm[0].y, Gm[1].x, Gm[1].y);
            reinterpret_cast<float4*>(st + K)[1] = make_float4(Gm[2].x, Gm[2].y, Gm[3].x, Gm[3].y);
        }
        float2 refq[4], refk[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            refq[p] = make_float2(-L2E * rr[p].x, -L2E * rr[p].y);
            refk[p] = make_float2(L2E * rr[p].x, L2E * rr[p].y);
        }
        const int blk = ch0 >> 6, col = ch0 & 63;
        uint8_t* qb = sQ + blk * 16384;
        uint8_t* kb = sK + blk * 16384;
#pragma unroll
        for (int r = 0; r < Tl::RPG; ++r) {
            const int t = row0 + r;
            float2 b[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) b[p] = add2(R.g[r][p], off[p]);
            scaled_row(R.q[r], b, refq, 1.f, qb + sw128_off(t, col), qb + sw128_off(64 + t, col));
            scaled_row(R.k[r], b, refk, -1.f, kb + sw128_off(t, col), kb + sw128_off(64 + t, col));
        }
        {   // next item's q / k / log alpha into the dead operand registers
            const int nx = item + gridDim.x;
            if (nx < nitems) load_chunk<K, TG, true, true>(R, q, k, g, crow_of(nx), row0, ch0);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t idPs = idesc_bf16(128, 128, 0, 0), idDP = idesc_bf16(64, 64, 0, 0);
            const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aD = smem_u32(sD), aV = smem_u32(sV);
#pragma unroll
            for (int kk = 0; kk < K / 16; ++kk) {   // P: [Q~hi; Q~lo] [K~hi; K~lo]^T
                const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
                mma_bf16(tP, sdesc_sw128(aQ + o, 16, 1024), sdesc_sw128(aK + o, 16, 1024), idPs, kk > 0);
            }
            for (int c = 0; c < K / 64; ++c) {     // Q~hi, K~hi -> HBM for the V-tiled walks
                tma_store_2d(&tmQ, sQ + c * 16384, 64 * c, (int)crow);
                tma_store_2d(&tmK, sK + c * 16384, 64 * c, (int)crow);
            }
            tma_store_commit();
            for (int rd = 0; rd < NR; ++rd) {      // dP = dO V^T over the full V, VR columns per round
                mbar_wait(&bar_in, (in_cnt++) & 1);
                tc_fence_after();
                for (int kk = 0; kk < VR / 16; ++kk) {
                    const uint32_t o = (kk >> 2) * 8192 + (kk & 3) * 32;
                    mma_bf16(tdP, sdesc_sw128(aD + o, 16, 1024), sdesc_sw128(aV + o, 16, 1024), idDP, (rd | kk) > 0);
                }
                if (rd + 1 < NR) {
                    mma_commit(&bar_m);
                    mbar_wait(&bar_m, (m_cnt++) & 1);   // the MMAs have consumed this round's tiles
                    load_round(item, rd + 1);
                }
            }
            mma_commit(&bar_done);
        }
        mbar_wait(&bar_done, done_ph);   // every MMA of this item has completed
        tc_fence_after();
        if (tid == 0 && item + (int)gridDim.x < nitems) load_round(item + gridDim.x, 0);   // overlaps the epilogue
        const int lq = warp & 3, half = warp >> 2;
        const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
        const int vrow = 32 * lq + lane;
        // dP (M=64 layout) -> causal bf16 [t][s]; the lo-row warps of P run the P exchange meanwhile
        if (half == 1) m64_epilogue(tdP, lane_base, lq, lane, sdP);
        if (lq >= 2 && half == 0) {
            for (int hc = 0; hc < 2; ++hc) {
                uint32_t a[32], b[32];
                tmem_ld32(tP + lane_base + 32 * hc, a);
                tmem_ld32(tP + lane_base + 64 + 32 * hc, b);
                tmem_wait_ld();
                const int t = vrow - 64;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    exch[t * 64 + ((32 * hc + j + t) & 63)] = __uint_as_float(a[j]) + __uint_as_float(b[j]);
            }
        }
        __syncthreads();
        if (lq < 2) {
            uint32_t a[32], b[32];
            tmem_ld32(tP + lane_base + 32 * half, a);
            tmem_ld32(tP + lane_base + 64 + 32 * half, b);
            tmem_wait_ld();
            const int t = vrow;
            uint32_t pk[16];
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
                const int s_ = 32 * half + j;
                float p0 = __uint_as_float(a[j]) + __uint_as_float(b[j]) + exch[t * 64 + ((s_ + t) & 63)];
                float p1 = __uint_as_float(a[j + 1]) + __uint_as_float(b[j + 1]) + exch[t * 64 + ((s_ + 1 + t) & 63)];
                pk[j / 2] = pack_bf16(s_ <= t ? p0 : 0.f, s_ + 1 <= t ? p1 : 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                *reinterpret_cast<uint4*>(sP + sw128_off(t, 32 * half + 8 * u)) =
                    make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();                         // P, dP staged; TMEM drained; exch free
        if (tid == 0) {
            tma_store_2d(&tmP, sP, 0, (int)crow);
            tma_store_2d(&tmDP, sdP, 0, (int)crow);
            tma_store_commit();
        }
    }
    if (tid == 0) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, 256);
}

// k_bwd_dp: dP = (dO V^T) (.) M per chunk over the full V, for the backward that reuses a forward's saved
// Q~, K~, P (gla_chunk_bwd_saved).  Persistent; warp 0 streams 64-column dO / V boxes through a 4-stage TMA
// ring, warp 1 issues the M=64 N=64 MMAs into a double-buffered accumulator (the next item's MMAs run while warps
// 2-5 drain this one: causal mask, bf16, TMA store).
// It also ORs the forward's per-chunk exact-path flags into the backward's flag (R9) when given them (the
// V-tiled walks have no exact path; the K-tiled ones and the reduce do, so the K-tiled backward passes NULL).
#ifndef GLA_ANCH_PF
#define GLA_ANCH_PF 1
#endif
#ifndef GLA_DP_GRID
#define GLA_DP_GRID 2   // bwd_dp CTAs per SM (persistent)
#endif
#ifndef GLA_DP_NSTG
#define GLA_DP_NSTG 4
#endif
constexpr int DP_NSTG = GLA_DP_NSTG;
__global__ void __launch_bounds__(192, 1)
k_bwd_dp(const __grid_constant__ CUtensorMap tmDP, const __grid_constant__ CUtensorMap tmV,
         const __grid_constant__ CUtensorMap tmD, const int* __restrict__ fflags, int* __restrict__ flag, int T,
         int V, int NC, int nitems) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sdP = sm + DP_NSTG * 16384;
    __shared__ uint64_t full[DP_NSTG], empty[DP_NSTG], acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NKB = V / 64;
    if (warp == 0) tmem_alloc(&tmem_base, 128);
    if (tid == 0) {
        for (int s2 = 0; s2 < DP_NSTG; ++s2) { mbar_init(&full[s2], 1); mbar_init(&empty[s2], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&acc_full[b], 1); mbar_init(&acc_empty[b], 1); }
        fence_mbar_init();
        prefetch_tmap(&tmDP); prefetch_tmap(&tmV); prefetch_tmap(&tmD);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tdP = tmem_base;
    if (warp == 0) {
        if (lane == 0) {
            int any = 0;
            uint32_t cnt = 0;
            for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
                const int row = (int)((size_t)(item / NC) * T + (size_t)(item % NC) * CH);
                if (fflags) any |= fflags[item];
                for (int kb = 0; kb < NKB; ++kb, ++cnt) {
                    const uint32_t s2 = cnt % DP_NSTG, use = cnt / DP_NSTG;
                    if (use > 0) mbar_wait(&empty[s2], (use - 1) & 1);
                    mbar_expect_tx(&full[s2], 16384);
                    tma_load_2d(sm + s2 * 16384, &tmD, &full[s2], 64 * kb, row);
                    tma_load_2d(sm + s2 * 16384 + 8192, &tmV, &full[s2], 64 * kb, row);
                }
            }
            if (any) atomicOr(flag, 1);
        }
    } else if (warp == 1) {
        const uint32_t idDP = idesc_bf16(64, 64, 0, 0);
        uint32_t cnt = 0, it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
            const uint32_t ab = it & 1, acc = tdP + 64 * ab;
            if (it >= 2) mbar_wait(&acc_empty[ab], ((it >> 1) - 1) & 1);
            tc_fence_after();
            for (int kb = 0; kb < NKB; ++kb, ++cnt) {
                const uint32_t s2 = cnt % DP_NSTG, use = cnt / DP_NSTG;
                mbar_wait(&full[s2], use & 1);
                tc_fence_after();
                const uint32_t aD = smem_u32(sm + s2 * 16384), aV = aD + 8192;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    mma_bf16_w(acc, sdesc_sw128(aD + kk * 32, 16, 1024), sdesc_sw128(aV + kk * 32, 16, 1024), idDP,
                               (kb | kk) > 0);
                mma_commit_w(&empty[s2]);
            }
            mma_commit_w(&acc_full[ab]);
            __syncwarp();
        }
    } else {
        const int lq = warp & 3, et = tid - 64;
        const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
        uint32_t it = 0;
        for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++it) {
            const int row = (int)((size_t)(item / NC) * T + (size_t)(item % NC) * CH);
            const uint32_t ab = it & 1;
            mbar_wait(&acc_full[ab], (it >> 1) & 1);
            tc_fence_after();
            if (et == 0) tma_store_wait_read();    // the previous item's dP store has read the staging tile
            named_bar_sync(1, 128);
            m64_epilogue(tdP + 64 * ab, lane_base, lq, lane, sdP);
            tc_fence_before();
            fence_async_smem();
            named_bar_sync(1, 128);
            if (et == 0) {
                mbar_arrive(&acc_empty[ab]);
                tma_store_2d(&tmDP, sdP, 0, row);
                tma_store_commit();
            }
        }
        if (et == 0) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, 128);
}


// k_bwd_dq3: the dq walk pipelined over 128-channel halves with double-buffered inputs.
//   warps 0-7   state pass, one channel half at a time (SB half -> smem, Y half decayed), each half signalled;
//   warp 8      state MMA per half (Y[:, half] += V^T K~[:, half], N = 128), commits bar_sh[half];
//   warps 9, 10 dq^T of one half each (SB^T[half] dO^T + K~^T[half] dP^T) into a double-buffered TMEM
//               accumulator, commits bar_dq[buffer][half];
//   warps 11-14 epilogue: the dq partial; the input loads two chunks ahead (double buffers, bar_free).
// The next chunk's half-h pass waits only for the half-h MMAs, so half 0's MMAs overlap half 1's pass.
// Barriers that one role waits on while another may run ahead are per buffer, so no wait can alias a later
// phase of the same barrier.
template <int K>
struct Dq3Cfg {
    static constexpr int KB = K / 64, NH = K / 128;
    static constexpr uint32_t OP = KB * 8192;                  // [KB][64 t][128 B]  K~hi
    static constexpr uint32_t OFF_K = 0;                       // 2 buffers
    static constexpr uint32_t OFF_SB = 2 * OP;                 // [KB][128 v][128 B]
    static constexpr uint32_t OFF_V = OFF_SB + KB * 16384;     // 2 buffers x [2][64 t][128 B]
    static constexpr uint32_t OFF_D = OFF_V + 2 * 16384;       // 2 buffers x [2][64 t][128 B]
    static constexpr uint32_t OFF_DP = OFF_D + 2 * 16384;      // 2 buffers x [64 t][128 B]
    static constexpr uint32_t OFF_F = OFF_DP + 2 * 8192;       // fsb, fy, pend, red[4][K]
    static constexpr uint32_t SMEM = OFF_F + 4 * 7 * K + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
    static constexpr int NST = 256, NTHR = NST + 3 * 32 + 128;
    static constexpr uint32_t DQB = 64 * NH, COL_DQ = K;
    static constexpr uint32_t TCOLS = K + 2 * DQB > 256 ? 512 : 256;
};

template <int K>
__global__ void __launch_bounds__(Dq3Cfg<K>::NTHR, 1)
k_bwd_dq3(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmDP,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmD,
          const float* __restrict__ stats, const float* __restrict__ h0, const float* __restrict__ dfinal,
          __nv_bfloat16* __restrict__ dqp, float* __restrict__ stdot, __nv_bfloat16* __restrict__ anch,
          const int* __restrict__ flag, int T, int V) {
    using DC = Dq3Cfg<K>;
    if (*flag) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sK = sm + DC::OFF_K;
    uint8_t* sSB = sm + DC::OFF_SB;
    uint8_t* sV = sm + DC::OFF_V;
    uint8_t* sD = sm + DC::OFF_D;
    uint8_t* sdP = sm + DC::OFF_DP;
    float* fsb = reinterpret_cast<float*>(sm + DC::OFF_F);
    float* fy = fsb + K;
    float* pend = fy + K;
    float* red = pend + K;
    __shared__ uint64_t bar_in[2], bar_free[2], bar_sbh[2], bar_sh[2], bar_dq[2][2], bar_efree[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vt = blockIdx.x, bh = blockIdx.y, v0 = vt * VT, NC = T / CH;
    const int rowb = bh * T;
    const bool intra = vt == 0;
    const uint32_t in_bytes = DC::OP + 32768 + (intra ? 8192 : 0);
    auto load_inputs = [&](int i) {
        const int row = rowb + i * CH, b = i & 1;
        mbar_expect_tx(&bar_in[b], in_bytes);
        for (int c = 0; c < K / 64; ++c) tma_load_2d(sK + b * DC::OP + c * 8192, &tmK, &bar_in[b], 64 * c, row);
        tma_load_2d(sV + b * 16384, &tmV, &bar_in[b], v0, row);
        tma_load_2d(sV + b * 16384 + 8192, &tmV, &bar_in[b], v0 + 64, row);
        tma_load_2d(sD + b * 16384, &tmD, &bar_in[b], v0, row);
        tma_load_2d(sD + b * 16384 + 8192, &tmD, &bar_in[b], v0 + 64, row);
        if (intra) tma_load_2d(sdP + b * 8192, &tmDP, &bar_in[b], 0, row);
    };
    if (warp == 0) tmem_alloc(&tmem_base, DC::TCOLS);
    if (tid == 0) {
        for (int j = 0; j < 2; ++j) {
            mbar_init(&bar_in[j], 1);
            mbar_init(&bar_free[j], 1 + DC::NH);
            mbar_init(&bar_sbh[j], 1);
            mbar_init(&bar_sh[j], 1);
            mbar_init(&bar_dq[j][0], 1);
            mbar_init(&bar_dq[j][1], 1);
            mbar_init(&bar_efree[j], 1);
        }
        fence_mbar_init();
        load_inputs(0);
        if (NC > 1) load_inputs(1);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tS = tmem_base, tdq = tmem_base + DC::COL_DQ;
    const int lq = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int vrow = 32 * lq + lane;

    if (warp < 8) {
        // ------------------------------------------------------------------ state warps
        const int sub = warp >> 2;             // 64-channel share of each 128-channel half
        for (int m = tid; m < K; m += DC::NST) pend[m] = 0.f;
        for (int c0 = 0; c0 < K; c0 += 32) {
            if (((c0 >> 6) & 1) != sub) continue;   // channels [128 h + 64 sub, +64)
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(h0 ? h0[((size_t)bh * K + c0 + j) * V + v0 + vrow] : 0.f);
            tmem_st32(tS + lane_base + c0, r);
        }
        tmem_wait_st();
        float st_r = 0.f, st_G = 0.f;          // per-chunk statistics, one chunk ahead
        if (tid < K) {
            st_r = stats[((size_t)bh * NC) * 2 * K + tid];
            st_G = stats[((size_t)bh * NC) * 2 * K + K + tid];
        }
        named_bar_sync(1, DC::NST);
        for (int i = 0; i < NC; ++i) {
            if (tid < K) {   // SB = bf16(H_i e^{r}); Y <- H_i e^{r}; next pending = Gamma - r
                const float r_ = st_r, G_ = st_G;
                if (i + 1 < NC) {
                    st_r = stats[((size_t)bh * NC + i + 1) * 2 * K + tid];
                    st_G = stats[((size_t)bh * NC + i + 1) * 2 * K + K + tid];
                }
                fsb[tid] = ex2f((pend[tid] + r_) * L2E);
                fy[tid] = fsb[tid];
                pend[tid] = G_ - r_;
            }
            named_bar_sync(1, DC::NST);        // fsb / fy visible
            __nv_bfloat16* arow = (anch && i > 0 && i % ANCH == 0)   // (NULL: the forward saved them)
                ? anch + (((size_t)(i / ANCH - 1) * gridDim.y + bh) * V + v0 + vrow) * K : nullptr;
#pragma unroll 1
            for (int hh = 0; hh < DC::NH; ++hh) {
                if (i > 0) {                   // half hh of chunk i-1: Y final, SB half free
                    mbar_wait(&bar_sh[hh], (i - 1) & 1);
                    mbar_wait(&bar_dq[(i - 1) & 1][hh], ((i - 1) >> 1) & 1);
                    tc_fence_after();
                }
                const int c0 = 128 * hh + 64 * sub;
                state_pass_cols<1>(tS, lane_base, c0, vrow, fsb, fy, sSB, arow);
                state_pass_cols<1>(tS, lane_base, c0 + 32, vrow, fsb, fy, sSB, arow);
                tmem_wait_st();
                fence_async_smem();
                tc_fence_before();
                named_bar_sync(1, DC::NST);
                if (tid == 0) mbar_arrive(&bar_sbh[hh]);
            }
        }
        for (int hh = 0; hh < DC::NH; ++hh) mbar_wait(&bar_sh[hh], (NC - 1) & 1);
        tc_fence_after();
        if (dfinal) {   // S_T . dS_T partial over this V tile
            for (int c0 = 0; c0 < K; c0 += 32) {
                if (((c0 >> 6) & 1) != sub) continue;
                uint32_t r[32];
                tmem_ld32(tS + lane_base + c0, r);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    float x = __uint_as_float(r[j]) * ex2f(pend[c0 + j] * L2E) * dfinal[((size_t)bh * K + c0 + j) * V + v0 + vrow];
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
                    if (lane == 0) red[lq * K + c0 + j] = x;
                }
            }
            named_bar_sync(1, DC::NST);
            for (int m = tid; m < K; m += DC::NST)
                stdot[((size_t)vt * gridDim.y + bh) * K + m] = red[m] + red[K + m] + red[2 * K + m] + red[3 * K + m];
        }
    } else if (warp == 8) {
        // ------------------------------------------------------------------ state MMA issuer (per half)
        const uint32_t idS = idesc_bf16(128, 128, 1, 1);
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            const uint32_t aK = smem_u32(sK + b * DC::OP), aV = smem_u32(sV + b * 16384);
            for (int hh = 0; hh < DC::NH; ++hh) {
                mbar_wait(&bar_sbh[hh], i & 1);
                if (hh == 0) mbar_wait(&bar_in[b], (i >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk)
                    mma_bf16_w(tS + 128 * hh, sdesc_sw128(aV + kk * 2048, 8192, 1024),
                               sdesc_sw128(aK + 2 * hh * 8192 + kk * 2048, 8192, 1024), idS, 1);
                mma_commit_w(&bar_sh[hh]);
            }
            mma_commit_w(&bar_free[b]);
            __syncwarp();
        }
    } else if (warp < 11) {
        // ------------------------------------------------------------------ dq^T issuers (one per half)
        const int hh = warp - 9;
        const uint32_t idDQ = idesc_bf16(128, 64, 1, 0);
        const uint32_t aSB = smem_u32(sSB);
        if (hh < DC::NH) {
            for (int i = 0; i < NC; ++i) {
                const int b = i & 1;
                const uint32_t aK = smem_u32(sK + b * DC::OP), aD = smem_u32(sD + b * 16384),
                               adP = smem_u32(sdP + b * 8192);
                mbar_wait(&bar_sbh[hh], i & 1);
                mbar_wait(&bar_in[b], (i >> 1) & 1);
                if (i >= 2) mbar_wait(&bar_efree[b], ((i >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t td = tdq + DC::DQB * b + 64 * hh;
#pragma unroll
                for (int kk = 0; kk < VT / 16; ++kk) {   // dq^T[ch][t] = SB^T dO^T (this V tile)
                    const uint32_t ob = (kk >> 2) * 8192 + (kk & 3) * 32;
                    mma_bf16_w(td, sdesc_sw128(aSB + 2 * hh * 16384 + kk * 2048, 16384, 1024),
                               sdesc_sw128(aD + ob, 16, 1024), idDQ, kk > 0);
                }
                if (intra)
#pragma unroll
                    for (int kk = 0; kk < CH / 16; ++kk)   // + K~^T dP^T (the full intra term, V tile 0 only)
                        mma_bf16_w(td, sdesc_sw128(aK + 2 * hh * 8192 + kk * 2048, 8192, 1024),
                                   sdesc_sw128(adP + kk * 32, 16, 1024), idDQ, 1);
                mma_commit_w(&bar_dq[b][hh]);
                mma_commit_w(&bar_free[b]);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue warps
        const int et = tid - DC::NST - 96;
        __nv_bfloat16* out = dqp + (size_t)vt * gridDim.y * T * K;
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            if (et == 0 && i + 2 < NC) {       // inputs of chunk i+2 into buffer b once chunk i's MMAs are done
                mbar_wait(&bar_free[b], (i >> 1) & 1);
                load_inputs(i + 2);
            }
            for (int hh = 0; hh < DC::NH; ++hh) mbar_wait(&bar_dq[b][hh], (i >> 1) & 1);
            tc_fence_after();
            const size_t row0 = (size_t)rowb + (size_t)i * CH;
#pragma unroll
            for (int hh = 0; hh < DC::NH; ++hh)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t r[32];
                    tmem_ld32(tdq + DC::DQB * b + 64 * hh + 32 * h + lane_base, r);
                    tmem_wait_ld();
                    const int ch = 128 * hh + vrow;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        out[(row0 + 32 * h + j) * K + ch] = __float2bfloat16_rn(__uint_as_float(r[j]));
                }
            tc_fence_before();
            named_bar_sync(2, 128);
            if (et == 0) mbar_arrive(&bar_efree[b]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, DC::TCOLS);
}

// k_bwd_dkv3: the dkv walk pipelined over 128-channel halves ("sides" A = channels 0-127, B = 128-255).
//   warps 0-7   state pass per half: dSB half -> smem (MN-major A of dk^T), Z half decayed; anchor carries; dh0.
//   warp 8  (A) Z half 0 += dO^T Q~[:, A];  dv = dSB[:, A] K~[:, A]^T + dO^T P        (dv double-buffered)
//   warp 9  (A) dk^T half 0 = dSB^T[A] V^T (+ Q~^T[A] dP on V tile 0)
//   warp 10 (B) Z half 1 += dO^T Q~[:, B];  dv += dSB[:, B] K~[:, B]^T (after side A's dv, fixed order)
//   warp 11 (B) dk^T half 1
//   warps 12-15 epilogue: dk partials and dv (direct global stores), and every TMA input load: the side-A
//               tiles (K~, Q~ halves, P) of the next chunk as soon as side A's MMAs are done, side B's after side
//               B, the shared tiles (V, dO, dP; double-buffered) two chunks ahead.
// The next chunk's half-0 pass needs only side A's MMAs, so side A's MMAs overlap the half-1 pass and side B's
// MMAs overlap the next half-0 pass.  Barriers that can be waited on while the producer runs ahead are per buffer.
template <int K>
struct Dkv3Cfg {
    static constexpr int KB = K / 64, NH = K / 128, CPH = 128;
    static constexpr uint32_t OP = KB * 8192;                   // Q~hi or K~hi [KB][64 t][128 B]
    static constexpr uint32_t OFF_SB = 0;                       // [KB][128 v][128 B]
    static constexpr uint32_t OFF_Q = KB * 16384, OFF_K = OFF_Q + OP;
    static constexpr uint32_t OFF_V = OFF_K + OP;               // 2 buffers x [2][64 t][128 B]
    static constexpr uint32_t OFF_D = OFF_V + 2 * 16384;        // 2 buffers
    static constexpr uint32_t OFF_P = OFF_D + 2 * 16384;        // [64 t][128 B]
    static constexpr uint32_t OFF_DP = OFF_P + 8192;            // 2 buffers
    static constexpr uint32_t OFF_F = OFF_DP + 2 * 8192;        // fsb, fy, pend, red[4][K]
    static constexpr uint32_t SMEM = OFF_F + 4 * 7 * K + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
    static constexpr int NST = 256, NTHR = 512;
    static constexpr uint32_t COL_DK = K, COL_DV = K + 64 * NH, TCOLS = 512;   // Z | dk^T halves | dv x 2
    static_assert(COL_DV + 128 <= TCOLS, "TMEM columns");
};

template <int K, int EMIT>
__global__ void __launch_bounds__(Dkv3Cfg<K>::NTHR, 1)
k_bwd_dkv3(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmDP,
           const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmD,
           const float* __restrict__ stats, const float* __restrict__ dfinal, __nv_bfloat16* __restrict__ dv_out,
           __nv_bfloat16* __restrict__ dkp, float* __restrict__ dh0, const __nv_bfloat16* __restrict__ anch,
           float* __restrict__ cpart, const int* __restrict__ flag, int T, int V, const int* __restrict__ cflags) {
    constexpr int emit = EMIT;   // compile-time: the unused roles' code is removed
    // cflags (emit == 2 only, else NULL): the forward's per-chunk exact-path flags; a flagged chunk's pass takes the
    // r = 0 frame of its exact operands (Q~ = q e^{b}, K~ = k e^{Gamma - b}): dSB = bf16(dH_{i+1}) (factor
    // e^{pend}), Z <- dH_{i+1} e^{Gamma} before the update, pending 0 (see k_bwd_kwalk).
    // emit == 0: adjoint-only walk (segment summaries dh_loc): only the Z updates run and only dh0 is written.
    // emit == 2: dv, the anchor carries and dh0 but no dk (dk comes from the K-tiled dk walk, tc_kwalk.cu).
    // (Keeping dSB in TMEM, in the then free dk^T columns, as the A operand of TS-mode dv MMAs measured slower:
    // 188 vs 177 us at 1.3B -- the operand reads compete with the state pass for TMEM bandwidth.)
    using DC = Dkv3Cfg<K>;
    constexpr int NH = DC::NH;
    if (*flag) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sSB = sm + DC::OFF_SB;
    uint8_t* sQ = sm + DC::OFF_Q;
    uint8_t* sK = sm + DC::OFF_K;
    uint8_t* sV = sm + DC::OFF_V;
    uint8_t* sD = sm + DC::OFF_D;
    uint8_t* sP = sm + DC::OFF_P;
    uint8_t* sdP = sm + DC::OFF_DP;
    float* fsb = reinterpret_cast<float*>(sm + DC::OFF_F);
    float* fy = fsb + K;
    float* pend = fy + K;
    float* red = pend + K;
    __shared__ uint64_t bar_inA, bar_inB, bar_inS[2], bar_sbh[2], bar_mA, bar_mB, bar_dva[2], bar_efdk[2],
        bar_efdv[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vt = blockIdx.x, bh = blockIdx.y, v0 = vt * VT, NC = T / CH;
    const int rowb = bh * T;
    const bool intra = vt == 0;
    // side-A tiles: K~ / Q~ channel blocks [0, 2 per side) (all blocks when NH = 1) and P; side B: blocks 2, 3
    auto loadA = [&](int i) {
        const int row = rowb + i * CH, nb = NH == 2 ? 2 : DC::KB;
        mbar_expect_tx(&bar_inA, 2 * nb * 8192 + 8192);
        for (int c = 0; c < nb; ++c) {
            tma_load_2d(sQ + c * 8192, &tmQ, &bar_inA, 64 * c, row);
            tma_load_2d(sK + c * 8192, &tmK, &bar_inA, 64 * c, row);
        }
        tma_load_2d(sP, &tmP, &bar_inA, 0, row);
    };
    auto loadB = [&](int i) {
        const int row = rowb + i * CH;
        mbar_expect_tx(&bar_inB, 4 * 8192);
        for (int c = 2; c < 4; ++c) {
            tma_load_2d(sQ + c * 8192, &tmQ, &bar_inB, 64 * c, row);
            tma_load_2d(sK + c * 8192, &tmK, &bar_inB, 64 * c, row);
        }
    };
    auto loadS = [&](int i) {                  // buffer = step parity (step = NC-1-i)
        const int row = rowb + i * CH, b = (NC - 1 - i) & 1;
        const bool dk = emit == 1;             // V and dP feed only the dk MMAs
        mbar_expect_tx(&bar_inS[b], 16384 + (dk ? 16384 + (intra ? 8192 : 0) : 0));
        if (dk) {
            tma_load_2d(sV + b * 16384, &tmV, &bar_inS[b], v0, row);
            tma_load_2d(sV + b * 16384 + 8192, &tmV, &bar_inS[b], v0 + 64, row);
        }
        tma_load_2d(sD + b * 16384, &tmD, &bar_inS[b], v0, row);
        tma_load_2d(sD + b * 16384 + 8192, &tmD, &bar_inS[b], v0 + 64, row);
        if (dk && intra) tma_load_2d(sdP + b * 8192, &tmDP, &bar_inS[b], 0, row);
    };
    if (warp == 0) tmem_alloc(&tmem_base, DC::TCOLS);
    if (tid == 0) {
        mbar_init(&bar_inA, 1); mbar_init(&bar_inB, 1);
        mbar_init(&bar_mA, 2); mbar_init(&bar_mB, 2);
        for (int j = 0; j < 2; ++j) {
            mbar_init(&bar_inS[j], 1); mbar_init(&bar_sbh[j], 1); mbar_init(&bar_dva[j], 1);
            mbar_init(&bar_efdk[j], 1); mbar_init(&bar_efdv[j], 1);
        }
        fence_mbar_init();
        loadA(NC - 1);
        if (NH == 2) loadB(NC - 1);
        loadS(NC - 1);
        if (NC > 1) loadS(NC - 2);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tZ = tmem_base, tdk = tmem_base + DC::COL_DK, tdv = tmem_base + DC::COL_DV;
    const int lq = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int vrow = 32 * lq + lane;

    if (warp < 8) {
        // ------------------------------------------------------------------ state warps
        const int sub = warp >> 2;             // 64-channel share of each half
        for (int m = tid; m < K; m += DC::NST) pend[m] = 0.f;
        for (int c0 = 0; c0 < K; c0 += 32) {
            if (((c0 >> 6) & 1) != sub) continue;
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 32; ++j)
                r[j] = __float_as_uint(dfinal ? dfinal[((size_t)bh * K + c0 + j) * V + v0 + vrow] : 0.f);
            tmem_st32(tZ + lane_base + c0, r);
        }
        tmem_wait_st();
        float st_r = 0.f, st_G = 0.f;          // per-chunk statistics, one chunk ahead
        int st_slow = 0;
        if (tid < K) {
            st_r = stats[((size_t)bh * NC + NC - 1) * 2 * K + tid];
            st_G = stats[((size_t)bh * NC + NC - 1) * 2 * K + K + tid];
            st_slow = cflags ? cflags[(size_t)bh * NC + NC - 1] : 0;
        }
        named_bar_sync(1, DC::NST);
        for (int i = NC - 1; i >= 0; --i) {
            const int j = NC - 1 - i;
            // The next step's anchor carry (boundary i, if it is one) reads this CTA's 128 rows of the anchor state
            // (one contiguous 64 KB block): prefetch them into L2 a chunk ahead, so the pass does not wait on HBM.
            if (GLA_ANCH_PF && tid == 0 && anch && i > 0 && i % ANCH == 0) {
                const uint8_t* a0 = reinterpret_cast<const uint8_t*>(
                    anch + (((size_t)(i / ANCH - 1) * gridDim.y + bh) * V + v0) * K);
                for (uint32_t o = 0; o < (uint32_t)VT * K * 2; o += 16384) prefetch_l2_bulk(a0 + o, 16384);
            }
            if (tid < K) {   // dSB = bf16(dH_{i+1} e^{Gamma - r}); Z <- same; next pending = r
                const float r_ = st_r, G_ = st_G;
                const bool slow = st_slow != 0;
                if (i > 0) {
                    st_r = stats[((size_t)bh * NC + i - 1) * 2 * K + tid];
                    st_G = stats[((size_t)bh * NC + i - 1) * 2 * K + K + tid];
                    st_slow = cflags ? cflags[(size_t)bh * NC + i - 1] : 0;
                }
                if (!slow) {
                    fsb[tid] = ex2f((pend[tid] + G_ - r_) * L2E);
                    fy[tid] = fsb[tid];
                    pend[tid] = r_;
                } else {     // exact-path chunk: dSB = bf16(dH_{i+1}), Z <- dH_{i+1} e^{Gamma}, pending 0
                    fsb[tid] = ex2f(pend[tid] * L2E);
                    fy[tid] = ex2f((pend[tid] + G_) * L2E);
                    pend[tid] = 0.f;
                }
            }
            named_bar_sync(1, DC::NST);        // fsb / fy visible
            const int bd = i + 1;              // exact d log alpha carry at boundary bd over this V tile
            const bool anc = j > 0 && anch != nullptr && bd % ANCH == 0;
#pragma unroll 1
            for (int hh = 0; hh < NH; ++hh) {
                if (j > 0) {                   // side hh's MMAs of chunk i+1 done: Z half final, dSB half free
                    mbar_wait(hh == 0 ? &bar_mA : &bar_mB, (j - 1) & 1);
                    tc_fence_after();
                }
                if (anc) {
                    const __nv_bfloat16* arow =
                        anch + (((size_t)(bd / ANCH - 1) * gridDim.y + bh) * V + v0 + vrow) * K;
#pragma unroll 1
                    for (int sl = 0; sl < 2; ++sl) {
                        const int c0 = 128 * hh + 64 * sub + 32 * sl;
                        uint32_t r[32];
                        tmem_ld32(tZ + lane_base + c0, r);
                        uint4 hv[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) hv[u] = __ldg(reinterpret_cast<const uint4*>(arow + c0 + 8 * u));
                        tmem_wait_ld();
                        float x[32];
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj) {
                            const uint32_t w = word(hv[jj >> 3], (jj & 7) >> 1);
                            x[jj] = ((jj & 1) ? bf16hi(w) : bf16lo(w)) * __uint_as_float(r[jj]);
                        }
#pragma unroll
                        for (int o = 16; o >= 1; o >>= 1) {
                            const bool up = (lane & o) != 0;
#pragma unroll
                            for (int jj = 0; jj < o; ++jj) {
                                const float send = up ? x[jj] : x[jj + o];
                                const float keep = up ? x[jj + o] : x[jj];
                                x[jj] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                            }
                        }
                        red[lq * K + c0 + lane] = x[0];
                    }
                }
                const int c0 = 128 * hh + 64 * sub;
                state_pass_cols<1>(tZ, lane_base, c0, vrow, fsb, fy, sSB, nullptr);
                state_pass_cols<1>(tZ, lane_base, c0 + 32, vrow, fsb, fy, sSB, nullptr);
                tmem_wait_st();
                fence_async_smem();
                tc_fence_before();
                named_bar_sync(1, DC::NST);
                if (tid == 0) mbar_arrive(&bar_sbh[hh]);
            }
            if (anc) {                         // red complete (the last half's barrier)
                for (int m = tid; m < K; m += DC::NST)
                    cpart[(((size_t)(bd / ANCH - 1) * gridDim.x + vt) * gridDim.y + bh) * K + m] =
                        red[m] + red[K + m] + red[2 * K + m] + red[3 * K + m];
                named_bar_sync(1, DC::NST);    // red may be reused
            }
        }
        mbar_wait(&bar_mA, (NC - 1) & 1);
        if (NH == 2) mbar_wait(&bar_mB, (NC - 1) & 1);
        tc_fence_after();
        if (dh0) {
            for (int c0 = 0; c0 < K; c0 += 32) {
                if (((c0 >> 6) & 1) != sub) continue;
                uint32_t r[32];
                tmem_ld32(tZ + lane_base + c0, r);
                tmem_wait_ld();
#pragma unroll
                for (int jj = 0; jj < 32; ++jj)
                    dh0[((size_t)bh * K + c0 + jj) * V + v0 + vrow] = __uint_as_float(r[jj]) * ex2f(pend[c0 + jj] * L2E);
            }
        }
    } else if (warp < 12) {
        // ------------------------------------------------------------------ MMA issuers
        const int role = warp - 8;             // 0: Z_A + dv_A, 1: dk_A, 2: Z_B + dv_B, 3: dk_B
        const int hh = role >> 1;
        const uint32_t idZ = idesc_bf16(128, NH == 2 ? 128 : K, 1, 1);   // Z[v][ch] += dO^T Q~ (one half)
        const uint32_t idV1 = idesc_bf16(128, 64, 0, 0);    // dv^T = dSB K~^T
        const uint32_t idV2 = idesc_bf16(128, 64, 1, 1);    // dv^T += dO^T P
        const uint32_t idK1 = idesc_bf16(128, 64, 1, 0);    // dk^T = dSB^T V^T
        const uint32_t idK2 = idesc_bf16(128, 64, 1, 1);    // dk^T += Q~^T dP
        const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aSB = smem_u32(sSB), aP = smem_u32(sP);
        if (hh < NH) {
            for (int i = NC - 1; i >= 0; --i) {
                const int j = NC - 1 - i, bs = j & 1;
                const uint32_t aV = smem_u32(sV + bs * 16384), aD = smem_u32(sD + bs * 16384),
                               adP = smem_u32(sdP + bs * 8192);
                mbar_wait(&bar_sbh[hh], j & 1);
                mbar_wait(hh == 0 ? &bar_inA : &bar_inB, j & 1);
                mbar_wait(&bar_inS[bs], (j >> 1) & 1);
                if ((role & 1) == 0) {         // Z half (+ dv part)
                    if (hh == 0 && emit && j >= 2) mbar_wait(&bar_efdv[bs], ((j >> 1) - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < CH / 16; ++kk)
                        mma_bf16_w(tZ + 128 * hh, sdesc_sw128(aD + kk * 2048, 8192, 1024),
                                   sdesc_sw128(aQ + 2 * hh * 8192 + kk * 2048, 8192, 1024), idZ, 1);
                    if (emit) {
                        if (hh == 1) {         // side A's dv MMAs of this buffer first (fixed accumulation order)
                            mbar_wait(&bar_dva[bs], (j >> 1) & 1);
                            tc_fence_after();
                        }
                        const int k0 = hh * (DC::CPH / 16), k1 = NH == 2 ? k0 + DC::CPH / 16 : K / 16;
                        for (int kk = k0; kk < k1; ++kk) {
                            const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32, ob = (kk >> 2) * 8192 + (kk & 3) * 32;
                            mma_bf16_w(tdv + 64 * bs, sdesc_sw128(aSB + o, 16, 1024), sdesc_sw128(aK + ob, 16, 1024),
                                       idV1, kk > 0);
                        }
                        if (hh == 0)
#pragma unroll
                            for (int kk = 0; kk < CH / 16; ++kk)
                                mma_bf16_w(tdv + 64 * bs, sdesc_sw128(aD + kk * 2048, 8192, 1024),
                                           sdesc_sw128(aP + kk * 2048, 8192, 1024), idV2, 1);
                    }
                    if (hh == 0) mma_commit_w(&bar_dva[bs]);
                } else if (emit == 1) {        // dk^T half
                    if (j >= 1) mbar_wait(&bar_efdk[hh], (j - 1) & 1);
                    tc_fence_after();
#pragma unroll
                    for (int kk = 0; kk < VT / 16; ++kk) {
                        const uint32_t ob = (kk >> 2) * 8192 + (kk & 3) * 32;
                        mma_bf16_w(tdk + 64 * hh, sdesc_sw128(aSB + 2 * hh * 16384 + kk * 2048, 16384, 1024),
                                   sdesc_sw128(aV + ob, 16, 1024), idK1, kk > 0);
                    }
                    if (intra)
#pragma unroll
                        for (int kk = 0; kk < CH / 16; ++kk)
                            mma_bf16_w(tdk + 64 * hh, sdesc_sw128(aQ + 2 * hh * 8192 + kk * 2048, 8192, 1024),
                                       sdesc_sw128(adP + kk * 2048, 8192, 1024), idK2, 1);
                } else {
                    tc_fence_after();
                }
                mma_commit_w(hh == 0 ? &bar_mA : &bar_mB);
                __syncwarp();
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue warps
        const int et = tid - DC::NST - 128;
        __nv_bfloat16* dko = dkp + (size_t)vt * gridDim.y * T * K;
        for (int i = NC - 1; i >= 0; --i) {
            const int j = NC - 1 - i, bs = j & 1;
            const size_t row0 = (size_t)rowb + (size_t)i * CH;
            for (int hh = 0; hh < NH; ++hh) {
                mbar_wait(hh == 0 ? &bar_mA : &bar_mB, j & 1);
                tc_fence_after();
                if (et == 0 && i > 0) { if (hh == 0) loadA(i - 1); else loadB(i - 1); }
                if (emit == 1) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        uint32_t r[32];
                        tmem_ld32(tdk + 64 * hh + 32 * h + lane_base, r);
                        tmem_wait_ld();
                        const int ch = 128 * hh + vrow;
#pragma unroll
                        for (int jj = 0; jj < 32; ++jj)
                            dko[(row0 + 32 * h + jj) * K + ch] = __float2bfloat16_rn(__uint_as_float(r[jj]));
                    }
                }
                tc_fence_before();
                named_bar_sync(2, 128);
                if (et == 0) mbar_arrive(&bar_efdk[hh]);
            }
            if (et == 0 && i >= 2) loadS(i - 2);   // both sides done: shared buffer bs free
            if (emit) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t r[32];
                    tmem_ld32(tdv + 64 * bs + 32 * h + lane_base, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int jj = 0; jj < 32; ++jj)
                        dv_out[(row0 + 32 * h + jj) * V + v0 + vrow] = __float2bfloat16_rn(__uint_as_float(r[jj]));
                }
            }
            tc_fence_before();
            named_bar_sync(2, 128);
            if (et == 0) mbar_arrive(&bar_efdv[bs]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, DC::TCOLS);
}

// ---------------------------------------------------------------------------------------------------------------
bool bwd_tc_supported(int K, int V) {
    const int nvt = V / 128;
    return (K == 128 || K == 256) && V % 128 == 0 && (nvt == 1 || nvt == 2 || nvt == 4 || nvt == 8);
}

static size_t al1k(size_t x) { return (x + 1023) & ~size_t(1023); }
// extra scratch of the split backward: Q~hi, K~hi, P, dP (bf16) and per-chunk (r, Gamma) statistics
static size_t split_ws(int B, int H, int T, int K) {
    const size_t BH = (size_t)B * H, rows = BH * T, NC = T / CH;
    return 2 * al1k(rows * K * 2) + 2 * al1k(rows * 64 * 2) + al1k(BH * NC * 2 * K * 4);
}

size_t bwd_tc_ws(int B, int H, int T, int K, int V, int C) {
    const size_t BH = (size_t)B * H, NVT = V / VT;
    size_t bytes = 256 + split_ws(B, H, T, K);                  // flag + split-backward scratch
    bytes += 2 * NVT * BH * T * K * sizeof(__nv_bfloat16);       // dq, dk partials
    const int Smax = fwd_segments((int)BH, V, T / CH);
    bytes += NVT * BH * Smax * K * sizeof(float);                // S_T . dS_T partials (per segment)
    bytes = (bytes + 255) & ~size_t(255);
    const size_t NA = (T / C > 1) ? (size_t)(T / C - 1) / ANCH : 0;
    bytes += NA * BH * V * K * sizeof(__nv_bfloat16);           // state anchors (bf16)
    bytes += NA * NVT * BH * K * sizeof(float);                 // anchor row-sum partials
    bytes = (bytes + 255) & ~size_t(255);
    if (Smax > 1)   // per-segment d_final states; d_initial states (the split summaries' partials before the chain)
        bytes += (1 + seg_parts((int)BH, K, V, T / CH, Smax)) * BH * Smax * K * V * sizeof(float) +
                 BH * Smax * K * sizeof(float);   // per-segment log decays
    return bytes + simt::bwd_ws(B, H, T, K, V, C);              // exact-path fallback scratch
}


// Split backward: prep + TMA-fed walks + reduce (+ exact CUDA-core fallback behind the guard flag).
// dst[bh] = src[bh * S + 0] for [K, V] fp32 states (segment 0's d_initial_state), unless the exact fallback
// (which writes dst itself) is running.
__global__ void k_copy_seg0(float* __restrict__ dst, const float* __restrict__ src, int BH, int S, size_t KV,
                            const int* __restrict__ flag) {
    if (*flag) return;
    const size_t n4 = (size_t)BH * KV / 4;
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const size_t e = 4 * i, bh = e / KV, off = e % KV;
    *reinterpret_cast<float4*>(dst + e) = *reinterpret_cast<const float4*>(src + bh * S * KV + off);
}

// Side stream for running the two backward walks concurrently: one non-blocking stream per (device, caller
// stream), created on first use, so callers on different streams never fence into each other's walks (and a
// stream being captured into a CUDA graph forks only onto its own side stream).  Fork/join events are
// per thread.  Returns nullptr if creation fails (the caller then stays on one stream).
static cudaStream_t side_stream(cudaStream_t caller, int idx = 0) {
    static std::map<std::pair<int, std::pair<cudaStream_t, int>>, cudaStream_t> streams;
    static std::mutex mu;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(mu);
    const auto key = std::make_pair(dev, std::make_pair(caller, idx));
    auto it = streams.find(key);
    if (it != streams.end()) return it->second;
    cudaStream_t s = nullptr;
    if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    streams[key] = s;
    return s;
}
static cudaEvent_t fork_event(int which) {
    thread_local cudaEvent_t evs[64][4] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    if (!evs[dev][which] && cudaEventCreateWithFlags(&evs[dev][which], cudaEventDisableTiming) != cudaSuccess)
        return nullptr;
    return evs[dev][which];
}

template <int K, typename TG>
static cudaError_t launch_bwd2(const BwdProblem& p, cudaStream_t st) {
    const int BH = p.B * p.H, NVT = p.V / VT, NC = p.T / CH;
    const size_t rows = (size_t)BH * p.T;
    uint8_t* w = (uint8_t*)p.ws;
    __nv_bfloat16* Qt = (__nv_bfloat16*)w; w += al1k(rows * K * 2);
    __nv_bfloat16* Kt = (__nv_bfloat16*)w; w += al1k(rows * K * 2);
    __nv_bfloat16* Pm = (__nv_bfloat16*)w; w += al1k(rows * 64 * 2);
    __nv_bfloat16* dPm = (__nv_bfloat16*)w; w += al1k(rows * 64 * 2);
    float* stats = (float*)w; w += al1k((size_t)BH * NC * 2 * K * 4);
    const bool saved = p.fwd_ws != nullptr && fwd_is_split();
    const int* fflags = nullptr;
    const __nv_bfloat16* saved_anch = nullptr;
    const float* h0v = nullptr;
    int S = 1;   // intra-GPU segments (the forward's choice; only with its saved segment-entry states)
    if (saved) {   // the forward's Q~hi, K~hi, P, (r, Gamma) and anchor states: only dP is left to form
        const FwdSaved f = fwd2_saved(p.fwd_ws, p.B, p.H, p.T, K, p.V);
        Qt = (__nv_bfloat16*)f.Qt; Kt = (__nv_bfloat16*)f.Kt; Pm = (__nv_bfloat16*)f.Pm;
        stats = (float*)f.stats; fflags = f.flags;
        if (saved_anchors()) saved_anch = (const __nv_bfloat16*)f.anch;
        if (f.S > 1) { S = f.S; h0v = f.h0v; }
    }
    const int BHv = BH * S, Tv = p.T / S;   // virtual units (segments) of the walks and the reduce
    uint8_t* ws = w;
    int* flag = (int*)ws;
    __nv_bfloat16* dqp = (__nv_bfloat16*)(ws + 256);
    __nv_bfloat16* dkp = dqp + (size_t)NVT * BH * p.T * K;
    float* stdot = (float*)(dkp + (size_t)NVT * BH * p.T * K);
    const int Smax = fwd_segments(BH, p.V, NC);
    size_t used = 256 + 2 * (size_t)NVT * BH * p.T * K * 2 + (size_t)NVT * BH * Smax * K * 4;
    used = (used + 255) & ~size_t(255);
    const size_t NA = (NC > 1) ? (size_t)(NC - 1) / ANCH : 0;
    __nv_bfloat16* anch = (__nv_bfloat16*)(ws + used);
    float* cpart = (float*)(ws + used + NA * BH * p.V * K * 2);
    used += NA * BH * p.V * K * 2 + NA * NVT * BH * K * 4;
    used = (used + 255) & ~size_t(255);
    float* dFv = (float*)(ws + used);                       // per-segment d_final_state (S > 1)
    float* dhv = dFv + (Smax > 1 ? (size_t)BH * Smax * K * p.V : 0);   // per-segment dh0 / dh_loc (partials)
    const int SP = (Smax > 1 && seg_summary_ok(K, p.V)) ? seg_parts(BH, K, p.V, NC, Smax) : 1;
    if (Smax > 1) used += (size_t)(1 + seg_parts(BH, K, p.V, NC, Smax)) * BH * Smax * K * p.V * 4;
    float* dec = (Smax > 1 && seg_summary_ok(K, p.V)) ? (float*)(ws + used) : nullptr;   // per-segment log decays
    if (Smax > 1) used += (size_t)BH * Smax * K * 4;
    cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    CUtensorMap mQ, mK, mP, mDP, mV, mD;
    if ((e = make_map_2d(&mQ, Qt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mK, Kt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mP, Pm, rows, 64, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mDP, dPm, rows, 64, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mV, p.v, rows, p.V, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mD, p.dO, rows, p.V, true)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_bwd_prep<K, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)BPrepCfg<K>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_bwd_dq3<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Dq3Cfg<K>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_bwd_dkv3<K, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Dkv3Cfg<K>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_bwd_dkv3<K, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Dkv3Cfg<K>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_bwd_dkv3<K, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Dkv3Cfg<K>::SMEM)))
        return e;
    // With the forward's anchors the walks are the K-tiled ones (tc_kwalk.cu): dq and dk leave them complete (no
    // V-tile partials), and they and the reduce follow the forward's exact path on flagged chunks.
    const bool kw = saved_anch && kwalk_ok(K, p.V);
    if (saved) {
        GLA_PROF("tc::bwd_dp", st);
        const int nitems = NC * BH;
        const int smem = DP_NSTG * 16384 + 8192 + 1024;
        if ((e = cudaFuncSetAttribute(k_bwd_dp, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess)
            return e;
        const int grid_dp = nitems < GLA_DP_GRID * num_sms() ? nitems : GLA_DP_GRID * num_sms();
        k_bwd_dp<<<(unsigned)grid_dp, 192, smem, st>>>(mDP, mV, mD, kw ? nullptr : fflags, flag, p.T, p.V, NC,
                                                        nitems);
    } else {
        GLA_PROF("tc::bwd_prep", st);
        const int nitems = NC * BH;
        k_bwd_prep<K, TG><<<(unsigned)(nitems < num_sms() ? nitems : num_sms()), NTH, BPrepCfg<K>::SMEM, st>>>(
            mQ, mK, mP, mDP, mV, mD, (const __nv_bfloat16*)p.q, (const __nv_bfloat16*)p.k, (const TG*)p.g, stats, flag,
            p.T, p.V, NC, nitems);
    }
    const dim3 grid(NVT, BHv);
    const float* dfin = p.dfinal;
    float* dh0w = p.dh0;
    if (S > 1) {
        // adjoint-only walks: every segment's d_initial_state with a zero d_final_state, then the reverse chain
        // gives every segment's true d_final_state (the segment-entry states h0v come from the forward)
        if (seg_summary_ok(K, p.V)) {   // one tensor-core contraction per segment (A = Q~hi e^{r + carry}, B = dO)
            GLA_PROF("tc::bwd_dstate_summary", st);
            if ((e = seg_summary(mD, mQ, stats, fflags, dhv, K, p.V, Tv, S, BHv, true, st, true, SP, dec)) != cudaSuccess)
                return e;
        } else {
            GLA_PROF("tc::bwd_dstate_summary", st);
            k_bwd_dkv3<K, 0><<<grid, Dkv3Cfg<K>::NTHR, Dkv3Cfg<K>::SMEM, st>>>(
                mQ, mK, mP, mDP, mV, mD, stats, nullptr, (__nv_bfloat16*)p.dv, dkp, dhv, nullptr, cpart, flag, Tv,
                p.V, nullptr);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        if ((e = seg_chain_bwd(stats, p.dfinal, dhv, dFv, BH, S, NC, K, p.V, st, SP,
                               seg_summary_ok(K, p.V) ? dec : nullptr)) != cudaSuccess) return e;
        dfin = dFv;
        dh0w = p.dh0 ? dhv : nullptr;
    }
    const float* h0w = S > 1 ? h0v : p.h0;
    // With the forward's anchors the two walks are independent: the dq walk runs on the library's side stream
    // concurrently with the dkv walk (each is 256 one-per-SM CTAs, 1.73 waves alone on 148 SMs).
    cudaStream_t sq = st;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    if (saved_anch && !prof::enabled()) {   // (the launch tracer times kernels one at a time)
        sq = side_stream(st);
        if (!sq || !(ev_in = fork_event(0)) || !(ev_out = fork_event(1))) sq = st;
    }
    if (sq != st) {
        if ((e = cudaEventRecord(ev_in, st)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(sq, ev_in, 0)) != cudaSuccess) return e;
    }
    float* dq32 = reinterpret_cast<float*>(dqp);   // (V/256) fp32 partials: the same bytes as NVT bf16 ones
    float* dk32 = reinterpret_cast<float*>(dkp);
    {
        GLA_PROF("tc::bwd_dq", sq);
        if (kw) {
            if ((e = dq_kwalk(K, p.V, mK, mDP, mV, mD, stats, h0w, dfin, dq32, dfin ? stdot : nullptr, flag, fflags,
                              Tv, BHv, sq)) != cudaSuccess)
                return e;
        } else {
            k_bwd_dq3<K><<<grid, Dq3Cfg<K>::NTHR, Dq3Cfg<K>::SMEM, sq>>>(mK, mDP, mV, mD, stats, h0w, dfin, dqp,
                                                                        dfin ? stdot : nullptr,
                                                                        saved_anch ? nullptr : anch, flag, Tv, p.V);
        }
    }
    if (kw) {
        GLA_PROF("tc::bwd_dk", st);
        if ((e = dk_kwalk(K, p.V, mQ, mDP, mD, mV, stats, dfin, dk32, flag, fflags, Tv, BHv, st)) != cudaSuccess)
            return e;
    }
    // K-tiled walks: the dv walk runs on a second side stream, concurrently with the dq and dk walks (three
    // independent 1-CTA-per-SM kernels of ~256 CTAs each fill the 148 SMs better together than one by one).
    cudaStream_t sv = st;
    cudaEvent_t ev_dv = nullptr;
    static const bool dv_side = !getenv("GLA_DV_MAIN");
    if (kw && sq != st && dv_side) {
        sv = side_stream(st, 1);
        if (!sv || !(ev_dv = fork_event(3))) sv = st;
        else if ((e = cudaStreamWaitEvent(sv, ev_in, 0)) != cudaSuccess) return e;
    }
    {
        GLA_PROF(kw ? "tc::bwd_dv" : "tc::bwd_dkv", sv);
        if (kw)
            k_bwd_dkv3<K, 2><<<grid, Dkv3Cfg<K>::NTHR, Dkv3Cfg<K>::SMEM, sv>>>(
                mQ, mK, mP, mDP, mV, mD, stats, dfin, (__nv_bfloat16*)p.dv, dkp, dh0w, saved_anch ? saved_anch : anch,
                cpart, flag, Tv, p.V, fflags);
        else
            k_bwd_dkv3<K, 1><<<grid, Dkv3Cfg<K>::NTHR, Dkv3Cfg<K>::SMEM, sv>>>(
                mQ, mK, mP, mDP, mV, mD, stats, dfin, (__nv_bfloat16*)p.dv, dkp, dh0w, saved_anch ? saved_anch : anch,
                cpart, flag, Tv, p.V, nullptr);
    }
    if (sv != st) {
        if ((e = cudaEventRecord(ev_dv, sv)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(st, ev_dv, 0)) != cudaSuccess) return e;
    }
    // The exact-fallback gate (one-warp kernel; tail-launches the CUDA-core backward only when a chunk failed
    // the guard) runs on the dq stream right after the dq walk, overlapping the dkv walk and the reduce; the TC
    // kernels return at once when the flag is set, so the fallback's writes never race with theirs.
    BwdProblem sp = p;
    sp.ws = ws + used;
    sp.run_if = flag;
    cudaEvent_t ev_gate = nullptr;
    if (sq != st) {
        if ((e = cudaEventRecord(ev_out, sq)) != cudaSuccess) return e;
        if ((e = simt::bwd(sp, sq)) != cudaSuccess) return e;
        if (!(ev_gate = fork_event(2))) return cudaErrorUnknown;
        if ((e = cudaEventRecord(ev_gate, sq)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(st, ev_out, 0)) != cudaSuccess) return e;
    }
    {
        GLA_PROF("tc::bwd_reduce", st);
        CUtensorMap mQr, mKr, mGr, mDQP, mDKP;
        const uint64_t prow = (uint64_t)NVT * BH * p.T;
        if ((e = make_map_2d_ex(&mQr, p.q, 2, rows, K, 64, 64, true)) != cudaSuccess) return e;
        if ((e = make_map_2d_ex(&mKr, p.k, 2, rows, K, 64, 64, true)) != cudaSuccess) return e;
        if ((e = make_map_2d_ex(&mGr, p.g, (int)sizeof(TG), rows, K, sizeof(TG) == 4 ? 32 : 64, 64, true)) != cudaSuccess)
            return e;
        if (kw) {   // fp32 [BH*T][K], boxes [64 rows][32 fp32]
            if ((e = make_map_2d_ex(&mDQP, dq32, 4, (uint64_t)rows, K, 32, 64, true)) != cudaSuccess)
                return e;
        } else if ((e = make_map_2d_ex(&mDQP, dqp, 2, prow, K, 64, 64, true)) != cudaSuccess) {
            return e;
        }
        if (kw) {
            if ((e = make_map_2d_ex(&mDKP, dk32, 4, (uint64_t)rows, K, 32, 64, true)) != cudaSuccess)
                return e;
        } else if ((e = make_map_2d_ex(&mDKP, dkp, 2, prow, K, 64, 64, true)) != cudaSuccess) {
            return e;
        }
        const float* sd = dfin ? stdot : nullptr;
        __nv_bfloat16 *dq_ = (__nv_bfloat16*)p.dq, *dk_ = (__nv_bfloat16*)p.dk;
        const int NCv = NC / S;
        const dim3 rg(K / 64, BHv, (NCv + ANCH - 1) / ANCH);
#define GLA_RED(N, NQ32)                                                                                           \
    case N:                                                                                                         \
        if ((e = cudaFuncSetAttribute(k_bwd_reduce_tma<K, N, TG, NQ32>, cudaFuncAttributeMaxDynamicSharedMemorySize,\
                                      (int)RedCfg<N, TG, NQ32>::SMEM)) != cudaSuccess)                              \
            return e;                                                                                               \
        k_bwd_reduce_tma<K, N, TG, NQ32><<<rg, 288, RedCfg<N, TG, NQ32>::SMEM, st>>>(                               \
            mQr, mKr, mGr, mDQP, mDKP, sd, NQ32 ? p.V / 256 : NVT, dq_, dk_, p.dg, cpart, flag, Tv, BHv,             \
            NQ32 ? fflags : nullptr, NQ32 ? dPm : nullptr);                                                         \
        break;
        if (kw) {   // one combined fp32 dq and dk per element (the walks sum the value halves)
            switch (NVT) {
                GLA_RED(2, 1) GLA_RED(4, 1)
                default: return cudaErrorNotSupported;
            }
        } else {
            switch (NVT) {
                GLA_RED(1, 0) GLA_RED(2, 0) GLA_RED(4, 0) GLA_RED(8, 0)
                default: return cudaErrorNotSupported;
            }
        }
#undef GLA_RED
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (S > 1 && p.dh0) {   // the first segment's d_initial_state of every (b,h) (skipped when the fallback runs)
        const size_t n4 = (size_t)BH * K * p.V / 4;
        k_copy_seg0<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(p.dh0, dhv, BH, S, (size_t)K * p.V, flag);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    if (sq != st) return cudaStreamWaitEvent(st, ev_gate, 0);
    return simt::bwd(sp, st);
}


cudaError_t bwd_tc(const BwdProblem& p, cudaStream_t st) {
    const bool gf = p.gate_dtype == 1;
    switch (p.K) {
        case 128:
            return gf ? launch_bwd2<128, float>(p, st) : launch_bwd2<128, __nv_bfloat16>(p, st);
        case 256:
            return gf ? launch_bwd2<256, float>(p, st) : launch_bwd2<256, __nv_bfloat16>(p, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace tc
}  // namespace gla
