// tc_fwd2.cu -- chunk-wise GLA forward as two tensor-core kernels (the default forward of the TC path).
//
//   k_fwd_prep  (chunk-parallel, one CTA per (b,h, chunk)): steps (1) and (3) of the method, everything that
//               does not depend on the state -- chunk-local log-space cumsum, the factorised
//               operands Q~ = q e^{b-r}, K~ = k e^{r-b} (r = b at the chunk's middle row), and the intra-chunk
//               score matrix P = (Q~ K~^T) (.) M as one stacked hi/lo tcgen05 MMA (fp32-class
//               accuracy on every sub-chunk block, in particular the diagonal ones).  Writes Q~hi, K~hi,
//               P (bf16, TMA stores) and the per-chunk per-channel r, Gamma (fp32) -- once per (b,h,chunk).
//   k_fwd_state (sequential over chunks, one CTA per (b,h) x 128-wide V tile): step (2) -- the inter-chunk
//               state passing with the d_k x 128 state tile resident in TMEM and the output
//               O = Q~ (H e^r) + P V.  All of its inputs arrive by TMA (Q~hi, K~hi, V, P double-buffered), so
//               no CUDA-core time goes to loading or rebuilding operands per V tile.
// Compared with one fused kernel per (b,h) x V tile (the first design, in git history), the operand
// construction and P run once per chunk instead of once per V tile (4x at d_v' = 512), at the price of writing /
// re-reading Q~hi, K~hi and P (2.1 KB per token-head at K = 256).  Exact path for chunks failing the
// factorisation guard: Q~ = q e^{b}, K~ = k e^{Gamma-b} (every factor <= 1; the state kernel applies the decay
// before the update) and P from the paper's per-sub-chunk-pair normalisers taken down to single
// tokens: six levels of sub-chunk pairs, each one stacked hi/lo tensor-core product whose two factors are <= 1
// (see k_fwd_prep).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>

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
#ifndef GLA_FWD_OB2
#define GLA_FWD_OB2 1
#endif
#ifndef GLA_PREP_PFD
#define GLA_PREP_PFD 1   // L2 prefetch distance of the prep, in items per CTA (measured: 1 86 us, 2 90.5, 3-4 106)
#endif
#ifndef GLA_PREP_PF
#define GLA_PREP_PF 1
#endif

// ---------------------------------------------------------------------------------------------------------------
template <int K>
struct PrepCfg {
    using Tl = Tile<K>;
    static constexpr int KB = K / 64;
    static constexpr uint32_t OP = KB * 16384;          // [KB][128 rows: hi | lo][128 B]
    static constexpr uint32_t OFF_Q = 0, OFF_K = OP, OFF_P = 2 * OP;       // P [64 t][128 B]
    static constexpr uint32_t OFF_X = OFF_P + 8192;     // exchange [64][64] fp32 and gtot
    static constexpr uint32_t OFF_B = OFF_X + 16384;    // exact path: b at each row group's last row [RG][K], diag [64]
    static constexpr uint32_t SMEM = OFF_B + Tl::RG * K * 4 + 256 + 1024;
    static_assert(Tl::RG * K * 4 <= 16384, "gtot fits the exchange buffer");
};

// The exact-path P of k_fwd_prep, for each of the calling CTA's items whose chunk failed the factorisation guard
// (R9).  P[t][s] = sum_k q_tk k_sk e^{b_tk - b_sk}, s <= t, with the paper's per-pair normalisers
// on a binary hierarchy of sub-chunks taken down to single tokens: at level h (half size 32, 16, ..., 1) the
// chunk splits into groups of 2h rows, an earlier half E and a later half F with normaliser c = the last row of E,
// and for t in F, s in E of the same group
//     P[t][s] = sum_k (q_tk e^{b_tk - b_ck}) (k_sk e^{b_ck - b_sk}),
// both factors <= 1 whatever the gates.  Every pair s < t lies in exactly one level's F x E block of one group
// (the level where t and s first separate); the diagonal P[t][t] = q_t . k_t needs no factor.  A level is the
// product of Q_h (rows in F scaled, rows in E zero) and K_h (rows in E scaled, rows in F zero); two levels share
// one 128 x 128 x K tensor-core MMA (level A on operand rows 0-63, level B on rows 64-127; the diagonal blocks of
// the product are the two levels), so the six levels take three MMA rounds.  Operands are bf16 (no hi/lo split:
// every factor is <= 1, and P is stored in bf16).  Returns the bar parity.
template <int K, typename TG>
__device__ __noinline__ uint32_t exact_P_phase(const CUtensorMap* tmP, const __nv_bfloat16* __restrict__ q,
                                               const __nv_bfloat16* __restrict__ k, const TG* __restrict__ g,
                                               const int* __restrict__ flags, int T, int NC, int nitems, uint8_t* sm,
                                               uint32_t tP, uint64_t* barp, uint32_t phase) {
    using Cfg = PrepCfg<K>;
    using Tl = typename Cfg::Tl;
    uint8_t* sQ = sm + Cfg::OFF_Q;
    uint8_t* sK = sm + Cfg::OFF_K;
    uint8_t* sP = sm + Cfg::OFF_P;
    float* gtot = reinterpret_cast<float*>(sm + Cfg::OFF_X);
    float* bnd = reinterpret_cast<float*>(sm + Cfg::OFF_B);
    float* diag = bnd + Tl::RG * K;
    uint64_t& bar = *barp;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int oc = tid % Tl::NOCT, rg = tid / Tl::NOCT;
    const int ch0 = 8 * oc, row0 = rg * Tl::RPG;
    const int blk = ch0 >> 6, col = ch0 & 63;
    uint8_t* qb = sQ + blk * 16384;
    uint8_t* kb = sK + blk * 16384;
    const int lq = warp & 3, half = warp >> 2;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int vrow = 32 * lq + lane;
    ChunkRegs<K> R;
    for (int it2 = blockIdx.x; it2 < nitems; it2 += gridDim.x) {
        if (!flags[it2]) continue;   // (written by this CTA in the main loop; ordered by its barriers)
        const int chunk = it2 % NC, bh = it2 / NC;
        const size_t crow = (size_t)bh * T + (size_t)chunk * CH;
        load_chunk<K, TG, true, true>(R, q, k, g, crow, row0, ch0);
        if (tid == 0) tma_store_wait_read();    // earlier stores have read sQ / sK / sP
        float2 off[4], rr[4], Gm[4];
        chunk_cumsum<K>(R, gtot, rg, ch0, off, rr, Gm);
#pragma unroll
        for (int r = 0; r < Tl::RPG; ++r)       // R.g <- b (chunk-local cumsum)
#pragma unroll
            for (int p = 0; p < 4; ++p) R.g[r][p] = add2(R.g[r][p], off[p]);
        {   // b at this thread's last row (the normaliser rows of the coarse levels) and the diagonal
            float4* bb = reinterpret_cast<float4*>(bnd + rg * K + ch0);
            const int rl = Tl::RPG - 1;
            bb[0] = make_float4(R.g[rl][0].x, R.g[rl][0].y, R.g[rl][1].x, R.g[rl][1].y);
            bb[1] = make_float4(R.g[rl][2].x, R.g[rl][2].y, R.g[rl][3].x, R.g[rl][3].y);
#pragma unroll
            for (int r = 0; r < Tl::RPG; ++r) {
                float d = 0.f;
#pragma unroll
                for (int p = 0; p < 4; ++p) {
                    const float2 qv = unpack2(word(R.q[r], p)), kv = unpack2(word(R.k[r], p));
                    d = fmaf(qv.x, kv.x, fmaf(qv.y, kv.y, d));
                }
#pragma unroll
                for (int o = Tl::NOCT / 2; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                if (oc == 0) diag[row0 + r] = d;
            }
        }
        __syncthreads();   // bnd, diag visible
        if (lq < 2) {      // P rows t, columns [32 half, +32): zeros above the diagonal, the diagonal
            const int t = vrow;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                *reinterpret_cast<uint4*>(sP + sw128_off(t, 32 * half + 8 * u)) = make_uint4(0u, 0u, 0u, 0u);
            if ((t >> 5) == half)
                *reinterpret_cast<__nv_bfloat16*>(sP + sw128_off(t, t)) = __float2bfloat16_rn(diag[t]);
        }
        // (P entries are written by the epilogue threads of later rounds: each owns disjoint (t, s))
#pragma unroll   // (unrolled: every level's normaliser rows are compile-time, own-row ones static registers)
        for (int hA = 32; hA >= 2; hA >>= 2) {   // rounds: levels (32, 16), (8, 4), (2, 1)
#pragma unroll
            for (int lv = 0; lv < 2; ++lv) {
                const int h = lv ? hA >> 1 : hA, ro = 64 * lv;   // operand rows ro + t
#pragma unroll
                for (int r = 0; r < Tl::RPG; ++r) {
                    const int t = row0 + r, c = (t / (2 * h)) * 2 * h + h - 1;
                    float2 bc[4];
                    if (h >= Tl::RPG) {   // c is the last row of row group (c + 1) / RPG - 1
                        const float4* bb = reinterpret_cast<const float4*>(bnd + ((c + 1) / Tl::RPG - 1) * K + ch0);
                        const float4 x0 = bb[0], x1 = bb[1];
                        bc[0] = make_float2(x0.x, x0.y); bc[1] = make_float2(x0.z, x0.w);
                        bc[2] = make_float2(x1.x, x1.y); bc[3] = make_float2(x1.z, x1.w);
                    } else {              // c is one of this thread's rows: row0 + (r / 2h) 2h + h - 1
                        const int rc = (r / (2 * h)) * 2 * h + h - 1;
#pragma unroll
                        for (int p = 0; p < 4; ++p) bc[p] = R.g[rc][p];
                    }
                    uint8_t* qh = qb + sw128_off(ro + t, col);
                    uint8_t* kh = kb + sw128_off(ro + t, col);
                    float2 ref[4];
                    if (t > c) {          // F: Q row q e^{b_t - b_c}, K row zero
#pragma unroll
                        for (int p = 0; p < 4; ++p) ref[p] = make_float2(-L2E * bc[p].x, -L2E * bc[p].y);
                        scaled_row(R.q[r], R.g[r], ref, 1.f, qh, nullptr);
                        *reinterpret_cast<uint4*>(kh) = make_uint4(0u, 0u, 0u, 0u);
                    } else {              // E: K row k e^{b_c - b_t}, Q row zero
#pragma unroll
                        for (int p = 0; p < 4; ++p) ref[p] = make_float2(L2E * bc[p].x, L2E * bc[p].y);
                        scaled_row(R.k[r], R.g[r], ref, -1.f, kh, nullptr);
                        *reinterpret_cast<uint4*>(qh) = make_uint4(0u, 0u, 0u, 0u);
                    }
                }
            }
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                tc_fence_after();
                const uint32_t idP = idesc_bf16(128, 128, 0, 0);
                const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK);
#pragma unroll
                for (int kk = 0; kk < K / 16; ++kk) {
                    const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
                    mma_bf16(tP, sdesc_sw128(aQ + o, 16, 1024), sdesc_sw128(aK + o, 16, 1024), idP, kk > 0);
                }
                mma_commit(&bar);
            }
            mbar_wait(&bar, phase);
            phase ^= 1;
            tc_fence_after();
            {   // lanes 0-63: level A's rows (columns 0-63), lanes 64-127: level B's rows (columns 64-127)
                const int lv = lq >> 1, h = lv ? hA >> 1 : hA, t = vrow - 64 * lv;
                uint32_t a[32];
                tmem_ld32(tP + lane_base + 64 * lv + 32 * half, a);
                tmem_wait_ld();
                const int g0 = (t / (2 * h)) * 2 * h;
                if (t >= g0 + h) {    // t in F: keep the E columns of its own group
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int s = 32 * half + j;
                        if (s >= g0 && s < g0 + h)
                            *reinterpret_cast<__nv_bfloat16*>(sP + sw128_off(t, s)) =
                                __float2bfloat16_rn(__uint_as_float(a[j]));
                    }
                }
            }
            tc_fence_before();
            __syncthreads();   // the TMEM accumulator free, sQ / sK writable again
        }
        fence_async_smem();
        __syncthreads();
        if (tid == 0) {
            tma_store_2d(tmP, sP, 0, (int)crow);
            tma_store_commit();
        }
    }
    return phase;
}

// Persistent: CTA c processes work items (b,h, chunk) c, c + gridDim.x, ...  The next item's q / k / log alpha
// are loaded into the (then dead) operand registers right after the current item's operand build, so their
// HBM latency overlaps this item's P MMA, epilogue and stores (one CTA per SM: the kernel is register- and
// shared-memory-heavy, so the overlap has to come from within the CTA).
template <int K, typename TG>
__global__ void __launch_bounds__(NTH, 1)
k_fwd_prep(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmP, const __nv_bfloat16* __restrict__ q,
           const __nv_bfloat16* __restrict__ k, const TG* __restrict__ g, float* __restrict__ stats,
           int* __restrict__ flags, int T, int NC, int nitems) {
    using Cfg = PrepCfg<K>;
    using Tl = typename Cfg::Tl;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sQ = sm + Cfg::OFF_Q;
    uint8_t* sK = sm + Cfg::OFF_K;
    uint8_t* sP = sm + Cfg::OFF_P;
    float* exch = reinterpret_cast<float*>(sm + Cfg::OFF_X);
    float* gtot = exch;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int oc = tid % Tl::NOCT, rg = tid / Tl::NOCT;
    const int ch0 = 8 * oc, row0 = rg * Tl::RPG;

    if (warp == 0) tmem_alloc(&tmem_base, 128);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmP);
    }
    ChunkRegs<K> R;
    int item = blockIdx.x;
    // L2 prefetch of a later item's q / k / log alpha rows (contiguous: rows [crow, crow + 64) x K), so HBM stays busy
    // through the operand build, when the register prefetch below has nothing in flight.
    auto prefetch_item = [&](int it) {
        if (it >= nitems) return;
        const size_t r0 = (size_t)(it / NC) * T + (size_t)(it % NC) * CH;
        constexpr uint32_t QB = CH * K * 2, GB = CH * K * sizeof(TG), PIECE = 16384;
        for (uint32_t o = 0; o < QB; o += PIECE) {
            prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(q + r0 * K) + o, PIECE < QB - o ? PIECE : QB - o);
            prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(k + r0 * K) + o, PIECE < QB - o ? PIECE : QB - o);
        }
        for (uint32_t o = 0; o < GB; o += PIECE)
            prefetch_l2_bulk(reinterpret_cast<const uint8_t*>(g + r0 * K) + o, PIECE < GB - o ? PIECE : GB - o);
    };
    if (tid == 32)
        for (int d = 1; d < GLA_PREP_PFD; ++d) prefetch_item(item + d * gridDim.x);
    if (item < nitems)
        load_chunk<K, TG, true, true>(R, q, k, g, (size_t)(item / NC) * T + (size_t)(item % NC) * CH, row0, ch0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tP = tmem_base;
    uint32_t phase = 0;                         // parity of the next wait on bar (one commit per MMA round)
    for (; item < nitems; item += gridDim.x) {
        const int chunk = item % NC, bh = item / NC;
        const size_t crow = (size_t)bh * T + (size_t)chunk * CH;
        if (tid == 0) tma_store_wait_read();    // the previous item's Q~ / K~ / P stores have read their smem
        if (tid == 32 && GLA_PREP_PF) prefetch_item(item + GLA_PREP_PFD * gridDim.x);
        float2 off[4], rr[4], Gm[4];
        chunk_cumsum<K>(R, gtot, rg, ch0, off, rr, Gm);   // (its barrier also orders the wait above)
        bool bad = false;
        if (rg == 0)
#pragma unroll
            for (int p = 0; p < 4; ++p)
                bad |= (-rr[p].x > GUARD) | (-rr[p].y > GUARD) | (rr[p].x - Gm[p].x > GUARD) | (rr[p].y - Gm[p].y > GUARD);
        const bool slow = __syncthreads_or(bad) != 0;
        if (rg == 0) {   // per-chunk statistics for the state kernel: r (row 31) and Gamma (row 63)
            float* st = stats + ((size_t)bh * NC + chunk) * 2 * K + ch0;
            reinterpret_cast<float4*>(st)[0] = make_float4(rr[0].x, rr[0].y, rr[1].x, rr[1].y);
            reinterpret_cast<float4*>(st)[1] = make_float4(rr[2].x, rr[2].y, rr[3].x, rr[3].y);
            reinterpret_cast<float4*>(st + K)[0] = make_float4(Gm[0].x, Gm[0].y, Gm[1].x, Gm[1].y);
            reinterpret_cast<float4*>(st + K)[1] = make_float4(Gm[2].x, Gm[2].y, Gm[3].x, Gm[3].y);
            if (tid == 0) flags[(size_t)bh * NC + chunk] = slow ? 1 : 0;
        }
        float2 refq[4], refk[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float2 rq = slow ? make_float2(0.f, 0.f) : rr[p], rk = slow ? Gm[p] : rr[p];
            refq[p] = make_float2(-L2E * rq.x, -L2E * rq.y);
            refk[p] = make_float2(L2E * rk.x, L2E * rk.y);
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
        {   // the operand registers are dead: start loading the next item (overlaps MMA, epilogue, stores)
            const int nx = item + gridDim.x;
            if (nx < nitems)
                load_chunk<K, TG, true, true>(R, q, k, g, (size_t)(nx / NC) * T + (size_t)(nx % NC) * CH, row0, ch0);
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            if (!slow) {
                const uint32_t idP = idesc_bf16(128, 128, 0, 0);
                const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK);
#pragma unroll
                for (int kk = 0; kk < K / 16; ++kk) {
                    const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
                    mma_bf16(tP, sdesc_sw128(aQ + o, 16, 1024), sdesc_sw128(aK + o, 16, 1024), idP, kk > 0);
                }
            }
            mma_commit(&bar);
            // Q~hi and K~hi (rows 0-63 of each 64-channel block) -> HBM, swizzle undone by the TMA engine
            for (int c = 0; c < K / 64; ++c) {
                tma_store_2d(&tmQ, sQ + c * 16384, 64 * c, (int)crow);
                tma_store_2d(&tmK, sK + c * 16384, 64 * c, (int)crow);
            }
            tma_store_commit();
        }
        const int lq = warp & 3, half = warp >> 2;
        const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
        const int vrow = 32 * lq + lane;
        mbar_wait(&bar, phase);   // the P MMA (if any) has completed
        phase ^= 1;
        tc_fence_after();
        if (!slow) {
            if (lq >= 2) {   // lo rows: lh + ll
                uint32_t a[32], b[32];
                tmem_ld32(tP + lane_base + 32 * half, a);
                tmem_ld32(tP + lane_base + 64 + 32 * half, b);
                tmem_wait_ld();
                const int t = vrow - 64;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    exch[t * 64 + ((32 * half + j + t) & 63)] = __uint_as_float(a[j]) + __uint_as_float(b[j]);
            }
            __syncthreads();
            if (lq < 2) {    // hi rows: hh + hl + exchange, causal mask, bf16
                uint32_t a[32], b[32];
                tmem_ld32(tP + lane_base + 32 * half, a);
                tmem_ld32(tP + lane_base + 64 + 32 * half, b);
                tmem_wait_ld();
                const int t = vrow;
                uint32_t pk[16];
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const int s = 32 * half + j;
                    float p0 = __uint_as_float(a[j]) + __uint_as_float(b[j]) + exch[t * 64 + ((s + t) & 63)];
                    float p1 = __uint_as_float(a[j + 1]) + __uint_as_float(b[j + 1]) + exch[t * 64 + ((s + 1 + t) & 63)];
                    pk[j / 2] = pack_bf16(s <= t ? p0 : 0.f, s + 1 <= t ? p1 : 0.f);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    *reinterpret_cast<uint4*>(sP + sw128_off(t, 32 * half + 8 * u)) =
                        make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            }
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();                         // P staged; TMEM P drained; exch free
        if (tid == 0 && !slow) {                 // (the exact path's P is written by the second phase below)
            tma_store_2d(&tmP, sP, 0, (int)crow);
            tma_store_commit();
        }
    }
    // Second phase: P of this CTA's chunks that failed the guard.  In the common case none did: one parallel read of
    // the CTA's flags (written above by this CTA, ordered by its barriers) skips it.  A separate, non-inlined
    // function so that its registers never compete with the prefetched operands above.
    bool any_exact = false;
    for (int b0 = 0; (size_t)blockIdx.x + (size_t)b0 * gridDim.x < (size_t)nitems; b0 += NTH) {
        const size_t it2 = blockIdx.x + (size_t)(b0 + tid) * gridDim.x;
        any_exact |= __syncthreads_or(it2 < (size_t)nitems && flags[it2] != 0) != 0;
    }
    if (any_exact) phase = exact_P_phase<K, TG>(&tmP, q, k, g, flags, T, NC, nitems, sm, tP, &bar, phase);
    if (tid == 0) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tP, 128);
}

// ---------------------------------------------------------------------------------------------------------------
// k_fwd_state: warp-specialised walk over the chunks of one (b,h) unit x 128-wide V tile.
//   warps 0-7   ("state"):    per chunk, the TMEM state pass: Y <- H_i e^{r} (in place, fp32) and
//                             SB = bf16(H_i e^{r}) written to TMEM as the A operand of the O MMAs;
//                             the next chunks' K~ / V / P loads; at the end final_state.
//   warp 8      ("mma S"):    the state update Y += V^T K~hi (N = K MMAs), commit bar_s.
//   warps 9, 10 ("mma O"):    O^T = SB Q~hi^T by channel half into one TMEM accumulator: warp 9 half 0 plus
//                             V^T P^T (intra-chunk), commit bar_oa; warp 10 half 1 after bar_oa
//                             (fixed accumulation order), commit bar_ob.
//   warps 11-14 ("epilogue"): O^T (TMEM) -> bf16 staging -> TMA store; the Q~ loads.
// Three issuing warps because one thread issues at most one tcgen05.mma per ~110 cycles whatever N is
// (profiles/r1_microbench.md): the state and output MMAs are issued from separate warps.  Serial chain per chunk: state MMA -> state pass -> state MMA; the O MMAs overlap the
// next pass; epilogue, TMA loads and stores overlap everything.  SB never touches shared memory.
template <int K>
struct StateCfg {
    static constexpr int KB = K / 64;
    static constexpr uint32_t OP = KB * 8192;            // [KB][64 t][128 B]  Q~hi or K~hi
    static constexpr uint32_t OFF_Q = 0, OFF_K = 2 * OP;        // 2 buffers each
    static constexpr uint32_t OFF_V = 4 * OP;                   // 2 buffers x [2][64 t][128 B]
    static constexpr uint32_t OFF_P = OFF_V + 2 * 16384;        // 2 buffers x [64 t][128 B]
    static constexpr uint32_t OFF_STG = OFF_P + 2 * 8192;       // O staging 2 buffers x [2][64 t][128 B]
    static constexpr uint32_t OFF_F = OFF_STG + 2 * 16384;      // fsb, fy, pend [K]
    static constexpr uint32_t SMEM = OFF_F + 4 * 3 * K + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
    // TMEM: Y [K] | SB bf16 pairs [K/2] | O [64] (64-column aligned; both O issuers accumulate into it in turn)
    static constexpr uint32_t COL_SB = K, COL_OA = (K + K / 2 + 63) / 64 * 64;
    // OB2: the two channel halves' output MMAs go to separate accumulators O_a, O_b, issued concurrently by warps 9
    // and 10 (one thread issues ~1 MMA per 120 cycles, so the ordered issue into one accumulator serialised ~16
    // issue slots per chunk); the epilogue sums O_a + O_b (fixed order: deterministic).
    static constexpr bool OB2 = GLA_FWD_OB2 && K >= 128;
    static constexpr uint32_t COL_OB = COL_OA + (OB2 ? 64 : 0);
    static constexpr uint32_t TCOLS = COL_OB + 64 > 256 ? 512 : 256;
    static constexpr int NST = 256, NTHR = NST + 3 * 32 + 128;  // state, 3 MMA issuers, epilogue
    static constexpr int NSB = K / 16;                           // K-steps of the SB Q~^T product
    static constexpr int NHALF = K >= 128 ? 2 : 1;               // channel halves of the pipelined state pass
    static constexpr int CPH = K / NHALF, CPT = CPH / 2;         // channels per half, per state thread and half
    static constexpr int NSB_A = NHALF == 2 ? NSB / 2 : NSB, NSB_B = NSB - NSB_A;   // O_a: half 0 (+ P V^T)
};

template <int K>
__global__ void __launch_bounds__(StateCfg<K>::NTHR, 1)
k_fwd_state(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmV,
            const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmA,
            const float* __restrict__ stats, const int* __restrict__ flags,
            const float* __restrict__ h0, float* __restrict__ final_state, __nv_bfloat16* __restrict__ anch, int T,
            int V, int emit) {
    // emit == 0: state-only walk (segment summaries): the output MMAs, epilogue and Q~ loads are skipped and
    // only final_state is produced (the barriers keep their arrivals so the schedule is unchanged).
    using Cfg = StateCfg<K>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sQ = sm + Cfg::OFF_Q;
    uint8_t* sK = sm + Cfg::OFF_K;
    uint8_t* sV = sm + Cfg::OFF_V;
    uint8_t* sP = sm + Cfg::OFF_P;
    uint8_t* stg = sm + Cfg::OFF_STG;
    float* fsb = reinterpret_cast<float*>(sm + Cfg::OFF_F);
    float* fy = fsb + K;
    float* pend = fy + K;
    __shared__ uint64_t bar_q[2], bar_k[2], bar_vp[2], bar_sbh[2], bar_sh[2], bar_oa, bar_ob, bar_ofree, bar_anch;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vt = blockIdx.x, bh = blockIdx.y;
    const int v0 = vt * VT, NC = T / CH;
    const int rowb = bh * T;
#ifdef GLA_PHASE_TIMING
    __shared__ long long trc[8][16];
#define TR(ev, i) do { if ((i) < 16) trc[ev][i] = clock64(); } while (0)
#else
#define TR(ev, i) do {} while (0)
#endif
    auto load_q = [&](int i) {
        const int b = i & 1;
        mbar_expect_tx(&bar_q[b], Cfg::OP);
        for (int c = 0; c < K / 64; ++c)
            tma_load_2d(sQ + b * Cfg::OP + c * 8192, &tmQ, &bar_q[b], 64 * c, rowb + i * CH);
    };
    auto load_k = [&](int i) {
        const int b = i & 1;
        mbar_expect_tx(&bar_k[b], Cfg::OP);
        for (int c = 0; c < K / 64; ++c)
            tma_load_2d(sK + b * Cfg::OP + c * 8192, &tmK, &bar_k[b], 64 * c, rowb + i * CH);
    };
    auto load_vp = [&](int i) {
        const int b = i & 1;
        mbar_expect_tx(&bar_vp[b], 16384 + 8192);
        tma_load_2d(sV + b * 16384, &tmV, &bar_vp[b], v0, rowb + i * CH);
        tma_load_2d(sV + b * 16384 + 8192, &tmV, &bar_vp[b], v0 + 64, rowb + i * CH);
        tma_load_2d(sP + b * 8192, &tmP, &bar_vp[b], 0, rowb + i * CH);
    };

    if (warp == 0) tmem_alloc(&tmem_base, Cfg::TCOLS);
    if (tid == 0) {
        mbar_init(&bar_q[0], 1); mbar_init(&bar_q[1], 1); mbar_init(&bar_k[0], 1); mbar_init(&bar_k[1], 1);
        mbar_init(&bar_vp[0], 1); mbar_init(&bar_vp[1], 1);
        mbar_init(&bar_sbh[0], 1); mbar_init(&bar_sbh[1], 1); mbar_init(&bar_sh[0], 1); mbar_init(&bar_sh[1], 1);
        mbar_init(&bar_oa, 1); mbar_init(&bar_ob, 1); mbar_init(&bar_ofree, 1); mbar_init(&bar_anch, 1);
        fence_mbar_init();
        prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmP); prefetch_tmap(&tmV); prefetch_tmap(&tmO);
        if (emit) load_q(0);
        load_k(0);
        load_vp(0);
        if (NC > 1) { if (emit) load_q(1); load_k(1); load_vp(1); }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tS = tmem_base, tSB = tmem_base + Cfg::COL_SB;
    const uint32_t tOa = tmem_base + Cfg::COL_OA, tOb = tmem_base + Cfg::COL_OB;
    const uint32_t lane_base = (uint32_t)(32 * (warp & 3)) << 16;
    const int vrow = 32 * (warp & 3) + lane;

    if (warp < 8) {
        // ------------------------------------------------------------------ state warps
        // Channel-half pipelining: the pass runs over channel half 0, signals, then half 1.  The state / output
        // MMAs of half 0 start while half 1 is being converted, and the next chunk's half-0 pass only waits for
        // the half-0 MMAs.  Warp w owns TMEM lane quadrant w%4 and the (w/4)-th quarter-share of every half.
        const int sub = warp >> 2;
        for (int m = tid; m < K; m += Cfg::NST) pend[m] = 0.f;
        for (int hh = 0; hh < Cfg::NHALF; ++hh)
            for (int c0 = hh * Cfg::CPH + sub * Cfg::CPT; c0 < hh * Cfg::CPH + (sub + 1) * Cfg::CPT; c0 += 32) {
                uint32_t r[32];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    r[j] = __float_as_uint(h0 ? h0[((size_t)bh * K + c0 + j) * V + v0 + vrow] : 0.f);
                tmem_st32(tS + lane_base + c0, r);
            }
        tmem_wait_st();
        float st_r = 0.f, st_G = 0.f;
        if (tid < K) {
            st_r = stats[((size_t)bh * NC) * 2 * K + tid];
            st_G = stats[((size_t)bh * NC) * 2 * K + K + tid];
        }
        int st_slow = flags[(size_t)bh * NC];
        named_bar_sync(1, Cfg::NST);           // pend initialised
        for (int i = 0; i < NC; ++i) {
            const float r_ = st_r, G_ = st_G;
            const bool slow = st_slow != 0;
            if (i + 1 < NC) {   // next chunk's statistics
                if (tid < K) {
                    st_r = stats[((size_t)bh * NC + i + 1) * 2 * K + tid];
                    st_G = stats[((size_t)bh * NC + i + 1) * 2 * K + K + tid];
                }
                st_slow = flags[(size_t)bh * NC + i + 1];
            }
            if (tid < K) {
                const float p = pend[tid];
                if (!slow) { fsb[tid] = ex2f((p + r_) * L2E); fy[tid] = fsb[tid]; pend[tid] = G_ - r_; }
                else { fsb[tid] = ex2f(p * L2E); fy[tid] = ex2f((p + G_) * L2E); pend[tid] = 0.f; }
            }
            named_bar_sync(1, Cfg::NST);       // fsb / fy visible
#pragma unroll 1
            for (int hh = 0; hh < Cfg::NHALF; ++hh) {
                if (i > 0) {                   // half hh of Y final for chunk i-1
                    mbar_wait(&bar_sh[hh], (i - 1) & 1);
                    tc_fence_after();
                    if (tid == 0 && hh == Cfg::NHALF - 1) {   // both state-MMA halves of chunk i-1 done: K~ buffer free
                        TR(0, i);
                        if (i + 1 < NC) load_k(i + 1);
                    }
                }
                const int cbeg = hh * Cfg::CPH + sub * Cfg::CPT;
                const uint32_t sba = tSB + lane_base + cbeg / 2;
#pragma unroll
                for (int s = 0; s < Cfg::CPT / 32; ++s) {   // 32-column slices of this thread's channels
                    const int cb = cbeg + 32 * s;
                    uint32_t pk[16];
                    uint32_t r[32];
                    tmem_ld32(tS + lane_base + cb, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 fs = *reinterpret_cast<const float4*>(fsb + cb + j);
                        const float4 fyv = *reinterpret_cast<const float4*>(fy + cb + j);
                        const float2 y0 = make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1]));
                        const float2 y1 = make_float2(__uint_as_float(r[j + 2]), __uint_as_float(r[j + 3]));
                        pk[j / 2] = pack2(mul2(y0, make_float2(fs.x, fs.y)));
                        pk[j / 2 + 1] = pack2(mul2(y1, make_float2(fs.z, fs.w)));
                        const float2 z0 = mul2(y0, make_float2(fyv.x, fyv.y)), z1 = mul2(y1, make_float2(fyv.z, fyv.w));
                        r[j] = __float_as_uint(z0.x); r[j + 1] = __float_as_uint(z0.y);
                        r[j + 2] = __float_as_uint(z1.x); r[j + 3] = __float_as_uint(z1.y);
                    }
                    tmem_st32(tS + lane_base + cb, r);
                    if (s == 0 && i > 0) {     // the output MMAs of chunk i-1 on this half (the readers of SB) done
                        if (tid == 0 && hh == 0) TR(6, i);
                        mbar_wait(hh == 0 ? &bar_oa : &bar_ob, (i - 1) & 1);
                        if (hh == 0 && anch && i - 1 > 0 && (i - 1) % ANCH == 0)   // epilogue copied SB_{i-1} out
                            mbar_wait(&bar_anch, ((i - 1) / ANCH - 1) & 1);
                        tc_fence_after();
                        if (tid == 0 && hh == Cfg::NHALF - 1) {   // V/P of chunk i+1 into the buffers i-1 used
                            TR(7, i);
                            // (O_a of chunk i-1, the P V reader, was waited for in half 0 by this thread; waiting
                            // on it again here could alias its next phase)
                            if (i + 1 < NC) load_vp(i + 1);
                        }
                    }
                    tmem_st16(sba + 16 * s, pk);
                }
                tmem_wait_st();
                tc_fence_before();
                named_bar_sync(1, Cfg::NST);   // half hh: SB written, Y decayed
                if (tid == 0) { if (hh == Cfg::NHALF - 1) TR(1, i); mbar_arrive(&bar_sbh[hh]); }
            }
        }
        mbar_wait(&bar_sh[Cfg::NHALF - 1], (NC - 1) & 1);
        if (Cfg::NHALF > 1) mbar_wait(&bar_sh[0], (NC - 1) & 1);
        tc_fence_after();
        if (final_state) {
            for (int hh = 0; hh < Cfg::NHALF; ++hh)
                for (int c0 = hh * Cfg::CPH + sub * Cfg::CPT; c0 < hh * Cfg::CPH + (sub + 1) * Cfg::CPT; c0 += 32) {
                    uint32_t r[32];
                    tmem_ld32(tS + lane_base + c0, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        final_state[((size_t)bh * K + c0 + j) * V + v0 + vrow] =
                            __uint_as_float(r[j]) * ex2f(pend[c0 + j] * L2E);
                }
        }
    } else if (warp == 8) {
        // ------------------------------------------------------------------ state MMA issuer (per channel half)
        const uint32_t idS = idesc_bf16(128, Cfg::CPH, 1, 1);   // Y[v][ch] += V^T K~hi over one channel half
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            const uint32_t aV = smem_u32(sV + b * 16384), aK = smem_u32(sK + b * Cfg::OP);
            for (int hh = 0; hh < Cfg::NHALF; ++hh) {
                mbar_wait(&bar_sbh[hh], i & 1);
                if (hh == 0) {
                    mbar_wait(&bar_k[b], (i >> 1) & 1);
                    mbar_wait(&bar_vp[b], (i >> 1) & 1);
                }
                tc_fence_after();
                if (lane == 0 && hh == 0) TR(2, i);
                const uint32_t aKh = aK + hh * (Cfg::CPH / 64) * 8192;
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk)
                    mma_bf16_w(tS + hh * Cfg::CPH, sdesc_sw128(aV + kk * 2048, 8192, 1024),
                               sdesc_sw128(aKh + kk * 2048, 8192, 1024), idS, 1);
                mma_commit_w(&bar_sh[hh]);
            }
            __syncwarp();
        }
    } else if (warp < 11) {
        // ------------------------------------------------------------------ O MMA issuers (a: half 0 + P V^T)
        const bool is_a = warp == 9;
        const uint32_t idO = idesc_bf16(128, 64, 0, 0);      // O^T[v][t] = SB . Q~hi^T  (SB from TMEM)
        const uint32_t idPV = idesc_bf16(128, 64, 1, 0);     // O^T += V^T P^T
        // O_b accumulates onto O_a after it (fixed order), or (OB2) into its own accumulator concurrently
        const uint32_t tD = (is_a || !Cfg::OB2) ? tOa : tOb;
        const int k0 = is_a ? 0 : Cfg::NSB_A, k1 = is_a ? Cfg::NSB_A : Cfg::NSB;
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            const uint32_t aQ = smem_u32(sQ + b * Cfg::OP);
            mbar_wait(&bar_sbh[is_a || Cfg::NHALF == 1 ? 0 : 1], i & 1);
            if (emit) mbar_wait(&bar_q[b], (i >> 1) & 1);
            if (is_a) mbar_wait(&bar_vp[b], (i >> 1) & 1);
            if (i >= 1) mbar_wait(&bar_ofree, (i - 1) & 1);
            if (!is_a && !Cfg::OB2) mbar_wait(&bar_oa, i & 1);   // O_a of this chunk complete: accumulate after it
            tc_fence_after();
            if (is_a && lane == 0) TR(3, i);
            if (emit)
                for (int kk = k0; kk < k1; ++kk)
                    mma_bf16_ta_w(tD, tSB + 8 * kk, sdesc_sw128(aQ + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), idO,
                                  (!is_a && !Cfg::OB2) || kk > k0);
            if (is_a && emit) {
                const uint32_t aV = smem_u32(sV + b * 16384), aP = smem_u32(sP + b * 8192);
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk)
                    mma_bf16_w(tD, sdesc_sw128(aV + kk * 2048, 8192, 1024), sdesc_sw128(aP + kk * 32, 16, 1024), idPV,
                               Cfg::NSB_A > 0 || kk > 0);
            }
            mma_commit_w(is_a ? &bar_oa : &bar_ob);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------------ epilogue warps
        const int et = tid - Cfg::NST - 96;    // 0..127
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            mbar_wait(&bar_oa, i & 1);
            mbar_wait(&bar_ob, i & 1);
            tc_fence_after();
            if (et == 0) {
                TR(4, i);
                if (emit && i + 2 < NC) load_q(i + 2);   // the O MMAs of chunk i (Q~ buffer b's readers) are complete
                tma_store_wait_read1();         // staging buffer b (chunk i-2) has been read
            }
            if (anch && i > 0 && i % ANCH == 0) {   // exact state SB_i = bf16(H_i e^{r}) for the backward's anchors
                // 64-channel pieces: TMEM -> alternately the two staging buffers (SW128) -> one TMA store each; a
                // buffer is reused only once its store two pieces earlier has been read, so stores overlap staging
                const int arow0 = (int)(((size_t)(i / ANCH - 1) * gridDim.y + bh) * V + v0);
                if (et == 0) tma_store_wait_read();   // both staging buffers free (incl. chunk i-1's O store)
#pragma unroll 1
                for (int pc = 0; pc < K / 64; ++pc) {   // TMEM column c holds channels 2c, 2c+1
                    uint8_t* tile = stg + (b ^ (pc & 1)) * 16384;
                    uint32_t r[32];
                    tmem_ld32(tSB + lane_base + 32 * pc, r);
                    tmem_wait_ld();
                    if (pc >= 2) {             // this buffer's previous piece has been read by its store
                        if (et == 0) tma_store_wait_read1();
                        named_bar_sync(2, 128);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        *reinterpret_cast<uint4*>(tile + sw128_off(vrow, 8 * u)) =
                            make_uint4(r[4 * u], r[4 * u + 1], r[4 * u + 2], r[4 * u + 3]);
                    fence_async_smem();
                    named_bar_sync(2, 128);
                    if (et == 0) {
                        tma_store_2d(&tmA, tile, 64 * pc, arow0);
                        tma_store_commit();
                    }
                }
                tc_fence_before();
                named_bar_sync(2, 128);        // every SB column has been read: the next pass may overwrite SB
                if (et == 0) {
                    mbar_arrive(&bar_anch);
                    tma_store_wait_read();     // staging buffers free again for the O drain below
                }
                named_bar_sync(2, 128);
            }
            if (!emit) {                       // state-only walk: nothing to drain, keep the schedule
                tc_fence_before();
                named_bar_sync(2, 128);
                if (et == 0) mbar_arrive(&bar_ofree);
                continue;
            }
            uint8_t* dst = stg + b * 16384 + (vrow >> 6) * 8192 + (vrow & 63) * 2;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t ra[32];
                tmem_ld32(tOa + 32 * h + lane_base, ra);   // O = O_a (O_b's MMAs accumulated onto it), or O_a + O_b
                if (Cfg::OB2) {
                    uint32_t rb[32];
                    tmem_ld32(tOb + 32 * h + lane_base, rb);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; ++j) ra[j] = __float_as_uint(__uint_as_float(ra[j]) + __uint_as_float(rb[j]));
                }
                tmem_wait_ld();
                if (h == 1) {
                    tc_fence_before();
                    named_bar_sync(2, 128);    // O drained; staging b free
                    if (et == 0) mbar_arrive(&bar_ofree);
                }
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    *reinterpret_cast<__nv_bfloat16*>(dst + (32 * h + j) * 128) =
                        __float2bfloat16_rn(__uint_as_float(ra[j]));
            }
            fence_async_smem();
            named_bar_sync(2, 128);
            if (et == 0) {
                const int trow = rowb + i * CH;
                tma_store_2d(&tmO, stg + b * 16384, v0, trow);
                tma_store_2d(&tmO, stg + b * 16384 + 8192, v0 + 64, trow);
                tma_store_commit();
                TR(5, i);
            }
        }
        if (et == 0) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
#ifdef GLA_PHASE_TIMING
    if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0) {
        const long long t0 = trc[1][0];
        printf("fwd_state trace (cycles from chunk 0 state-pass end): S0=bar_s(i-1) seen, s0done/obar=slice 0 "
               "done / O MMAs of i-1 seen, S1=pass done, M0=state MMA issue, M1=O_a issue, E0=O ready, E1=stored\n");
        for (int i = 1; i < 16 && i < NC; ++i)
            printf("  chunk %2d: S0 %7lld s0done %7lld obar %7lld S1 %7lld M0 %7lld M1 %7lld E0 %7lld E1 %7lld\n", i,
                   trc[0][i] - t0, trc[6][i] - t0, trc[7][i] - t0, trc[1][i] - t0, trc[2][i] - t0, trc[3][i] - t0,
                   trc[4][i] - t0, trc[5][i] - t0);
    }
#endif
    if (warp == 0) tmem_dealloc(tmem_base, Cfg::TCOLS);
}

// ---------------------------------------------------------------------------------------------------------------
// k_seg_summary: the end state of one segment from a zero start, as ONE contraction over the segment's tokens
// instead of a serial walk (segment split):
//     S_loc[k][v] = sum_{t in seg} k_t[k] e^{sum_{u=t+1}^{end} log alpha_u[k]} v_t[v]
// (the recurrence S_t = diag(alpha_t) S_{t-1} + k_t^T v_t of P:188-189 unrolled over the segment; every decay
// factor is <= 1, so no normaliser and no exact path are needed).  One CTA per (128 channels, 256 values, unit):
// it walks the segment's 64-token blocks, scales the TMA-loaded K~hi tile in shared memory by a per-channel factor
// from the chunk statistics (see the kernel), and issues the 128 x 256 x 64 MMA of the block into a TMEM
// accumulator.  Blocks are independent apart from the carried per-channel sum of Gamma, so the scaling of block j
// overlaps the MMAs of earlier blocks and the loads of later ones.
struct SumCfg {
    static constexpr int NS = 4;   // TMA stages (loads run NS-1 blocks ahead of the scaling warps)
    static constexpr uint32_t A_BYTES = 2 * 8192, B_BYTES = 4 * 8192, STAGE = A_BYTES + B_BYTES;
    static constexpr uint32_t SMEM = NS * STAGE + 1024;
};
// ADJ = 1: the adjoint summary of the backward (a segment's d_initial_state with a zero d_final_state),
//     dh_loc[k][v] = sum_{t in seg} q_t[k] e^{sum_{u=start}^{t} log alpha_u[k]} dO_t[v],
// the same contraction with A = Q~hi (.) e^{r + carry} (Q~hi = q e^{b - r}; exact-path chunks q e^{b}) walked from
// the segment's start, B = dO.
template <int ADJ>
__global__ void __launch_bounds__(288, 1)
k_seg_summary(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmK,
              const float* __restrict__ stats, const int* __restrict__ flags, float* __restrict__ S_loc, int K, int V,
              int Tv, int S, int skip, int P, float* __restrict__ dec) {
    // skip = 1 (segment split): the summary nobody reads is not computed -- the last segment's end state (the
    // forward chain stops before it; the full walk writes the final state) / the first segment's adjoint (the
    // backward chain stops after segment 1; the dv walk writes d_initial_state).  blockIdx.z then enumerates the
    // (b,h) x (S - 1) remaining segments.
    // ADJ = 0: A = K~hi (.) e^{Gamma - r + carry}: the prep kernel's K~hi = k e^{r - b} (exact-path chunks:
    // k e^{Gamma - b}) times a per-channel factor <= 1, so A_t = k_t e^{sum_{u > t} log alpha_u} (suffix to the
    // segment's end); the carry (sum of Gamma over the later chunks) comes from the per-chunk statistics.
    // (tmK / tmV name the forward's operands; ADJ = 1 passes Q~hi / dO.)
    // Warps 0-7 scale the A tiles; warp 8 issues the TMA loads and the MMAs (handed over through bar_a), so the
    // scaling warps never wait for the tensor pipe.
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    constexpr int NS = SumCfg::NS;
    __shared__ uint64_t bar_v[NS], bar_free[NS], bar_a[NS];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(16) float fac[2][128];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int k0 = 128 * blockIdx.x, v0 = 256 * blockIdx.y;
    // P > 1: blockIdx.z also enumerates P token ranges of the segment (walk steps [part nbp, (part+1) nbp)); the
    // partial sums go to S_loc[(unit P + part)] and the chains add them in part order.
    const int nseg = S - skip, part = (int)(blockIdx.z % P), zz = (int)(blockIdx.z / P);
    const int bh = zz / nseg, seg = zz % nseg + (ADJ ? skip : 0);
    const size_t unit = (size_t)bh * S + seg, rowb = unit * (size_t)Tv;
    const int nbs = Tv / CH, NC = nbs * S, nb = nbs / P, j0 = part * nb;   // this CTA's walk steps: j0 + [0, nb)
    if (warp == 0) tmem_alloc(&tmem_base, 256);
    if (tid == 0) {
        for (int j = 0; j < NS; ++j) { mbar_init(&bar_v[j], 1); mbar_init(&bar_free[j], 1); mbar_init(&bar_a[j], 256); }
        fence_mbar_init();
        prefetch_tmap(&tmV); prefetch_tmap(&tmK);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tD = tmem_base;
    if (warp == 8) {
        // ------------------------------------------------------------ producer + MMA issuer (one lane)
        if (lane == 0) {
            const uint32_t idS = idesc_bf16(128, 256, 1, 1);   // D[k][v] += A^T[k][t] B[t][v], both MN-major
            auto load_blk = [&](int j) {                       // K~hi and V of block j -> stage j % NS
                uint8_t* sA = sm + (j % NS) * SumCfg::STAGE;
                uint64_t* bar = &bar_v[j % NS];
                const int r0 = (int)(rowb + (size_t)(ADJ ? j0 + j : nbs - 1 - (j0 + j)) * CH);
                mbar_expect_tx(bar, SumCfg::STAGE);
                tma_load_2d(sA, &tmK, bar, k0, r0);
                tma_load_2d(sA + 8192, &tmK, bar, k0 + 64, r0);
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4)
                    tma_load_2d(sA + SumCfg::A_BYTES + q4 * 8192, &tmV, bar, v0 + 64 * q4, r0);
            };
            for (int j = 0; j < NS - 1 && j < nb; ++j) load_blk(j);
            for (int j = 0; j < nb; ++j) {
                const int bs = j % NS;
                mbar_wait(&bar_a[bs], (j / NS) & 1);   // A of block j scaled
                tc_fence_after();
                const uint32_t aA = smem_u32(sm + bs * SumCfg::STAGE), aB = aA + SumCfg::A_BYTES;
#pragma unroll
                for (int kk = 0; kk < CH / 16; ++kk)
                    mma_bf16(tD, sdesc_sw128(aA + kk * 2048, 8192, 1024), sdesc_sw128(aB + kk * 2048, 8192, 1024),
                             idS, (j | kk) > 0);
                mma_commit(&bar_free[bs]);
                if (j + NS - 1 < nb) {                 // block j+NS-1 into the stage block j-1 used
                    if (j >= 1) mbar_wait(&bar_free[(j - 1) % NS], ((j - 1) / NS) & 1);
                    load_blk(j + NS - 1);
                }
            }
        }
        __syncwarp();
    } else {
        // ------------------------------------------------------------ scaling warps 0-7
        float carry = 0.f;                             // channel tid (< 128): sum of Gamma over the passed chunks
        float nr = 0.f, nG = 0.f;                      // (r, Gamma, flag) of the next block, loaded one ahead
        int nf = 0;
        auto chunk_idx = [&](int j) {                  // walk step j of the segment -> chunk index
            return (size_t)bh * NC + (size_t)seg * nbs + (ADJ ? j : nbs - 1 - j);
        };
        auto load_st = [&](int j) {
            const size_t ci = chunk_idx(j0 + j);
            nr = stats[ci * 2 * K + k0 + tid];
            nG = stats[ci * 2 * K + K + k0 + tid];
            nf = flags[ci];
        };
        if (tid < 128) {
            for (int j = 0; j < j0; ++j) carry += stats[chunk_idx(j) * 2 * K + K + k0 + tid];   // earlier parts' chunks
            load_st(0);
        }
        for (int j = 0; j < nb; ++j) {
            const int bs = j % NS;
            uint8_t* sA = sm + bs * SumCfg::STAGE;
            float* fj = fac[j & 1];
            if (tid < 128) {
                const float r_ = nr, G_ = nG;
                fj[tid] = ex2f(((nf ? 0.f : (ADJ ? r_ : G_ - r_)) + carry) * L2E);
                carry += G_;
                if (j + 1 < nb) load_st(j + 1);
            }
            named_bar_sync(1, 256);                    // fac[j & 1] written (its readers of block j-2 are done)
            // thread tid scales channels 8 (tid % 16) + [0, 8) of rows tid / 16 + 16 e: its 8 factors are read once
            // (two 16-byte loads), and each quarter-warp touches the 8 positions of one 128-byte row (no conflicts)
            const int c8 = tid & 15, blk = c8 >> 3;
            const float4 f0 = *reinterpret_cast<const float4*>(fj + 8 * c8);
            const float4 f1 = *reinterpret_cast<const float4*>(fj + 8 * c8 + 4);
            const float fv[8] = {f0.x, f0.y, f0.z, f0.w, f1.x, f1.y, f1.z, f1.w};
            mbar_wait(&bar_v[bs], (j / NS) & 1);
#pragma unroll
            for (int e = 0; e < 4; ++e) {              // 1024 16-byte chunks of the two SW128 blocks
                const int row = (tid >> 4) + 16 * e, pos = (c8 & 7) ^ (row & 7);
                uint4* pch = reinterpret_cast<uint4*>(sA + blk * 8192 + row * 128 + pos * 16);
                uint4 w = *pch;
                uint32_t* u = reinterpret_cast<uint32_t*>(&w);
#pragma unroll
                for (int m = 0; m < 4; ++m)
                    u[m] = pack_bf16(bf16lo(u[m]) * fv[2 * m], bf16hi(u[m]) * fv[2 * m + 1]);
                *pch = w;
            }
            fence_async_smem();
            mbar_arrive(&bar_a[bs]);
        }
        // the segment's total log decay (sum of Gamma over all its chunks) for the chains, if asked for
        if (dec && tid < 128 && blockIdx.y == 0 && part == P - 1) dec[unit * K + k0 + tid] = carry;
    }
    mbar_wait(&bar_free[(nb - 1) % NS], ((nb - 1) / NS) & 1);
    tc_fence_after();
    if (warp < 8) {   // epilogue: warp w reads lanes 32 (w % 4) + [0, 32) (channels), columns 128 (w / 4) + [0, 128)
        const int kr = 32 * (warp & 3) + lane, cb = 128 * (warp >> 2);
        float* out = S_loc + ((unit * P + part) * K + k0 + kr) * (size_t)V + v0 + cb;
        const uint32_t lb = (uint32_t)(32 * (warp & 3)) << 16;
#pragma unroll 1
        for (int q = 0; q < 4; ++q) {
            uint32_t r[32];
            tmem_ld32(tD + lb + cb + 32 * q, r);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 8; ++u)
                reinterpret_cast<float4*>(out + 32 * q)[u] =
                    make_float4(__uint_as_float(r[4 * u]), __uint_as_float(r[4 * u + 1]),
                                __uint_as_float(r[4 * u + 2]), __uint_as_float(r[4 * u + 3]));
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tD, 256);
}

bool seg_summary_ok(int K, int V) { return K % 128 == 0 && V % 256 == 0 && !getenv("GLA_SUMMARY_WALK"); }

cudaError_t seg_summary(const CUtensorMap& mB, const CUtensorMap& mA, const float* stats, const int* flags, float* out,
                        int K, int V, int Tv, int S, int units, bool adj, cudaStream_t st, bool skip_edge, int parts,
                        float* dec) {
    cudaError_t e;
    const int skip = (skip_edge && S > 1) ? 1 : 0;
    const dim3 grid(K / 128, V / 256, (unsigned)(units / S * (S - skip) * parts));
    if (adj) {
        if ((e = cudaFuncSetAttribute(k_seg_summary<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)SumCfg::SMEM)))
            return e;
        k_seg_summary<1><<<grid, 288, SumCfg::SMEM, st>>>(mB, mA, stats, flags, out, K, V, Tv, S, skip, parts, dec);
    } else {
        if ((e = cudaFuncSetAttribute(k_seg_summary<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)SumCfg::SMEM)))
            return e;
        k_seg_summary<0><<<grid, 288, SumCfg::SMEM, st>>>(mB, mA, stats, flags, out, K, V, Tv, S, skip, parts, dec);
    }
    return cudaGetLastError();
}

static size_t al(size_t x) { return (x + 1023) & ~size_t(1023); }

static size_t n_anch(int T) { const int NC = T / CH; return NC > 1 ? (size_t)(NC - 1) / ANCH : 0; }

size_t fwd2_ws(int B, int H, int T, int K, int V) {
    const size_t BH = (size_t)B * H, NC = T / CH;
    const int S = fwd_segments((int)BH, V, (int)NC);
    return al(BH * T * K * 2) * 2 + al(BH * T * 64 * 2) + al(BH * NC * 2 * K * 4) + al(BH * NC * 4) +
           al(n_anch(T) * BH * V * K * 2) +
           (S > 1 ? al(BH * S * K * V * 4) + al(BH * S * K * V * 4 * seg_parts((int)BH, K, V, (int)NC, S)) +
                        al(BH * S * K * 4) : 0);
}

FwdSaved fwd2_saved(const void* ws, int B, int H, int T, int K, int V) {
    const size_t BH = (size_t)B * H, NC = T / CH, rows = BH * T;
    const uint8_t* w = (const uint8_t*)ws;
    FwdSaved f;
    f.Qt = w; w += al(rows * K * 2);
    f.Kt = w; w += al(rows * K * 2);
    f.Pm = w; w += al(rows * 64 * 2);
    f.stats = (const float*)w; w += al(BH * NC * 2 * K * 4);
    f.flags = (const int*)w; w += al(BH * NC * 4);
    f.anch = w; w += al(n_anch(T) * BH * V * K * 2);
    f.S = fwd_segments((int)BH, V, (int)NC);
    f.h0v = f.S > 1 ? (const float*)w : nullptr;
    return f;
}

template <int K, typename TG>
static cudaError_t launch_fwd2(const Problem& p, cudaStream_t st) {
    const size_t BH = (size_t)p.B * p.H, NC = p.T / CH, rows = BH * p.T;
    uint8_t* w = (uint8_t*)p.ws;
    __nv_bfloat16* Qt = (__nv_bfloat16*)w; w += al(rows * K * 2);
    __nv_bfloat16* Kt = (__nv_bfloat16*)w; w += al(rows * K * 2);
    __nv_bfloat16* Pm = (__nv_bfloat16*)w; w += al(rows * 64 * 2);
    float* stats = (float*)w; w += al(BH * NC * 2 * K * 4);
    int* flags = (int*)w; w += al(BH * NC * 4);
    __nv_bfloat16* anch = (__nv_bfloat16*)w; w += al(n_anch(p.T) * BH * p.V * K * 2);
    const int S = fwd_segments((int)BH, p.V, (int)NC);
    float* h0v = (float*)w; w += S > 1 ? al(BH * S * K * p.V * 4) : 0;   // segment-entry states (saved for bwd)
    float* slv = (float*)w;                                              // segment summaries / final states
    const int SP = S > 1 && seg_summary_ok(K, p.V) ? seg_parts((int)BH, K, p.V, (int)NC, S) : 1;
    w += S > 1 ? al(BH * S * K * p.V * 4 * seg_parts((int)BH, K, p.V, (int)NC, S)) : 0;
    float* dec = S > 1 && seg_summary_ok(K, p.V) ? (float*)w : nullptr;  // per-segment log decays (summaries)
    CUtensorMap mQ, mK, mP, mV, mO, mA;
    cudaError_t e;
    if ((e = make_map_2d(&mQ, Qt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mK, Kt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mP, Pm, rows, 64, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mV, p.v, rows, p.V, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mO, p.out, rows, p.V, false)) != cudaSuccess) return e;
    const size_t n_arows = n_anch(p.T) * BH * p.V;   // anchor states [(anchor, b,h, v)][K] bf16
    if ((e = make_map_2d_ex(&mA, n_arows ? (const void*)anch : (const void*)Qt, 2, n_arows ? n_arows : rows, K, 64, 128,
                            true)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k_fwd_prep<K, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)PrepCfg<K>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_fwd_state<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)StateCfg<K>::SMEM)))
        return e;
    {
        GLA_PROF("tc::fwd_prep", st);
        const int nitems = (int)(NC * BH);
        k_fwd_prep<K, TG><<<(unsigned)(nitems < num_sms() ? nitems : num_sms()), NTH, PrepCfg<K>::SMEM, st>>>(
            mQ, mK, mP, (const __nv_bfloat16*)p.q, (const __nv_bfloat16*)p.k, (const TG*)p.g, stats, flags, p.T,
            (int)NC, nitems);
    }
    __nv_bfloat16* an = saved_anchors() ? anch : nullptr;
    if (S == 1) {
        GLA_PROF("tc::fwd_state", st);
        k_fwd_state<K><<<dim3(p.V / VT, (unsigned)BH), StateCfg<K>::NTHR, StateCfg<K>::SMEM, st>>>(
            mQ, mK, mP, mV, mO, mA, stats, flags, p.h0, p.final_state, an, p.T, p.V, 1);
        return cudaGetLastError();
    }
    // Long sequences: B*H*S virtual units of T/S tokens (same rows).  (1) state-only walks give each segment's
    // end state from a zero start, (2) the chain turns them into every segment's entry state, (3) the full walks
    // run all segments in parallel from those states (P:516-518's two-stage scan, inside one GPU).
    const int Tv = p.T / S;
    const dim3 gv(p.V / VT, (unsigned)(BH * S));
    if (seg_summary_ok(K, p.V)) {
        // chunk-parallel summaries: one tensor-core contraction per (channel tile, value tile, segment)
        GLA_PROF("tc::fwd_state_summary", st);
        if ((e = seg_summary(mV, mK, stats, flags, slv, K, p.V, Tv, S, (int)(BH * S), false, st, true, SP, dec)) !=
            cudaSuccess)
            return e;
    } else {
        GLA_PROF("tc::fwd_state_summary", st);
        k_fwd_state<K><<<gv, StateCfg<K>::NTHR, StateCfg<K>::SMEM, st>>>(mQ, mK, mP, mV, mO, mA, stats, flags, nullptr,
                                                                         slv, nullptr, Tv, p.V, 0);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = seg_chain_fwd(stats, p.h0, slv, h0v, (int)BH, S, (int)NC, K, p.V, st, SP, dec)) != cudaSuccess) return e;
    {
        GLA_PROF("tc::fwd_state", st);
        k_fwd_state<K><<<gv, StateCfg<K>::NTHR, StateCfg<K>::SMEM, st>>>(mQ, mK, mP, mV, mO, mA, stats, flags, h0v,
                                                                         p.final_state ? slv : nullptr, an, Tv, p.V, 1);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (p.final_state) {   // the last segment's end state of every (b,h)
        const size_t KV = (size_t)K * p.V;
        if ((e = cudaMemcpy2DAsync(p.final_state, KV * 4, slv + (S - 1) * KV, S * KV * 4, KV * 4, BH,
                                   cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
            return e;
    }
    return cudaGetLastError();
}

// Standalone segment summaries (gla_state_summary / gla_dstate_summary on the TC path, the per-rank step of the
// sequence-parallel scan): the prep kernel forms the chunk statistics and the factorised operands
// (K~hi, Q~hi) once, then one k_seg_summary contraction per (b,h) unit (a single segment) gives
//   adj = false: S_loc = sum_t (k_t (.) e^{LA_T - LA_t})^T v_t     and log_decay = LA_T (sum of the chunk totals)
//   adj = true : dh_loc = sum_t (q_t (.) e^{LA_t})^T dO_t
// The prep's other outputs (P, the exact-path cumsums) are written to the workspace and not used.
__global__ void k_sum_gamma(const float* __restrict__ stats, float* __restrict__ log_decay, int BH, int NC, int K) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= BH * K) return;
    const int bh = i / K, m = i % K;
    float d = 0.f;
    for (int c = 0; c < NC; ++c) d += stats[((size_t)bh * NC + c) * 2 * K + K + m];
    log_decay[i] = d;
}

template <int K, typename TG>
static cudaError_t launch_summary(const Problem& p, const void* B_op, float* out, float* log_decay, bool adj,
                                  cudaStream_t st) {
    const size_t BH = (size_t)p.B * p.H, NC = p.T / CH, rows = BH * p.T;
    uint8_t* w = (uint8_t*)p.ws;
    __nv_bfloat16* Qt = (__nv_bfloat16*)w; w += al(rows * K * 2);
    __nv_bfloat16* Kt = (__nv_bfloat16*)w; w += al(rows * K * 2);
    __nv_bfloat16* Pm = (__nv_bfloat16*)w; w += al(rows * 64 * 2);
    float* stats = (float*)w; w += al(BH * NC * 2 * K * 4);
    int* flags = (int*)w;
    CUtensorMap mQ, mK, mP, mB;
    cudaError_t e;
    if ((e = make_map_2d(&mQ, Qt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mK, Kt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mP, Pm, rows, 64, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mB, B_op, rows, p.V, true)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_fwd_prep<K, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)PrepCfg<K>::SMEM)))
        return e;
    {
        GLA_PROF("tc::fwd_prep", st);
        const int nitems = (int)(NC * BH);
        k_fwd_prep<K, TG><<<(unsigned)(nitems < num_sms() ? nitems : num_sms()), NTH, PrepCfg<K>::SMEM, st>>>(
            mQ, mK, mP, (const __nv_bfloat16*)p.q, (const __nv_bfloat16*)p.k, (const TG*)p.g, stats, flags, p.T,
            (int)NC, nitems);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    {
        GLA_PROF(adj ? "tc::dstate_summary" : "tc::state_summary", st);
        if ((e = seg_summary(mB, adj ? mQ : mK, stats, flags, out, K, p.V, p.T, 1, (int)BH, adj, st)) != cudaSuccess)
            return e;
    }
    if (!adj && log_decay) {
        const int n = (int)(BH * K);
        k_sum_gamma<<<(n + 255) / 256, 256, 0, st>>>(stats, log_decay, (int)BH, (int)NC, K);
    }
    return cudaGetLastError();
}

bool summary_tc_ok(int K, int V) { return (K == 128 || K == 256) && seg_summary_ok(K, V); }

cudaError_t summary_tc(const Problem& p, const void* B_op, float* out, float* log_decay, bool adj, cudaStream_t st) {
    const bool gf = p.gate_dtype == 1;
    switch (p.K) {
        case 128: return gf ? launch_summary<128, float>(p, B_op, out, log_decay, adj, st)
                            : launch_summary<128, __nv_bfloat16>(p, B_op, out, log_decay, adj, st);
        case 256: return gf ? launch_summary<256, float>(p, B_op, out, log_decay, adj, st)
                            : launch_summary<256, __nv_bfloat16>(p, B_op, out, log_decay, adj, st);
        default: return cudaErrorNotSupported;
    }
}

cudaError_t fwd2_tc(const Problem& p, cudaStream_t st) {
    const bool gf = p.gate_dtype == 1;
    switch (p.K) {
        case 64: return gf ? launch_fwd2<64, float>(p, st) : launch_fwd2<64, __nv_bfloat16>(p, st);
        case 128: return gf ? launch_fwd2<128, float>(p, st) : launch_fwd2<128, __nv_bfloat16>(p, st);
        case 256: return gf ? launch_fwd2<256, float>(p, st) : launch_fwd2<256, __nv_bfloat16>(p, st);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace tc
}  // namespace gla

// ---------------------------------------------------------------------------------------------------------------
// Segment state chains (see tc.h).  One thread per (b,h, k, 4 v): the S-step chain is sequential, every element
// independent; D_s is re-summed per thread from the statistics (S x NC/S floats, L2-resident).
namespace gla {
namespace tc {
namespace {
constexpr int SEG_CH = 64;
// Sum of Gamma over segment s for channel k, by the whole warp (its 32 lanes share (bh, k): V/4 is a multiple
// of 32): lane-strided partial sums, then a butterfly (every lane gets the same, fixed-order result).
__device__ __forceinline__ float seg_decay(const float* stats, int bh, int s, int NCs, int NC, int K, int k) {
    const int lane = threadIdx.x & 31;
    float d = 0.f;
    for (int c = s * NCs + lane; c < (s + 1) * NCs; c += 32) d += stats[((size_t)bh * NC + c) * 2 * K + K + k];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    return d;
}
__global__ void k_seg_chain_fwd(const float* __restrict__ stats, const float* __restrict__ h0,
                                const float* __restrict__ S_loc, float* __restrict__ Hv, int BH, int S, int NC, int K,
                                int V, int P, const float* __restrict__ dec) {
    const size_t n = (size_t)BH * K * (V / 4);
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    const int bh = (int)(idx / ((size_t)K * (V / 4)));
    const size_t rem = idx % ((size_t)K * (V / 4));
    const int k = (int)(rem / (V / 4)), v = 4 * (int)(rem % (V / 4));
    const size_t KV = (size_t)K * V, off = (size_t)k * V + v;
    float4 H = h0 ? *reinterpret_cast<const float4*>(h0 + bh * KV + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    const int NCs = NC / S;
    // groups of 4 segments: the group's summaries and decays are loaded first (independent loads in flight), then
    // the chain steps through them
    for (int s0 = 0; s0 < S; s0 += 4) {
        float4 L[4];
        float A[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int s = s0 + u;
            if (s + 1 < S) {
                A[u] = __expf(dec ? dec[((size_t)bh * S + s) * K + k] : seg_decay(stats, bh, s, NCs, NC, K, k));
                L[u] = *reinterpret_cast<const float4*>(S_loc + ((size_t)bh * S + s) * P * KV + off);
                for (int pp = 1; pp < P; ++pp) {   // the summary's token-range partials, in part order
                    const float4 m = *reinterpret_cast<const float4*>(S_loc + (((size_t)bh * S + s) * P + pp) * KV + off);
                    L[u] = make_float4(L[u].x + m.x, L[u].y + m.y, L[u].z + m.z, L[u].w + m.w);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int s = s0 + u;
            if (s < S) *reinterpret_cast<float4*>(Hv + ((size_t)bh * S + s) * KV + off) = H;
            if (s + 1 < S)
                H = make_float4(A[u] * H.x + L[u].x, A[u] * H.y + L[u].y, A[u] * H.z + L[u].z, A[u] * H.w + L[u].w);
        }
    }
}
__global__ void k_seg_chain_bwd(const float* __restrict__ stats, const float* __restrict__ dfinal,
                                const float* __restrict__ dh_loc, float* __restrict__ dFv, int BH, int S, int NC, int K,
                                int V, int P, const float* __restrict__ dec) {
    const size_t n = (size_t)BH * K * (V / 4);
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n) return;
    const int bh = (int)(idx / ((size_t)K * (V / 4)));
    const size_t rem = idx % ((size_t)K * (V / 4));
    const int k = (int)(rem / (V / 4)), v = 4 * (int)(rem % (V / 4));
    const size_t KV = (size_t)K * V, off = (size_t)k * V + v;
    float4 F = dfinal ? *reinterpret_cast<const float4*>(dfinal + bh * KV + off) : make_float4(0.f, 0.f, 0.f, 0.f);
    const int NCs = NC / S;
    for (int s0 = S - 1; s0 >= 0; s0 -= 4) {   // groups of 4 segments, loads first (see k_seg_chain_fwd)
        float4 L[4];
        float A[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int s = s0 - u;
            if (s > 0) {
                A[u] = __expf(dec ? dec[((size_t)bh * S + s) * K + k] : seg_decay(stats, bh, s, NCs, NC, K, k));
                L[u] = *reinterpret_cast<const float4*>(dh_loc + ((size_t)bh * S + s) * P * KV + off);
                for (int pp = 1; pp < P; ++pp) {
                    const float4 m = *reinterpret_cast<const float4*>(dh_loc + (((size_t)bh * S + s) * P + pp) * KV + off);
                    L[u] = make_float4(L[u].x + m.x, L[u].y + m.y, L[u].z + m.z, L[u].w + m.w);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int s = s0 - u;
            if (s >= 0) *reinterpret_cast<float4*>(dFv + ((size_t)bh * S + s) * KV + off) = F;
            if (s > 0)
                F = make_float4(A[u] * F.x + L[u].x, A[u] * F.y + L[u].y, A[u] * F.z + L[u].z, A[u] * F.w + L[u].w);
        }
    }
}
}  // namespace

cudaError_t seg_chain_fwd(const float* stats, const float* h0, const float* S_loc, float* Hv, int BH, int S, int NC,
                          int K, int V, cudaStream_t st, int parts, const float* dec) {
    const size_t n = (size_t)BH * K * (V / 4);
    GLA_PROF("tc::seg_chain", st);
    k_seg_chain_fwd<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stats, h0, S_loc, Hv, BH, S, NC, K, V, parts, dec);
    return cudaGetLastError();
}
cudaError_t seg_chain_bwd(const float* stats, const float* dfinal, const float* dh_loc, float* dFv, int BH, int S,
                          int NC, int K, int V, cudaStream_t st, int parts, const float* dec) {
    const size_t n = (size_t)BH * K * (V / 4);
    GLA_PROF("tc::seg_chain", st);
    k_seg_chain_bwd<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(stats, dfinal, dh_loc, dFv, BH, S, NC, K, V, parts,
                                                                 dec);
    return cudaGetLastError();
}
}  // namespace tc
}  // namespace gla
