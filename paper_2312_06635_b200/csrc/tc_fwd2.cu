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
// Compared with the single fused kernel (tc_fwd.cu), the operand construction and P run once per chunk
// instead of once per V tile (4x at d_v' = 512), at the price of writing / re-reading Q~hi, K~hi and P
// (2.1 KB per token-head at K = 256).  Exact path for chunks failing the factorisation guard: as tc_fwd.cu
// (prep computes P in fp32 log space with factors <= 1; the state kernel applies the decay before the update).
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
template <int K>
struct PrepCfg {
    using Tl = Tile<K>;
    static constexpr int KB = K / 64;
    static constexpr uint32_t OP = KB * 16384;          // [KB][128 rows: hi | lo][128 B]
    static constexpr uint32_t OFF_Q = 0, OFF_K = OP, OFF_P = 2 * OP;       // P [64 t][128 B]
    static constexpr uint32_t OFF_X = OFF_P + 8192;     // exchange [64][64] fp32 and gtot
    static constexpr uint32_t SMEM = OFF_X + 16384 + 1024;
    static_assert(Tl::RG * K * 4 <= 16384, "gtot fits the exchange buffer");
};

template <int K, typename TG>
__global__ void __launch_bounds__(NTH, 1)
k_fwd_prep(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmP, const __nv_bfloat16* __restrict__ q,
           const __nv_bfloat16* __restrict__ k, const TG* __restrict__ g, float* __restrict__ stats,
           int* __restrict__ flags, float* __restrict__ bws, int T) {
    using Cfg = PrepCfg<K>;
    using Tl = typename Cfg::Tl;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm + Cfg::OFF_Q;
    uint8_t* sK = sm + Cfg::OFF_K;
    uint8_t* sP = sm + Cfg::OFF_P;
    float* exch = reinterpret_cast<float*>(sm + Cfg::OFF_X);
    float* gtot = exch;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int chunk = blockIdx.x, bh = blockIdx.y, NC = gridDim.x;
    const int oc = tid % Tl::NOCT, rg = tid / Tl::NOCT;
    const int ch0 = 8 * oc, row0 = rg * Tl::RPG;
    const size_t crow = (size_t)bh * T + (size_t)chunk * CH;

    if (warp == 0) tmem_alloc(&tmem_base, 128);
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    ChunkRegs<K> R;
    load_chunk<K, TG, true, true>(R, q, k, g, crow, row0, ch0);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tP = tmem_base;

    float2 off[4], rr[4], Gm[4];
    chunk_cumsum<K>(R, gtot, rg, ch0, off, rr, Gm);
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
        if (slow) {
            float4* wb = reinterpret_cast<float4*>(bws + (crow + t) * K + ch0);
            wb[0] = make_float4(b[0].x, b[0].y, b[1].x, b[1].y);
            wb[1] = make_float4(b[2].x, b[2].y, b[3].x, b[3].y);
        }
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
        prefetch_tmap(&tmQ);
        for (int c = 0; c < K / 64; ++c) {
            tma_store_2d(&tmQ, sQ + c * 16384, 64 * c, (int)crow);
            tma_store_2d(&tmK, sK + c * 16384, 64 * c, (int)crow);
        }
        tma_store_commit();
    }
    const int lq = warp & 3, half = warp >> 2;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int vrow = 32 * lq + lane;
    if (!slow) {
        mbar_wait(&bar, 0);
        tc_fence_after();
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
    } else {
        // exact path: P[t][s] = sum_m q_tm k_sm e^{b_tm - b_sm}, s <= t, every exponent <= 0
        __syncthreads();
        for (int e = tid; e < CH * CH; e += NTH) {
            const int t = e >> 6, s = e & 63;
            float a = 0.f;
            if (s <= t) {
                const __nv_bfloat16* qt = q + (crow + t) * K;
                const __nv_bfloat16* ks = k + (crow + s) * K;
                const float* bt = bws + (crow + t) * K;
                const float* bs = bws + (crow + s) * K;
                for (int m = 0; m < K; ++m)
                    a += __bfloat162float(qt[m]) * __bfloat162float(ks[m]) * ex2f((bt[m] - bs[m]) * L2E);
            }
            *reinterpret_cast<__nv_bfloat16*>(sP + sw128_off(t, s)) = __float2bfloat16_rn(a);
        }
    }
    fence_async_smem();
    __syncthreads();
    if (tid == 0) {
        tma_store_2d(&tmP, sP, 0, (int)crow);
        tma_store_commit();
        tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tP, 128);
}

// ---------------------------------------------------------------------------------------------------------------
template <int K>
struct StateCfg {
    static constexpr int KB = K / 64;
    static constexpr uint32_t OP = KB * 8192;            // [KB][64 t][128 B]  Q~hi or K~hi
    static constexpr uint32_t OFF_Q = 0, OFF_K = OP, OFF_SB = 2 * OP;
    static constexpr uint32_t OFF_V = OFF_SB + KB * 16384;      // 2 buffers x [2][64 t][128 B]
    static constexpr uint32_t OFF_P = OFF_V + 2 * 16384;        // 2 buffers x [64 t][128 B]
    static constexpr uint32_t OFF_STG = OFF_P + 2 * 8192;       // O staging [2][64 t][128 B]
    static constexpr uint32_t OFF_F = OFF_STG + 16384;          // fsb, fy, pend [K]
    static constexpr uint32_t SMEM = OFF_F + 4 * 3 * K + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
    static constexpr uint32_t TCOLS = 2 * K >= 256 ? 512 : 256;
};

template <int K>
__global__ void __launch_bounds__(NTH, 1)
k_fwd_state(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmV,
            const __grid_constant__ CUtensorMap tmO, const float* __restrict__ stats, const int* __restrict__ flags,
            const float* __restrict__ h0, float* __restrict__ final_state, int T, int V) {
    using Cfg = StateCfg<K>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = sm + Cfg::OFF_Q;
    uint8_t* sK = sm + Cfg::OFF_K;
    uint8_t* sSB = sm + Cfg::OFF_SB;
    uint8_t* sV = sm + Cfg::OFF_V;
    uint8_t* sP = sm + Cfg::OFF_P;
    uint8_t* stg = sm + Cfg::OFF_STG;
    float* fsb = reinterpret_cast<float*>(sm + Cfg::OFF_F);
    float* fy = fsb + K;
    float* pend = fy + K;
    __shared__ uint64_t bar_qk, bar_vp[2], bar_m;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vt = blockIdx.x, bh = blockIdx.y;
    const int v0 = vt * VT, NC = T / CH;
    const int rowb = bh * T;

    if (warp == 0) tmem_alloc(&tmem_base, Cfg::TCOLS);
    if (tid == 0) {
        mbar_init(&bar_qk, 1);
        mbar_init(&bar_vp[0], 1);
        mbar_init(&bar_vp[1], 1);
        mbar_init(&bar_m, 1);
        fence_mbar_init();
        prefetch_tmap(&tmQ); prefetch_tmap(&tmK); prefetch_tmap(&tmP); prefetch_tmap(&tmV); prefetch_tmap(&tmO);
        // chunk 0 inputs
        mbar_expect_tx(&bar_qk, 2 * Cfg::OP);
        for (int c = 0; c < K / 64; ++c) {
            tma_load_2d(sQ + c * 8192, &tmQ, &bar_qk, 64 * c, rowb);
            tma_load_2d(sK + c * 8192, &tmK, &bar_qk, 64 * c, rowb);
        }
        mbar_expect_tx(&bar_vp[0], 16384 + 8192);
        tma_load_2d(sV, &tmV, &bar_vp[0], v0, rowb);
        tma_load_2d(sV + 8192, &tmV, &bar_vp[0], v0 + 64, rowb);
        tma_load_2d(sP, &tmP, &bar_vp[0], 0, rowb);
    }
    for (int m = tid; m < K; m += NTH) pend[m] = 0.f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    const uint32_t tS = tm, tO = tm + K;
    const int lq = warp & 3, half = warp >> 2;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int vrow = 32 * lq + lane;
    for (int c0 = half * (K / 2); c0 < (half + 1) * (K / 2); c0 += 32) {
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
            r[j] = __float_as_uint(h0 ? h0[((size_t)bh * K + c0 + j) * V + v0 + vrow] : 0.f);
        tmem_st32(tS + lane_base + c0, r);
    }
    tmem_wait_st();

    const uint32_t idO = idesc_bf16(128, 64, 0, 0);      // O^T[v][t] = SB . Q~hi^T
    const uint32_t idS = idesc_bf16(128, K, 1, 1);       // Y[v][ch] += V^T K~hi
    const uint32_t idPV = idesc_bf16(128, 64, 1, 0);     // O^T += V^T P^T
    const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aSB = smem_u32(sSB);
    // per-chunk statistics (r, Gamma) for this thread's channel, one chunk ahead
    float st_r = 0.f, st_G = 0.f;
    int st_slow = 0;
    if (tid < K) {
        st_r = stats[((size_t)bh * NC) * 2 * K + tid];
        st_G = stats[((size_t)bh * NC) * 2 * K + K + tid];
    }
    st_slow = flags[(size_t)bh * NC];

    for (int i = 0; i < NC; ++i) {
        const int buf = i & 1;
        const int trow = rowb + i * CH;
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
        if (tid == 0 && i > 0) tma_store_wait_read();   // O staging of chunk i-1 consumed (it sits after SB)
        __syncthreads();
        state_pass2<K>(tS, lane_base, half, vrow, fsb, fy, sSB);   // SB = bf16(H_i e^{r}); Y <- decayed
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            mbar_wait(&bar_qk, i & 1);
            mbar_wait(&bar_vp[buf], (i >> 1) & 1);
            tc_fence_after();
            const uint32_t aV = smem_u32(sV + buf * 16384), aP = smem_u32(sP + buf * 8192);
#pragma unroll
            for (int kk = 0; kk < K / 16; ++kk) {
                const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32, ob = (kk >> 2) * 8192 + (kk & 3) * 32;
                mma_bf16(tO, sdesc_sw128(aSB + o, 16, 1024), sdesc_sw128(aQ + ob, 16, 1024), idO, kk > 0);
            }
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk)
                mma_bf16(tO, sdesc_sw128(aV + kk * 2048, 8192, 1024), sdesc_sw128(aP + kk * 32, 16, 1024), idPV, 1);
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk)
                mma_bf16(tS, sdesc_sw128(aV + kk * 2048, 8192, 1024), sdesc_sw128(aK + kk * 2048, 8192, 1024), idS, 1);
            mma_commit(&bar_m);
            if (i + 1 < NC) {   // V, P of chunk i+1 into the other buffers (their last reader, chunk i-1, is done)
                const int nb = buf ^ 1;
                mbar_expect_tx(&bar_vp[nb], 16384 + 8192);
                tma_load_2d(sV + nb * 16384, &tmV, &bar_vp[nb], v0, trow + CH);
                tma_load_2d(sV + nb * 16384 + 8192, &tmV, &bar_vp[nb], v0 + 64, trow + CH);
                tma_load_2d(sP + nb * 8192, &tmP, &bar_vp[nb], 0, trow + CH);
            }
        }
        mbar_wait(&bar_m, i & 1);
        tc_fence_after();
        if (tid == 0 && i + 1 < NC) {   // Q~hi, K~hi of chunk i+1 (the MMAs that read them are complete)
            mbar_expect_tx(&bar_qk, 2 * Cfg::OP);
            for (int c = 0; c < K / 64; ++c) {
                tma_load_2d(sQ + c * 8192, &tmQ, &bar_qk, 64 * c, trow + CH);
                tma_load_2d(sK + c * 8192, &tmK, &bar_qk, 64 * c, trow + CH);
            }
        }
        {   // O^T (TMEM) -> bf16 staging [box][t][64 v] -> TMA store
            uint32_t r[32];
            tmem_ld32(tO + lane_base + 32 * half, r);
            tmem_wait_ld();
            uint8_t* dst = stg + (vrow >> 6) * 8192 + (vrow & 63) * 2;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                *reinterpret_cast<__nv_bfloat16*>(dst + (32 * half + j) * 128) = __float2bfloat16_rn(__uint_as_float(r[j]));
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                tma_store_2d(&tmO, stg, v0, trow);
                tma_store_2d(&tmO, stg + 8192, v0 + 64, trow);
                tma_store_commit();
            }
        }
    }
    if (final_state) {
        for (int c0 = half * (K / 2); c0 < (half + 1) * (K / 2); c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tS + lane_base + c0, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
                final_state[((size_t)bh * K + c0 + j) * V + v0 + vrow] = __uint_as_float(r[j]) * ex2f(pend[c0 + j] * L2E);
        }
    }
    if (tid == 0) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, Cfg::TCOLS);
}

// ---------------------------------------------------------------------------------------------------------------
static size_t al(size_t x) { return (x + 1023) & ~size_t(1023); }

size_t fwd2_ws(int B, int H, int T, int K, int V) {
    const size_t BH = (size_t)B * H, NC = T / CH;
    return al(BH * T * K * 2) * 2 + al(BH * T * 64 * 2) + al(BH * NC * 2 * K * 4) + al(BH * NC * 4) +
           al(BH * T * K * 4);
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
    float* bws = (float*)w;
    CUtensorMap mQ, mK, mP, mV, mO;
    cudaError_t e;
    if ((e = make_map_2d(&mQ, Qt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mK, Kt, rows, K, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mP, Pm, rows, 64, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mV, p.v, rows, p.V, true)) != cudaSuccess) return e;
    if ((e = make_map_2d(&mO, p.out, rows, p.V, false)) != cudaSuccess) return e;
    if ((e = cudaFuncSetAttribute(k_fwd_prep<K, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)PrepCfg<K>::SMEM)))
        return e;
    if ((e = cudaFuncSetAttribute(k_fwd_state<K>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)StateCfg<K>::SMEM)))
        return e;
    {
        GLA_PROF("tc::fwd_prep", st);
        k_fwd_prep<K, TG><<<dim3((unsigned)NC, (unsigned)BH), NTH, PrepCfg<K>::SMEM, st>>>(
            mQ, mK, mP, (const __nv_bfloat16*)p.q, (const __nv_bfloat16*)p.k, (const TG*)p.g, stats, flags, bws, p.T);
    }
    {
        GLA_PROF("tc::fwd_state", st);
        k_fwd_state<K><<<dim3(p.V / VT, (unsigned)BH), NTH, StateCfg<K>::SMEM, st>>>(
            mQ, mK, mP, mV, mO, stats, flags, p.h0, p.final_state, p.T, p.V);
    }
    return cudaGetLastError();
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
