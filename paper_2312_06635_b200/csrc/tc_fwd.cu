// tc_fwd.cu -- fused chunk-wise GLA forward on sm_100a tensor cores (tcgen05 + TMEM + TMA).
//
// One CTA = one (b,h) unit x one 128-wide V tile; it walks the T/64 chunks in order, keeping the state in
// TMEM for the whole sequence (never in HBM, unlike the paper's materialised chunk states).
// Per chunk i (C = 64 tokens), PAPER.md P:245-284 with SURVEY App. A.1/A.2 equations:
//   (1) b = chunk-local inclusive cumsum of log alpha, per channel, from registers
//   (2) cross-chunk output  O^T  = (H_i e^{r})^T (Q (.) e^{b-r})^T          (first term)
//       state passing       Y   += V^T (K (.) e^{r-b}) ;  H_{i+1} = e^{Gamma - r} (.) Y
//   (3) intra-chunk scores  P    = (Q (.) e^{b-r}) (K (.) e^{r-b})^T (.) M   and  O^T += V^T P^T
// where r = b at the chunk's middle row (a per-channel normaliser, every factor within e^{+-G}).
// Precision: Q~, K~ are formed in fp32 from log-space differences and split into bf16 hi + lo; P is one
// M=128 x N=128 tcgen05 MMA of [Q~hi; Q~lo] x [K~hi; K~lo]^T whose four 64x64 blocks sum to Q~ K~^T at
// ~2^-16 relative precision, so the diagonal sub-chunk blocks get the paper's "full precision"
// at the same tensor-core cost a diagonal-only correction would have.  O_inter and the state update use
// the bf16 hi parts with fp32 accumulation (the paper's half-precision matmuls).
// Guard: if a chunk's half-chunk log decay exceeds G = 60 in any channel, that chunk takes the exact path:
// P in fp32 log space on CUDA cores (per-element exponent b_t - b_s <= 0), Q~ = q e^{b}, K^ = k e^{Gamma-b}
// (all factors <= 1) and the state decay applied before the update.
//
// Thread roles (256 threads): every thread builds operands for 2 channels x 64/RG rows; all 8 warps run the
// TMEM passes (warp w -> TMEM lanes 32(w%4).., column half w/4); thread 0 issues TMA and tcgen05.mma.
#include <cuda.h>
#include <cstdio>
#include <cuda_bf16.h>

#include "common.cuh"
#include "prof.h"
#include "tc.h"
#include "tc_build.cuh"
#include "tc_common.cuh"

namespace gla {
namespace tc {

constexpr int CH = 64;          // chunk length C
constexpr int VT = 128;         // V tile per CTA (TMEM lanes)
constexpr int NTH = 256;
constexpr float L2E = 1.4426950408889634f;
constexpr float GUARD = 60.f;   // max half-chunk |log decay| for the factorised fast path

template <int K>
struct FwdCfg {
    static constexpr int RG = Tile<K>::RG;          // row groups of the operand build (tc_build.cuh)
    static constexpr int KB = K / 64;               // 64-channel blocks
    static constexpr uint32_t QT_BYTES = KB * 16384;  // [KB][128 rows: hi 0-63, lo 64-127][128 B]
    static constexpr uint32_t SB_BYTES = KB * 16384;  // [KB][128 rows v][128 B]
    static constexpr uint32_t OFF_QT = 0;
    static constexpr uint32_t OFF_KB = OFF_QT + QT_BYTES;
    static constexpr uint32_t OFF_SB = OFF_KB + QT_BYTES;
    static constexpr uint32_t OFF_V = OFF_SB + SB_BYTES;       // [2 boxes][64 t][128 B]
    static constexpr uint32_t OFF_P = OFF_V + 16384;           // [64 t][128 B]
    static constexpr uint32_t OFF_STG = K >= 128 ? OFF_SB + 16384 : OFF_P + 8192;   // O staging [2][64 t][128 B]
    static constexpr uint32_t OFF_F = K >= 128 ? OFF_P + 8192 : OFF_STG + 16384;     // fsb, fy, pend
    static constexpr uint32_t SMEM = OFF_F + 4 * 3 * K + 1024;
    static_assert(RG * K * 4 <= 8192, "gtot aliases the 8 KB P buffer");
    static_assert(SMEM <= 232448, "dynamic shared memory");
    static constexpr uint32_t TCOLS = 512;
    static constexpr uint32_t COL_S = 0, COL_O = K, COL_P = 2 * K >= 256 ? 384 : 2 * K;  // P needs 128 cols
};

template <int K, typename TG>
__global__ void __launch_bounds__(NTH, 1)
k_fwd(const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
      const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, const TG* __restrict__ g,
      const float* __restrict__ h0, float* __restrict__ final_state, float* __restrict__ ws, int T, int V) {
    using Cfg = FwdCfg<K>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    uint8_t* sQT = sm + Cfg::OFF_QT;
    uint8_t* sKB = sm + Cfg::OFF_KB;
    uint8_t* sSB = sm + Cfg::OFF_SB;
    uint8_t* sV = sm + Cfg::OFF_V;
    uint8_t* sP = sm + Cfg::OFF_P;
    float* fsb = reinterpret_cast<float*>(sm + Cfg::OFF_F);
    float* fy = fsb + K;
    float* pend = fy + K;
    float* gtot = reinterpret_cast<float*>(sP);   // [RG][K] cumsum exchange; aliases P (free at chunk start)
    __shared__ uint64_t bar_v, bar_p, bar_m1, bar_m2;
    __shared__ uint32_t tmem_base;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vtile = blockIdx.x, bh = blockIdx.y;
    const int v0 = vtile * VT;
    const int NC = T / CH;
    const int oc = tid % Tile<K>::NOCT, rg = tid / Tile<K>::NOCT;
    const int ch0 = 8 * oc;                       // this thread's channels [ch0, ch0 + 8)
    const int row0 = rg * Tile<K>::RPG;

    if (warp == 0) tmem_alloc(&tmem_base, Cfg::TCOLS);
    if (tid == 0) {
        mbar_init(&bar_v, 1);
        mbar_init(&bar_p, 1);
        mbar_init(&bar_m1, 1);
        mbar_init(&bar_m2, 1);
        fence_mbar_init();
        prefetch_tmap(&tmV);
        prefetch_tmap(&tmO);
    }
    for (int m = tid; m < K; m += NTH) pend[m] = 0.f;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tm = tmem_base;
    const uint32_t tS = tm + Cfg::COL_S, tO = tm + Cfg::COL_O, tP = tm + Cfg::COL_P;
    const int lq = warp & 3, half = warp >> 2;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int vrow = 32 * lq + lane;              // v index (TMEM lane) of this thread in TMEM passes

    // ---- initial state Y_0 = h0 (or 0) into TMEM columns [0, K) ----
    for (int c0 = half * (K / 2); c0 < (half + 1) * (K / 2); c0 += 32) {
        uint32_t r[32];
#pragma unroll
        for (int j = 0; j < 32; ++j)
            r[j] = __float_as_uint(h0 ? h0[((size_t)bh * K + c0 + j) * V + v0 + vrow] : 0.f);
        tmem_st32(tS + lane_base + c0, r);
    }
    tmem_wait_st();

    // ---- register prefetch of q, k, g for chunk 0 ----
    const size_t head_row = (size_t)bh * T;
    ChunkRegs<K> R;
    load_chunk<K, TG, true, true>(R, q, k, g, head_row, row0, ch0);

    const uint32_t idO = idesc_bf16(128, 64, 0, 0);      // O^T[v][t]: A = SB (K-major), B = Q~hi (K-major)
    const uint32_t idP = idesc_bf16(128, 128, 0, 0);     // P blocks: A = Q~ hi|lo, B = K~ hi|lo
    const uint32_t idS = idesc_bf16(128, K, 1, 1);       // Y[v][ch]: A = V^T (MN-major), B = K~hi (MN-major)
    const uint32_t idPV = idesc_bf16(128, 64, 1, 0);     // O^T += V^T P^T: A = V (MN), B = P (K-major)
    const uint32_t aQT = smem_u32(sQT), aKB = smem_u32(sKB), aSB = smem_u32(sSB), aV = smem_u32(sV),
                   aP = smem_u32(sP);

#ifdef GLA_PHASE_TIMING
    long long tph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
#define PHASE(n) do { long long _t = clock64(); tph[n] += _t - tlast; tlast = _t; } while (0)
#else
#define PHASE(n) do {} while (0)
#endif
    for (int i = 0; i < NC; ++i) {
        const uint32_t ph = i & 1;
        const int trow = (int)(head_row + (size_t)i * CH);
        if (tid == 0) {   // (TMA) V_i -> smem, two [64 t x 64 v] SW128 boxes
            mbar_expect_tx(&bar_v, 16384);
            tma_load_2d(sV, &tmV, &bar_v, v0, trow);
            tma_load_2d(sV + 8192, &tmV, &bar_v, v0 + 64, trow);
        }
        // ---- (1) chunk-local cumsum; r = b at row 31, Gamma = b at row 63 ----
        float2 off[4], rr[4], Gm[4];
        chunk_cumsum<K>(R, gtot, rg, ch0, off, rr, Gm);
        bool bad_here = false;
        if (rg == 0)   // guard: both half-chunk decays within GUARD for every channel
#pragma unroll
            for (int p = 0; p < 4; ++p)
                bad_here |= (-rr[p].x > GUARD) | (-rr[p].y > GUARD) | (rr[p].x - Gm[p].x > GUARD) |
                            (rr[p].y - Gm[p].y > GUARD);
        const bool slow = __syncthreads_or(bad_here) != 0;
        PHASE(0);
        // ---- factor references: Q~ = q e^{b - rq}, K~ = k e^{rk - b} ----
        float2 refq[4], refk[4];
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            const float2 rq = slow ? make_float2(0.f, 0.f) : rr[p], rk = slow ? Gm[p] : rr[p];
            refq[p] = make_float2(-L2E * rq.x, -L2E * rq.y);
            refk[p] = make_float2(L2E * rk.x, L2E * rk.y);
        }
        if (rg == 0) {   // TMEM-pass factors + pending exponent (one owner per channel)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int m = ch0 + u;
                const float p = pend[m];
                const float r_ = (u & 1) ? rr[u >> 1].y : rr[u >> 1].x, G_ = (u & 1) ? Gm[u >> 1].y : Gm[u >> 1].x;
                if (!slow) { fsb[m] = ex2f((p + r_) * L2E); fy[m] = fsb[m]; pend[m] = G_ - r_; }
                else { fsb[m] = ex2f(p * L2E); fy[m] = ex2f((p + G_) * L2E); pend[m] = 0.f; }
            }
        }
        const int blk = ch0 >> 6, col = ch0 & 63;
        uint8_t* qbase = sQT + blk * 16384;
        uint8_t* kbase = sKB + blk * 16384;
#pragma unroll
        for (int r = 0; r < Tile<K>::RPG; ++r) {
            const int t = row0 + r;
            float2 b[4];
#pragma unroll
            for (int p = 0; p < 4; ++p) b[p] = add2(R.g[r][p], off[p]);
            scaled_row(R.q[r], b, refq, 1.f, qbase + sw128_off(t, col), qbase + sw128_off(64 + t, col));
            scaled_row(R.k[r], b, refk, -1.f, kbase + sw128_off(t, col), kbase + sw128_off(64 + t, col));
            if (slow) {   // exact path needs b in fp32
                float4* wb = reinterpret_cast<float4*>(ws + ((size_t)(blockIdx.y * gridDim.x + blockIdx.x) * CH + t) * K + ch0);
                wb[0] = make_float4(b[0].x, b[0].y, b[1].x, b[1].y);
                wb[1] = make_float4(b[2].x, b[2].y, b[3].x, b[3].y);
            }
        }
        PHASE(1);
        if (i + 1 < NC) load_chunk<K, TG, true, true>(R, q, k, g, head_row + (size_t)(i + 1) * CH, row0, ch0);
        if (tid == 0 && i > 0) tma_store_wait_read();   // O staging (in SB) of chunk i-1 consumed
        __syncthreads();
        PHASE(2);
        // ---- TMEM pass: SB = bf16(Y * e^{sb}), Y <- Y * e^{y} ----
        state_pass2<K>(tS, lane_base, half, vrow, fsb, fy, sSB);
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        PHASE(3);
        // ---- (2)+(3) MMAs ----
        if (tid == 0) {   // P first: its epilogue overlaps the O_inter / state MMAs
            tc_fence_after();
            if (!slow) {
#pragma unroll
                for (int kk = 0; kk < K / 16; ++kk) {
                    const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
                    mma_bf16(tP, sdesc_sw128(aQT + o, 16, 1024), sdesc_sw128(aKB + o, 16, 1024), idP, kk > 0);
                }
            }
            mma_commit(&bar_p);
#pragma unroll
            for (int kk = 0; kk < K / 16; ++kk) {
                const uint32_t o = (kk >> 2) * 16384 + (kk & 3) * 32;
                mma_bf16(tO, sdesc_sw128(aSB + o, 16, 1024), sdesc_sw128(aQT + o, 16, 1024), idO, kk > 0);
            }
            mbar_wait(&bar_v, ph);
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk)
                mma_bf16(tS, sdesc_sw128(aV + kk * 2048, 8192, 1024), sdesc_sw128(aKB + kk * 2048, 16384, 1024),
                         idS, 1);
            mma_commit(&bar_m1);
        }
        mbar_wait(&bar_p, ph);
        tc_fence_after();
        PHASE(4);
        // ---- P epilogue: P (bf16, causal) -> smem [t][s] ----
        if (!slow) {
            // fp32 exchange [64 t][64 s] in the lo rows of Q~ / K~ block 0: only the finished P MMA read them
            // (the O_inter / state MMAs still in flight read the hi rows, SB and V).
            auto exch_at = [&](int t, int s) -> float* {
                uint8_t* base = (t < 32 ? sQT : sKB) + 8192 + (t & 31) * 256;
                return reinterpret_cast<float*>(base) + ((s + t) & 63);
            };
            if (lq >= 2) {
                uint32_t a[32], b[32];
                tmem_ld32(tP + lane_base + 32 * half, a);
                tmem_ld32(tP + lane_base + 64 + 32 * half, b);
                tmem_wait_ld();
                const int t = vrow - 64;
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    *exch_at(t, 32 * half + j) = __uint_as_float(a[j]) + __uint_as_float(b[j]);
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
                    const int s = 32 * half + j;
                    float p0 = __uint_as_float(a[j]) + __uint_as_float(b[j]) + *exch_at(t, s);
                    float p1 = __uint_as_float(a[j + 1]) + __uint_as_float(b[j + 1]) + *exch_at(t, s + 1);
                    p0 = s <= t ? p0 : 0.f;
                    p1 = s + 1 <= t ? p1 : 0.f;
                    pk[j / 2] = pack_bf16(p0, p1);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    *reinterpret_cast<uint4*>(sP + sw128_off(t, 32 * half + 8 * u)) =
                        make_uint4(pk[4 * u], pk[4 * u + 1], pk[4 * u + 2], pk[4 * u + 3]);
            }
        } else {
            // exact path: P[t][s] = sum_m q_tm k_sm e^{b_tm - b_sm}, s <= t, every exponent <= 0
            const float* wb = ws + (size_t)(blockIdx.y * gridDim.x + blockIdx.x) * CH * K;
            for (int e = tid; e < CH * CH; e += NTH) {
                const int t = e >> 6, s = e & 63;
                float a = 0.f;
                if (s <= t) {
                    const __nv_bfloat16* qt = q + (head_row + (size_t)i * CH + t) * K;
                    const __nv_bfloat16* ks = k + (head_row + (size_t)i * CH + s) * K;
                    for (int m = 0; m < K; ++m)
                        a += __bfloat162float(qt[m]) * __bfloat162float(ks[m]) *
                             ex2f((wb[t * K + m] - wb[s * K + m]) * L2E);
                }
                *reinterpret_cast<__nv_bfloat16*>(sP + sw128_off(t, s)) = __float2bfloat16_rn(a);
            }
        }
        fence_async_smem();
        tc_fence_before();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < CH / 16; ++kk)
                mma_bf16(tO, sdesc_sw128(aV + kk * 2048, 8192, 1024), sdesc_sw128(aP + kk * 32, 16, 1024), idPV, 1);
            mma_commit(&bar_m2);
        }
        PHASE(5);
        mbar_wait(&bar_m1, ph);
        mbar_wait(&bar_m2, ph);
        tc_fence_after();
        PHASE(6);
        // ---- O epilogue: O^T (TMEM) -> bf16 staging [box][t][64 v] -> TMA store ----
        {
            uint8_t* stg = sm + Cfg::OFF_STG;
            uint32_t r[32];
            tmem_ld32(tO + lane_base + 32 * half, r);
            tmem_wait_ld();
            uint8_t* dst = stg + (vrow >> 6) * 8192 + (vrow & 63) * 2;
#pragma unroll
            for (int j = 0; j < 32; ++j)
                *reinterpret_cast<__nv_bfloat16*>(dst + (32 * half + j) * 128) =
                    __float2bfloat16_rn(__uint_as_float(r[j]));
            fence_async_smem();
            tc_fence_before();
            __syncthreads();
            if (tid == 0) {
                tma_store_2d(&tmO, stg, v0, trow);
                tma_store_2d(&tmO, stg + 8192, v0 + 64, trow);
                tma_store_commit();
            }
        }
        PHASE(7);
    }
#ifdef GLA_PHASE_TIMING
    if ((tid == 0 || tid == 255) && blockIdx.x == 0 && blockIdx.y == 0)
        printf("tid %d phases/chunk: cumsum+guard %lld build %lld prefetch+sync %lld statepass %lld mma1 %lld pepi+issue %lld pv %lld oepi %lld\n", tid,
               tph[0] / NC, tph[1] / NC, tph[2] / NC, tph[3] / NC, tph[4] / NC, tph[5] / NC, tph[6] / NC, tph[7] / NC);
#endif
    // ---- final state: H_T = Y (.) e^{pend} ----
    if (final_state) {
        for (int c0 = half * (K / 2); c0 < (half + 1) * (K / 2); c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tS + lane_base + c0, r);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j)
                final_state[((size_t)bh * K + c0 + j) * V + v0 + vrow] =
                    __uint_as_float(r[j]) * ex2f(pend[c0 + j] * L2E);
        }
    }
    if (tid == 0) tma_store_wait_all();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tm, Cfg::TCOLS);
}

// ---------------------------------------------------------------------------------------------------------------
typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encoder() {
    static EncodeFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess)
            fn = (EncodeFn)p;
    }
    return fn;
}

// 2-D bf16 map over a [rows][cols] row-major tensor with a {64 cols, 64 rows} box.
cudaError_t make_map_2d_ex(CUtensorMap* map, const void* base, int elem_bytes, uint64_t rows, uint64_t cols,
                           uint32_t box_cols, uint32_t box_rows, bool swizzle) {
    EncodeFn fn = encoder();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * (uint64_t)elem_bytes};
    cuuint32_t box[2] = {box_cols, box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, elem_bytes == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                    const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

cudaError_t make_map_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, bool swizzle) {
    EncodeFn fn = encoder();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {cols * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int K, typename TG>
static cudaError_t launch_fwd(const Problem& p, cudaStream_t st) {
    CUtensorMap mV, mO;
    const uint64_t rows = (uint64_t)p.B * p.H * p.T;
    cudaError_t e = make_map_2d(&mV, p.v, rows, p.V, true);
    if (e != cudaSuccess) return e;
    e = make_map_2d(&mO, p.out, rows, p.V, false);
    if (e != cudaSuccess) return e;
    const uint32_t smem = FwdCfg<K>::SMEM;
    e = cudaFuncSetAttribute(k_fwd<K, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grid(p.V / VT, p.B * p.H);
    {
        GLA_PROF("tc::fwd", st);
        k_fwd<K, TG><<<grid, NTH, smem, st>>>(mV, mO, (const __nv_bfloat16*)p.q, (const __nv_bfloat16*)p.k,
                                              (const TG*)p.g, p.h0, p.final_state, (float*)p.ws, p.T, p.V);
    }
    return cudaGetLastError();
}

cudaError_t fwd_tc(const Problem& p, cudaStream_t st) {
    const bool gf = p.gate_dtype == 1;
    switch (p.K) {
        case 64: return gf ? launch_fwd<64, float>(p, st) : launch_fwd<64, __nv_bfloat16>(p, st);
        case 128: return gf ? launch_fwd<128, float>(p, st) : launch_fwd<128, __nv_bfloat16>(p, st);
        case 256: return gf ? launch_fwd<256, float>(p, st) : launch_fwd<256, __nv_bfloat16>(p, st);
        default: return cudaErrorNotSupported;
    }
}

size_t fwd_tc_ws(int B, int H, int T, int K, int V) {
    return sizeof(float) * (size_t)B * H * (V / VT) * CH * K;   // fp32 b of the exact-path chunks
}

}  // namespace tc
}  // namespace gla
