// tc_kwalk.cu -- the dq walk of the backward with the key channels on the TMEM lanes ("dq walk").
//
// dq = e^{b - r} (.) [ dO (H_i e^r)^T + dP K~ ]       (the inter term contracts over the values v)
// One CTA per (unit, 128-channel group, 256-value half).  Its TMEM holds the state tile transposed,
// X[k][v] = (H_i e^{...})^T for 128 channels k (lanes) x 256 values v (columns), so
//   * the per-chunk decay of the state pass is one scalar per thread (a channel per lane);
//   * SB = bf16(H_i e^r) stays in TMEM as the A operand (K-major: k rows, v packed in pairs) of the
//     dq^T[k][t] = SB[k][v] dO^T[v][t] MMAs (TS mode): SB never touches shared memory;
//   * the state update X[k][v] += K~^T[k][s] V[s][v] is one N = 128 MMA per value half and 16-token step.
// At V = 512 the two value halves of a channel group form a 2-CTA cluster: each CTA owns 64 of the 128 channels
// of the final dq, sends its fp32 partial of the other 64 to its partner's shared memory (DSMEM) and adds the
// partner's partial to its own in fp32 (sum of two terms: order-independent, deterministic).  So dq leaves the
// walk complete and scaled (bf16), with no V-tile partials through HBM.
//   warps 0-7   state pass, one value half at a time (X half decayed in place, SB half written), signalled per half
//   warp 8      state MMA per value half (X[:, half] += K~^T V[:, half]), commits bar_sh[half]
//   warps 9, 10 dq^T = SB[:, half 0] dO^T (+ K~^T dP^T on value half 0) then += SB[:, half 1] dO^T (fixed order)
//               into a double-buffered TMEM accumulator
//   warps 11-14 epilogue: accumulator -> DSMEM exchange -> e^{b - r} scale -> dq (bf16); TMA loads two chunks ahead
// The statistics (r, Gamma per chunk and channel) come from the forward's prep kernel; b is re-summed from
// log alpha by the owning thread (one channel per thread: a sequential in-register scan over the 64 tokens).
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
constexpr float L2E = 1.4426950408889634f;

struct KwCfg {
    static constexpr uint32_t KT = 2 * 8192;                  // K~ tile [64 s][128 k]   (2 SW128 blocks)
    static constexpr uint32_t VTB = 4 * 8192;                 // V tile  [64 s][256 v]   (4 blocks)
    static constexpr uint32_t DTB = 4 * 8192;                 // dO tile [64 t][256 v]
    static constexpr uint32_t PTB = 8192;                     // dP tile [64 t][64 s]
    static constexpr uint32_t OFF_V = KT, OFF_D = KT + VTB, OFF_P = KT + VTB + DTB;
    static constexpr uint32_t STAGE = KT + VTB + DTB + PTB;
    static constexpr uint32_t RROW = 68;                      // recv row stride (floats): conflict-free v4 reads
    static constexpr uint32_t RBUF = 64 * RROW * 4;
    static constexpr uint32_t OFF_R = 2 * STAGE;              // recv [2][64 ch][RROW] fp32
    static constexpr uint32_t OFF_RED = OFF_R + 2 * RBUF;     // [2][128] fp32 (final-state row sums)
    static constexpr uint32_t SMEM = OFF_RED + 2 * 128 * 4 + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
    static constexpr int NST = 256, NTHR = NST + 96 + 128;
    static constexpr uint32_t COL_SB = 256, COL_ACC = 384;   // TMEM: X [256] | SB [128] | acc x2 [64 each]
};

__device__ __forceinline__ float ld_gate(const float* g, size_t i) { return __ldg(g + i); }
__device__ __forceinline__ float ld_gate(const __nv_bfloat16* g, size_t i) { return __bfloat162float(g[i]); }
}  // namespace

template <int K, int NVH, typename TG>
__global__ void __launch_bounds__(KwCfg::NTHR, 1)
k_bwd_dqk(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmDP,
          const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmD,
          const float* __restrict__ stats, const TG* __restrict__ g, const float* __restrict__ h0,
          const float* __restrict__ dfinal, __nv_bfloat16* __restrict__ dq, float* __restrict__ stdot,
          const int* __restrict__ flag, int T, int V) {
    using Cfg = KwCfg;
    if (*flag) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    float* recv = reinterpret_cast<float*>(sm + Cfg::OFF_R);
    float* red = reinterpret_cast<float*>(sm + Cfg::OFF_RED);
    __shared__ uint64_t bar_in[2], bar_free[2], bar_sbh[2], bar_sh[2], bar_da[2], bar_db[2], bar_efree[2];
    __shared__ uint64_t rfull[2], rempty[2];
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vh = blockIdx.x, k0 = 128 * blockIdx.y, unit = blockIdx.z;
    const int v0 = 256 * vh, NC = T / CH;
    const size_t rowb = (size_t)unit * T;
    const bool intra = vh == 0;
    const uint32_t partner = (uint32_t)(vh ^ 1);
    auto load_inputs = [&](int i) {
        const int b = i & 1, row = (int)(rowb + (size_t)i * CH);
        uint8_t* st = sm + b * Cfg::STAGE;
        mbar_expect_tx(&bar_in[b], Cfg::KT + Cfg::VTB + Cfg::DTB + (intra ? Cfg::PTB : 0));
        tma_load_2d(st, &tmK, &bar_in[b], k0, row);
        tma_load_2d(st + 8192, &tmK, &bar_in[b], k0 + 64, row);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            tma_load_2d(st + Cfg::OFF_V + j * 8192, &tmV, &bar_in[b], v0 + 64 * j, row);
            tma_load_2d(st + Cfg::OFF_D + j * 8192, &tmD, &bar_in[b], v0 + 64 * j, row);
        }
        if (intra) tma_load_2d(st + Cfg::OFF_P, &tmDP, &bar_in[b], 0, row);
    };
    if (warp == 0) tmem_alloc(&tmem_base, 512);
    if (tid == 0) {
        for (int j = 0; j < 2; ++j) {
            mbar_init(&bar_in[j], 1);
            mbar_init(&bar_free[j], 3);
            mbar_init(&bar_sbh[j], 1);
            mbar_init(&bar_sh[j], 1);
            mbar_init(&bar_da[j], 1);
            mbar_init(&bar_db[j], 1);
            mbar_init(&bar_efree[j], 1);
            mbar_init(&rfull[j], 64);
            mbar_init(&rempty[j], 64);
        }
        fence_mbar_init();
        prefetch_tmap(&tmK); prefetch_tmap(&tmV); prefetch_tmap(&tmD); prefetch_tmap(&tmDP);
        load_inputs(0);
        if (NC > 1) load_inputs(1);
    }
    tc_fence_before();
    __syncthreads();
    if (NVH == 2) cluster_sync_all();        // the partner's barriers are initialised before any remote arrive
    tc_fence_after();
    const uint32_t tX = tmem_base, tSB = tmem_base + Cfg::COL_SB, tAcc = tmem_base + Cfg::COL_ACC;
    const int lq = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int kk = 32 * lq + lane;           // channel within the group (TMEM lane)
    const int kg = k0 + kk;                  // global channel

    if (warp < 8) {
        // ------------------------------------------------------------------ state warps
        const int cs = 64 * (warp >> 2);     // this warp's 64-column share of each 128-column value half
        const float* h0r = h0 ? h0 + ((size_t)unit * K + kg) * V + v0 : nullptr;
#pragma unroll 1
        for (int c = 0; c < 256; c += 32) {
            if (((c >> 6) & 1) != (warp >> 2)) continue;
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 x = h0r ? __ldg(reinterpret_cast<const float4*>(h0r + c + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
                r[j] = __float_as_uint(x.x); r[j + 1] = __float_as_uint(x.y);
                r[j + 2] = __float_as_uint(x.z); r[j + 3] = __float_as_uint(x.w);
            }
            tmem_st32(tX + lane_base + c, r);
        }
        tmem_wait_st();
        const float* st_ch = stats + (size_t)unit * NC * 2 * K + kg;   // (r, Gamma) of chunk i at [i * 2K], [i * 2K + K]
        float pend = 0.f, n_r = st_ch[0], n_G = st_ch[K];
        named_bar_sync(1, Cfg::NST);
        for (int i = 0; i < NC; ++i) {
            const float r_ = n_r, G_ = n_G;
            if (i + 1 < NC) { n_r = st_ch[(size_t)(i + 1) * 2 * K]; n_G = st_ch[(size_t)(i + 1) * 2 * K + K]; }
            const float f = ex2f((pend + r_) * L2E);   // X <- H_i e^{r}, SB = bf16(X)
            pend = G_ - r_;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (i > 0) {                 // half h of chunk i-1: state MMA done, SB half h read by the dq MMAs
                    mbar_wait(&bar_sh[h], (i - 1) & 1);
                    mbar_wait(h == 0 ? &bar_da[(i - 1) & 1] : &bar_db[(i - 1) & 1], ((i - 1) >> 1) & 1);
                    tc_fence_after();
                }
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int c = 128 * h + cs + 32 * s;
                    uint32_t r[32], pk[16];
                    tmem_ld32(tX + lane_base + c, r);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const float2 y = mul2(make_float2(__uint_as_float(r[j]), __uint_as_float(r[j + 1])),
                                              make_float2(f, f));
                        r[j] = __float_as_uint(y.x);
                        r[j + 1] = __float_as_uint(y.y);
                        pk[j / 2] = pack2(y);
                    }
                    tmem_st32(tX + lane_base + c, r);
                    tmem_st16(tSB + lane_base + c / 2, pk);
                }
                tmem_wait_st();
                tc_fence_before();
                named_bar_sync(1, Cfg::NST);
                if (tid == 0) mbar_arrive(&bar_sbh[h]);
            }
        }
        mbar_wait(&bar_sh[0], (NC - 1) & 1);
        mbar_wait(&bar_sh[1], (NC - 1) & 1);
        tc_fence_after();
        if (dfinal) {   // rowsum over this CTA's values of S_T (.) dS_T: one partial per value half
            const float fe = ex2f(pend * L2E);
            const float* dfr = dfinal + ((size_t)unit * K + kg) * V + v0;
            float acc = 0.f;
#pragma unroll 1
            for (int c = 0; c < 256; c += 32) {
                if (((c >> 6) & 1) != (warp >> 2)) continue;
                uint32_t r[32];
                tmem_ld32(tX + lane_base + c, r);
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    const float4 d = __ldg(reinterpret_cast<const float4*>(dfr + c + j));
                    acc += __uint_as_float(r[j]) * d.x + __uint_as_float(r[j + 1]) * d.y +
                           __uint_as_float(r[j + 2]) * d.z + __uint_as_float(r[j + 3]) * d.w;
                }
            }
            red[(warp >> 2) * 128 + kk] = acc * fe;
            named_bar_sync(1, Cfg::NST);
            if (warp < 4) stdot[((size_t)vh * gridDim.z + unit) * K + kg] = red[kk] + red[128 + kk];
        }
    } else if (warp == 8) {
        // ------------------------------------------------------------------ state MMA issuer (per value half)
        const uint32_t idS = idesc_bf16(128, 128, 1, 1);   // X[k][v] += K~^T[k][s] V[s][v]: A, B MN-major
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            const uint32_t aK = smem_u32(sm + b * Cfg::STAGE), aV = aK + Cfg::OFF_V;
            for (int h = 0; h < 2; ++h) {
                mbar_wait(&bar_sbh[h], i & 1);
                if (h == 0) mbar_wait(&bar_in[b], (i >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < CH / 16; ++s)
                    mma_bf16_w(tX + 128 * h, sdesc_sw128(aK + s * 2048, 8192, 1024),
                               sdesc_sw128(aV + 2 * h * 8192 + s * 2048, 8192, 1024), idS, 1);
                mma_commit_w(&bar_sh[h]);
            }
            mma_commit_w(&bar_free[b]);
            __syncwarp();
        }
    } else if (warp < 11) {
        // ------------------------------------------------------------------ dq^T issuers (value half 0, then 1)
        const int h = warp - 9;
        const uint32_t idDQ = idesc_bf16(128, 64, 0, 0);   // dq^T[k][t] += SB[k][v] dO[t][v]: A in TMEM
        const uint32_t idIN = idesc_bf16(128, 64, 1, 0);   // dq^T[k][t] += K~^T[k][s] dP[t][s]
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            const uint32_t aK = smem_u32(sm + b * Cfg::STAGE), aD = aK + Cfg::OFF_D, adP = aK + Cfg::OFF_P;
            const uint32_t acc = tAcc + 64 * b;
            mbar_wait(&bar_sbh[h], i & 1);
            mbar_wait(&bar_in[b], (i >> 1) & 1);
            if (h == 0 && i >= 2) mbar_wait(&bar_efree[b], ((i >> 1) - 1) & 1);
            if (h == 1) mbar_wait(&bar_da[b], (i >> 1) & 1);   // accumulate after half 0 (fixed order)
            tc_fence_after();
#pragma unroll
            for (int s = 0; s < 8; ++s)
                mma_bf16_ta_w(acc, tSB + 64 * h + 8 * s,
                              sdesc_sw128(aD + (2 * h + (s >> 2)) * 8192 + (s & 3) * 32, 16, 1024), idDQ,
                              (h == 1 || s > 0) ? 1u : 0u);
            if (h == 0 && intra)
#pragma unroll
                for (int s = 0; s < CH / 16; ++s)
                    mma_bf16_w(acc, sdesc_sw128(aK + s * 2048, 8192, 1024), sdesc_sw128(adP + s * 32, 16, 1024), idIN, 1);
            mma_commit_w(h == 0 ? &bar_da[b] : &bar_db[b]);
            mma_commit_w(&bar_free[b]);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------------ epilogue warps
        const int et = tid - Cfg::NST - 96;
        const bool owner = NVH == 1 || (kk >> 6) == vh;
        const float* st_ch = stats + (size_t)unit * NC * 2 * K + kg;
        uint32_t r_recv = 0, r_full[2] = {0, 0}, r_empty[2] = {0, 0};
        if (NVH == 2) {
            // sender: my row in the partner's recv buffers; owner: the partner's rempty barriers
            r_recv = mapa_shared(recv + (kk & 63) * Cfg::RROW, partner);
            for (int j = 0; j < 2; ++j) {
                r_full[j] = mapa_shared(&rfull[j], partner);
                r_empty[j] = mapa_shared(&rempty[j], partner);
            }
        }
        for (int i = 0; i < NC; ++i) {
            const int b = i & 1;
            if (et == 0 && i + 2 < NC) {     // inputs of chunk i+2 into buffer b once chunk i's MMAs are done
                mbar_wait(&bar_free[b], (i >> 1) & 1);
                load_inputs(i + 2);
            }
            mbar_wait(&bar_db[b], (i >> 1) & 1);
            tc_fence_after();
            uint32_t a[32], a2[32];
            tmem_ld32(tAcc + 64 * b + lane_base, a);
            tmem_ld32(tAcc + 64 * b + 32 + lane_base, a2);
            tmem_wait_ld();
            tc_fence_before();
            named_bar_sync(2, 128);          // accumulator b drained
            if (et == 0) mbar_arrive(&bar_efree[b]);
            if (!owner) {                    // fp32 partial of the partner's channels -> its shared memory
                if (i >= 2) mbar_wait_cluster(&rempty[b], ((i >> 1) - 1) & 1);
                const uint32_t dst = r_recv + b * Cfg::RBUF;
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    st_cluster_v4(dst + 4 * j, make_float4(__uint_as_float(a[j]), __uint_as_float(a[j + 1]),
                                                           __uint_as_float(a[j + 2]), __uint_as_float(a[j + 3])));
                    st_cluster_v4(dst + 128 + 4 * j, make_float4(__uint_as_float(a2[j]), __uint_as_float(a2[j + 1]),
                                                                 __uint_as_float(a2[j + 2]), __uint_as_float(a2[j + 3])));
                }
                mbar_arrive_remote(r_full[b]);
                continue;
            }
            float x[64];
#pragma unroll
            for (int j = 0; j < 32; ++j) { x[j] = __uint_as_float(a[j]); x[32 + j] = __uint_as_float(a2[j]); }
            if (NVH == 2) {                  // + the partner's partial of my channels
                mbar_wait_cluster(&rfull[b], (i >> 1) & 1);
                const float* rr = recv + b * (Cfg::RBUF / 4) + (kk & 63) * Cfg::RROW;
#pragma unroll
                for (int j = 0; j < 64; j += 4) {
                    const float4 y = *reinterpret_cast<const float4*>(rr + j);
                    x[j] += y.x; x[j + 1] += y.y; x[j + 2] += y.z; x[j + 3] += y.w;
                }
                mbar_arrive_remote(r_empty[b]);
            }
            // dq_t = e^{b_t - r} x_t, b = chunk-local inclusive cumsum of log alpha (sequential, this channel)
            const float r_ = st_ch[(size_t)i * 2 * K];
            const size_t row0 = rowb + (size_t)i * CH;
            const TG* gp = g + row0 * K + kg;
            __nv_bfloat16* out = dq + row0 * K + kg;
            float bs = 0.f;
#pragma unroll
            for (int t = 0; t < CH; ++t) {
                bs += ld_gate(gp, (size_t)t * K);
                out[(size_t)t * K] = __float2bfloat16_rn(x[t] * ex2f((bs - r_) * L2E));
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (NVH == 2) cluster_sync_all();        // no remote access to this CTA's shared memory after this point
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}

bool dq_kwalk_ok(int K, int V) { return (K == 128 || K == 256) && (V == 256 || V == 512) && !getenv("GLA_DQ3"); }

template <int K, int NVH, typename TG>
static cudaError_t launch_dqk(const CUtensorMap& mK, const CUtensorMap& mDP, const CUtensorMap& mV,
                              const CUtensorMap& mD, const float* stats, const void* g, const float* h0,
                              const float* dfinal, void* dq, float* stdot, const int* flag, int T, int V, int units,
                              cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(k_bwd_dqk<K, NVH, TG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)KwCfg::SMEM);
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(NVH, K / 128, (unsigned)units);
    cfg.blockDim = dim3(KwCfg::NTHR);
    cfg.dynamicSmemBytes = KwCfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = NVH;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_bwd_dqk<K, NVH, TG>, mK, mDP, mV, mD, stats, (const TG*)g, h0, dfinal,
                              (__nv_bfloat16*)dq, stdot, flag, T, V);
}

cudaError_t dq_kwalk(int K, int V, bool gate_f32, const CUtensorMap& mK, const CUtensorMap& mDP,
                     const CUtensorMap& mV, const CUtensorMap& mD, const float* stats, const void* g, const float* h0,
                     const float* dfinal, void* dq, float* stdot, const int* flag, int T, int units, cudaStream_t st) {
#define GLA_DQK(KK, NV)                                                                                           \
    if (K == KK && V == 256 * NV)                                                                                 \
        return gate_f32 ? launch_dqk<KK, NV, float>(mK, mDP, mV, mD, stats, g, h0, dfinal, dq, stdot, flag, T, V, \
                                                    units, st)                                                    \
                        : launch_dqk<KK, NV, __nv_bfloat16>(mK, mDP, mV, mD, stats, g, h0, dfinal, dq, stdot, flag, \
                                                            T, V, units, st);
    GLA_DQK(128, 1) GLA_DQK(128, 2) GLA_DQK(256, 1) GLA_DQK(256, 2)
#undef GLA_DQK
    return cudaErrorNotSupported;
}

}  // namespace tc
}  // namespace gla
