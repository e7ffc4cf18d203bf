// tc_kwalk.cu -- the dq and dk walks of the backward with the key channels on the TMEM lanes ("K-tiled walks",
// DESIGN.md §5).  DESIGN.md §4 (P:250-262 differentiated):
//   dq = e^{b-r} (.) [ dO (H_i e^r)^T + dP K~ ]              forward walk over the chunks, state H
//   dk = e^{r-b} (.) [ V (e^{Gamma-r} dH_{i+1})^T + dP^T Q~ ]  reverse walk over the chunks, adjoint state dH
// Both inter terms contract over the values v.  One CTA per (unit, 128-channel group, 256-value half).  Its TMEM
// holds the (adjoint) state tile transposed, X[k][v], 128 channels k on the lanes x 256 values v on the columns:
//   * the per-chunk decay of the state pass is one scalar per thread (a channel per lane);
//   * SB = bf16(X) stays in TMEM as the A operand (K-major: k rows, v packed in pairs) of the output MMAs
//     out^T[k][t] = SB[k][v] B^T[v][t] (TS mode) -- SB never touches shared memory;
//   * the state update X[k][v] += A^T[k][s] B[s][v] is one N = 128 MMA per value half and 16-token step.
// At V = 512 the two value halves of a channel group run as a 2-CTA cluster and combine their partials through
// distributed shared memory: each CTA pushes its partial of the other half's 32 tokens of every chunk into the
// peer's shared memory (st.async, completion counted on the peer's mbarrier), adds the peer's partial of its own
// 32 tokens (own + peer: fixed order, deterministic) and writes the combined unscaled fp32 rows of those tokens.
// The reduce kernel then reads ONE fp32 dq and one dk per element, scales by e^{+-(b - r)} and forms d log alpha.
//   dq walk (REV = 0): A = K~hi, state B = V, output B = dO (K-major), intra + K~^T dP^T; X_0 = h0; f = e^{pend + r}
//   dk walk (REV = 1): A = Q~hi, state B = dO, output B = V (K-major), intra + Q~^T dP;  X = dfinal; f = e^{pend + Gamma - r}
//   warps 0-7   state pass, one value half at a time (X half scaled in place, SB half written), signalled per half
//   warp 8      state MMA per value half, commits bar_sh[half]
//   warps 9, 10 out^T = SB[:, half 0] B^T (+ the intra term on value half 0) then += SB[:, half 1] B^T (fixed
//               order) into a double-buffered TMEM accumulator
//   warps 11-14 epilogue: accumulator -> (peer exchange) -> combined fp32 rows (coalesced)
//   warp 15     TMA producer: inputs two chunks ahead
// Measured alternatives (1.3B shapes): a 2-CTA cluster exchanging the dq partials through DSMEM and scaling by
// e^{b-r} in the walk's epilogue took the dq walk from ~100 us to ~350 us (the exchange and the per-channel
// strided scan of log alpha each cost ~100 us); one single-buffered accumulator per value half (so the two
// halves' MMAs never wait for each other) was 9 us slower than the ordered double-buffered one.
#include <cstdlib>
#include <type_traits>
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
    static constexpr uint32_t AT = 2 * 8192;                  // A tile (K~ or Q~) [64 s][128 k] (2 SW128 blocks)
    static constexpr uint32_t ST = 4 * 8192;                  // state B tile (V or dO) [64 s][256 v] (4 blocks)
    static constexpr uint32_t OT = 4 * 8192;                  // output B tile (dO or V) [64 t][256 v]
    static constexpr uint32_t PTB = 8192;                     // dP tile [64 t][64 s]
    static constexpr uint32_t OFF_S = AT, OFF_O = AT + ST, OFF_P = AT + ST + OT;
    static constexpr uint32_t STAGE = AT + ST + OT + PTB;
    static constexpr uint32_t OFF_RED = 2 * STAGE;            // [2][128] fp32 (final-state row sums)
    // NVH = 2: the peer's partial of our 32 tokens, pushed by the peer: [128 k][32 t + 4 pad] fp32 (the pad
    // keeps the 16-byte row reads of a quarter warp on distinct banks)
    static constexpr uint32_t PRS = 36, OFF_PR = OFF_RED + 2 * 128 * 4;
    static constexpr uint32_t SMEM = OFF_PR + 128 * PRS * 4 + 1024;
    static_assert(SMEM <= 232448, "dynamic shared memory");
    static constexpr int NST = 256, NTHR = NST + 96 + 128 + 32;   // + warp 15: TMA producer
    static constexpr uint32_t COL_SB = 256, COL_ACC = 384;   // TMEM: X [256] | SB [128] | acc x2 [64 each]
};
}  // namespace

template <int K, bool REV, int NVH>
__global__ void __launch_bounds__(KwCfg::NTHR, 1)
k_bwd_kwalk(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmDP,
            const __grid_constant__ CUtensorMap tmS, const __grid_constant__ CUtensorMap tmO,
            const float* __restrict__ stats, const float* __restrict__ x0, const float* __restrict__ dfinal,
            float* __restrict__ out32, float* __restrict__ stdot, const int* __restrict__ flag,
            const int* __restrict__ cflags, int T, int V, int dbg) {
    // x0: the state entering the walk (REV 0: h0, REV 1: d_final_state), NULL = 0.  dfinal (REV 0 only): with
    // stdot, the final-state row sums rowsum(S_T (.) dS_T) of this value half.  out32: [units * T][K] fp32, the
    // unscaled dq^T / dk^T rows summed over all values.
    // cflags: the forward's per-chunk exact-path flags [units][NC] (R9), or NULL.  A flagged chunk's saved
    // operands are the exact forms (K~ = k e^{Gamma - b}, Q~ = q e^{b}), so its state pass takes the r = 0 frame:
    // X <- X e^{pend + Gamma} (the decay before the update), SB <- bf16(X e^{pend}) (the state at the chunk's
    // start), pending 0 -- the forward walk's exact path -- and its intra term is left to the reduce (the
    // factorised product would overflow there).
    // dbg (GLA_KW_DBG, timing experiments only; results are wrong when set): 4 epilogue only drains the
    // accumulator, 8 no output MMAs, 16 no peer exchange, 32 no global stores of the rows
    using Cfg = KwCfg;
    if (*flag) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* sm = smem_align1k(smem_raw);
    float* red = reinterpret_cast<float*>(sm + Cfg::OFF_RED);
    __shared__ uint64_t bar_in[2], bar_free[2], bar_sbh[2], bar_sh[2], bar_da[2], bar_db[2], bar_efree[2];
    // NVH = 2 peer handshake (one-arrival barriers of the receiving CTA): bar_pr = the peer's partial landed
    // (armed with its bytes by us, completed by the peer's st.async), bar_pfree = the peer has read our partial
    __shared__ uint64_t bar_pr, bar_pfree;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int vh = blockIdx.x, k0 = 128 * blockIdx.y, unit = blockIdx.z;
    const int v0 = 256 * vh, NC = T / CH;
    const size_t rowb = (size_t)unit * T;
    const bool intra = vh == 0;
    auto chunk_of = [&](int j) { return REV ? NC - 1 - j : j; };   // step j -> chunk
    auto load_inputs = [&](int j) {
        const int b = j & 1, row = (int)(rowb + (size_t)chunk_of(j) * CH);
        uint8_t* st = sm + b * Cfg::STAGE;
        mbar_expect_tx(&bar_in[b], Cfg::AT + Cfg::ST + Cfg::OT + (intra ? Cfg::PTB : 0));
        tma_load_2d(st, &tmA, &bar_in[b], k0, row);
        tma_load_2d(st + 8192, &tmA, &bar_in[b], k0 + 64, row);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            tma_load_2d(st + Cfg::OFF_S + q * 8192, &tmS, &bar_in[b], v0 + 64 * q, row);
            tma_load_2d(st + Cfg::OFF_O + q * 8192, &tmO, &bar_in[b], v0 + 64 * q, row);
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
        }
        mbar_init(&bar_pr, 1);
        mbar_init(&bar_pfree, 1);
        fence_mbar_init();
        if (NVH == 2) mbar_expect_tx(&bar_pr, 32 * 128 * 4);   // phase 0 (the peer may push once in sync)
        prefetch_tmap(&tmA); prefetch_tmap(&tmS); prefetch_tmap(&tmO); prefetch_tmap(&tmDP);
        load_inputs(0);
        if (NC > 1) load_inputs(1);
    }
    tc_fence_before();
    __syncthreads();
    if (NVH == 2) cluster_sync_all();        // the peer's barriers are initialised before any remote access
    tc_fence_after();
    const uint32_t tX = tmem_base, tSB = tmem_base + Cfg::COL_SB, tAcc = tmem_base + Cfg::COL_ACC;
    const int lq = warp & 3;
    const uint32_t lane_base = (uint32_t)(32 * lq) << 16;
    const int kk = 32 * lq + lane;           // channel within the group (TMEM lane)
    const int kg = k0 + kk;                  // global channel

    if (warp < 8) {
        // ------------------------------------------------------------------ state warps
        const int cs = 64 * (warp >> 2);     // this warp's 64-column share of each 128-column value half
        const float* x0r = x0 ? x0 + ((size_t)unit * K + kg) * V + v0 : nullptr;
#pragma unroll 1
        for (int c = 0; c < 256; c += 32) {
            if (((c >> 6) & 1) != (warp >> 2)) continue;
            uint32_t r[32];
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
                const float4 x = x0r ? __ldg(reinterpret_cast<const float4*>(x0r + c + j)) : make_float4(0.f, 0.f, 0.f, 0.f);
                r[j] = __float_as_uint(x.x); r[j + 1] = __float_as_uint(x.y);
                r[j + 2] = __float_as_uint(x.z); r[j + 3] = __float_as_uint(x.w);
            }
            tmem_st32(tX + lane_base + c, r);
        }
        tmem_wait_st();
        const float* st_ch = stats + (size_t)unit * NC * 2 * K + kg;   // (r, Gamma) of chunk i at [i * 2K], [i * 2K + K]
        const int* cf = cflags ? cflags + (size_t)unit * NC : nullptr;
        float pend = 0.f, n_r = st_ch[(size_t)chunk_of(0) * 2 * K], n_G = st_ch[(size_t)chunk_of(0) * 2 * K + K];
        int n_slow = cf ? cf[chunk_of(0)] : 0;
        named_bar_sync(1, Cfg::NST);
        for (int j = 0; j < NC; ++j) {
            const float r_ = n_r, G_ = n_G;
            const bool slow = n_slow != 0;
            if (j + 1 < NC) {
                const size_t c1 = (size_t)chunk_of(j + 1) * 2 * K;
                n_r = st_ch[c1];
                n_G = st_ch[c1 + K];
                n_slow = cf ? cf[chunk_of(j + 1)] : 0;
            }
            // REV 0: X <- H_i e^{r} (SB = bf16(X)), pending Gamma - r.  REV 1: X <- dH_{i+1} e^{Gamma - r}, pending r.
            // Exact-path chunk: X <- X e^{pend + Gamma}, SB = bf16(X e^{pend}), pending 0.
            const float f = slow ? ex2f((pend + G_) * L2E) : REV ? ex2f((pend + G_ - r_) * L2E) : ex2f((pend + r_) * L2E);
            const float fsb = slow ? ex2f(pend * L2E) : f;
            pend = slow ? 0.f : REV ? r_ : G_ - r_;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (j > 0) {                 // half h of the previous step: state MMA done, SB half h read
                    mbar_wait(&bar_sh[h], (j - 1) & 1);
                    mbar_wait(h == 0 ? &bar_da[(j - 1) & 1] : &bar_db[(j - 1) & 1], ((j - 1) >> 1) & 1);
                    tc_fence_after();
                }
#pragma unroll
                for (int s = 0; s < 2; ++s) {
                    const int c = 128 * h + cs + 32 * s;
                    uint32_t r[32], pk[16];
                    tmem_ld32(tX + lane_base + c, r);
                    tmem_wait_ld();
                    if (!slow) {
#pragma unroll
                        for (int q = 0; q < 32; q += 2) {
                            const float2 y = mul2(make_float2(__uint_as_float(r[q]), __uint_as_float(r[q + 1])),
                                                  make_float2(f, f));
                            r[q] = __float_as_uint(y.x);
                            r[q + 1] = __float_as_uint(y.y);
                            pk[q / 2] = pack2(y);
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < 32; q += 2) {
                            const float2 x = make_float2(__uint_as_float(r[q]), __uint_as_float(r[q + 1]));
                            const float2 y = mul2(x, make_float2(f, f));
                            r[q] = __float_as_uint(y.x);
                            r[q + 1] = __float_as_uint(y.y);
                            pk[q / 2] = pack2(mul2(x, make_float2(fsb, fsb)));
                        }
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
        if (!REV && dfinal && stdot) {   // rowsum over this CTA's values of S_T (.) dS_T (one partial per half)
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
                for (int q = 0; q < 32; q += 4) {
                    const float4 d = __ldg(reinterpret_cast<const float4*>(dfr + c + q));
                    acc += __uint_as_float(r[q]) * d.x + __uint_as_float(r[q + 1]) * d.y +
                           __uint_as_float(r[q + 2]) * d.z + __uint_as_float(r[q + 3]) * d.w;
                }
            }
            red[(warp >> 2) * 128 + kk] = acc * fe;
            named_bar_sync(1, Cfg::NST);
            if (warp < 4) stdot[((size_t)vh * gridDim.z + unit) * K + kg] = red[kk] + red[128 + kk];
        }
    } else if (warp == 8) {
        // ------------------------------------------------------------------ state MMA issuer (per value half)
        const uint32_t idS = idesc_bf16(128, 128, 1, 1);   // X[k][v] += A^T[k][s] B[s][v]: A, B MN-major
        for (int j = 0; j < NC; ++j) {
            const int b = j & 1;
            const uint32_t aA = smem_u32(sm + b * Cfg::STAGE), aS = aA + Cfg::OFF_S;
            for (int h = 0; h < 2; ++h) {
                mbar_wait(&bar_sbh[h], j & 1);
                if (h == 0) mbar_wait(&bar_in[b], (j >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int s = 0; s < CH / 16; ++s)
                    mma_bf16_w(tX + 128 * h, sdesc_sw128(aA + s * 2048, 8192, 1024),
                               sdesc_sw128(aS + 2 * h * 8192 + s * 2048, 8192, 1024), idS, 1);
                mma_commit_w(&bar_sh[h]);
            }
            mma_commit_w(&bar_free[b]);
            __syncwarp();
        }
    } else if (warp < 11) {
        // ------------------------------------------------------------------ output issuers (value half 0, then 1)
        const int h = warp - 9;
        const uint32_t idO = idesc_bf16(128, 64, 0, 0);            // out^T[k][t] += SB[k][v] B[t][v]: A in TMEM
        const uint32_t idIN = idesc_bf16(128, 64, 1, REV ? 1 : 0); // += A^T[k][s] dP^T (dq) / dP (dk)
        const int* cf = (h == 0 && intra && cflags) ? cflags + (size_t)unit * NC : nullptr;
        int n_exact = cf ? cf[chunk_of(0)] : 0;   // exact-path flag of chunk j, loaded one step ahead
        for (int j = 0; j < NC; ++j) {
            const bool exact = n_exact != 0;
            if (cf && j + 1 < NC) n_exact = cf[chunk_of(j + 1)];
            const int b = j & 1;
            const uint32_t aA = smem_u32(sm + b * Cfg::STAGE), aO = aA + Cfg::OFF_O, adP = aA + Cfg::OFF_P;
            const uint32_t acc = tAcc + 64 * b;
            mbar_wait(&bar_sbh[h], j & 1);
            mbar_wait(&bar_in[b], (j >> 1) & 1);
            if (h == 0 && j >= 2) mbar_wait(&bar_efree[b], ((j >> 1) - 1) & 1);
            if (h == 1) mbar_wait(&bar_da[b], (j >> 1) & 1);   // accumulate after half 0 (fixed order)
            tc_fence_after();
            if (!(dbg & 8))
#pragma unroll
                for (int s = 0; s < 8; ++s)
                    mma_bf16_ta_w(acc, tSB + 64 * h + 8 * s,
                                  sdesc_sw128(aO + (2 * h + (s >> 2)) * 8192 + (s & 3) * 32, 16, 1024), idO,
                                  (h == 1 || s > 0) ? 1u : 0u);
            if (h == 0 && intra && !exact)   // (exact-path chunks: the intra term is formed in the reduce)
#pragma unroll
                for (int s = 0; s < CH / 16; ++s)   // dq: B = dP[t][s] K-major; dk: B = dP[t][s] MN-major (N = s)
                    mma_bf16_w(acc, sdesc_sw128(aA + s * 2048, 8192, 1024),
                               REV ? sdesc_sw128(adP + s * 2048, 8192, 1024) : sdesc_sw128(adP + s * 32, 16, 1024),
                               idIN, 1);
            mma_commit_w(h == 0 ? &bar_da[b] : &bar_db[b]);
            mma_commit_w(&bar_free[b]);
            __syncwarp();
        }
    } else if (warp == 15) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0)
            for (int j = 2; j < NC; ++j) {   // inputs of step j into buffer j & 1 once step j-2's MMAs are done
                mbar_wait(&bar_free[j & 1], ((j - 2) >> 1) & 1);
                load_inputs(j);
            }
    } else {
        // ------------------------------------------------------------------ epilogue warps
        // Each thread drains one channel row of the accumulator (64 tokens, fp32).  It writes the unscaled rows
        // out32[unit rows][K] of the tokens this CTA finishes (all 64, or with NVH = 2 the 32 of value half vh,
        // after adding the peer's partial): for a fixed token the 32 lanes of a warp write 32 consecutive channels
        // (128 B), so every store instruction is fully coalesced.
        const int et = tid - Cfg::NST - 96;
        float* outp = out32 + rowb * K + kg;
        float* prbuf = reinterpret_cast<float*>(sm + Cfg::OFF_PR);
        const uint32_t peer_pr = NVH == 2 ? mapa_shared(prbuf, vh ^ 1) : 0u;
        const uint32_t peer_prb = NVH == 2 ? mapa_shared(&bar_pr, vh ^ 1) : 0u;
        const uint32_t peer_pfree = NVH == 2 ? mapa_shared(&bar_pfree, vh ^ 1) : 0u;
        auto walk = [&](auto Hc) {           // H: this CTA's value half, compile-time (static register indexing)
            constexpr int H = decltype(Hc)::value, T0 = NVH == 2 ? 32 * H : 0, PT = 32 * (H ^ 1);
            for (int j = 0; j < NC; ++j) {
                const int b = j & 1;
                mbar_wait(&bar_db[b], (j >> 1) & 1);
                tc_fence_after();
                uint32_t a[32], a2[32];
                tmem_ld32(tAcc + 64 * b + lane_base, a);
                tmem_ld32(tAcc + 64 * b + 32 + lane_base, a2);
                tmem_wait_ld();
                tc_fence_before();
                named_bar_sync(2, 128);      // accumulator b drained
                if (et == 0) mbar_arrive(&bar_efree[b]);
                if (dbg & 4) continue;
                float acc[64];
#pragma unroll
                for (int t = 0; t < 32; ++t) {
                    acc[t] = __uint_as_float(a[t]);
                    acc[32 + t] = __uint_as_float(a2[t]);
                }
                if (NVH == 2 && !(dbg & 16)) {
                    // our partial of the peer's 32 tokens -> the peer's buffer (row kk) once the peer has read the
                    // previous one; then the peer's partial of ours, added in a fixed order (own + peer)
                    if (j > 0) mbar_wait_cluster(&bar_pfree, (j - 1) & 1);
                    const uint32_t dst = peer_pr + 4u * (uint32_t)(kk * Cfg::PRS);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        st_async_v4(dst + 16u * q, make_float4(acc[PT + 4 * q], acc[PT + 4 * q + 1], acc[PT + 4 * q + 2],
                                                               acc[PT + 4 * q + 3]), peer_prb);
                    mbar_wait_cluster(&bar_pr, j & 1);
                    const float4* src = reinterpret_cast<const float4*>(prbuf + kk * Cfg::PRS);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const float4 v = src[q];
                        acc[T0 + 4 * q] += v.x; acc[T0 + 4 * q + 1] += v.y;
                        acc[T0 + 4 * q + 2] += v.z; acc[T0 + 4 * q + 3] += v.w;
                    }
                    named_bar_sync(2, 128);  // buffer read by every thread
                    if (et == 0) {
                        if (j + 1 < NC) mbar_expect_tx(&bar_pr, 32 * 128 * 4);   // arm the next phase first
                        mbar_arrive_remote_relaxed(peer_pfree);
                    }
                }
                float* o = outp + ((size_t)chunk_of(j) * CH + T0) * K;
                if (!(dbg & 32))
#pragma unroll
                for (int t = 0; t < (NVH == 2 ? 32 : 64); ++t) o[(size_t)t * K] = acc[T0 + t];
            }
        };
        if (NVH == 1 || vh == 0) walk(std::integral_constant<int, 0>{});
        else walk(std::integral_constant<int, 1>{});
    }
    if (NVH == 2) {                          // no CTA leaves while its peer may still write to it
        tc_fence_before();
        cluster_sync_all();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem_base, 512);
}

bool kwalk_ok(int K, int V) { return (K == 128 || K == 256) && (V == 256 || V == 512) && !getenv("GLA_DQ3"); }

template <int K, bool REV, int NVH>
static cudaError_t launch_kw(const CUtensorMap& mA, const CUtensorMap& mDP, const CUtensorMap& mS, const CUtensorMap& mO,
                             const float* stats, const float* x0, const float* dfinal, float* out32, float* stdot,
                             const int* flag, const int* cflags, int T, int V, int units, cudaStream_t st) {
    auto kern = k_bwd_kwalk<K, REV, NVH>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KwCfg::SMEM);
    if (e != cudaSuccess) return e;
    static const int dbg = getenv("GLA_KW_DBG") ? atoi(getenv("GLA_KW_DBG")) : 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(NVH, K / 128, (unsigned)units);
    cfg.blockDim = dim3(KwCfg::NTHR);
    cfg.dynamicSmemBytes = KwCfg::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;   // the value halves of a channel group: one cluster
    attr[0].val.clusterDim.x = NVH;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if ((e = cudaLaunchKernelEx(&cfg, kern, mA, mDP, mS, mO, stats, x0, dfinal, out32, stdot, flag, cflags, T, V, dbg)) !=
        cudaSuccess)
        return e;
    return cudaGetLastError();
}

template <bool REV>
static cudaError_t kw_dispatch(int K, int V, const CUtensorMap& mA, const CUtensorMap& mDP, const CUtensorMap& mS,
                               const CUtensorMap& mO, const float* stats, const float* x0, const float* dfinal,
                               float* out32, float* stdot, const int* flag, const int* cflags, int T, int units,
                               cudaStream_t st) {
#define GLA_KW(KK, NV)                                                                                              \
    if (K == KK && V == 256 * NV)                                                                                   \
        return launch_kw<KK, REV, NV>(mA, mDP, mS, mO, stats, x0, dfinal, out32, stdot, flag, cflags, T, V, units, st);
    GLA_KW(128, 1) GLA_KW(128, 2) GLA_KW(256, 1) GLA_KW(256, 2)
#undef GLA_KW
    return cudaErrorNotSupported;
}

cudaError_t dq_kwalk(int K, int V, const CUtensorMap& mK, const CUtensorMap& mDP, const CUtensorMap& mV,
                     const CUtensorMap& mD, const float* stats, const float* h0, const float* dfinal, float* dq32,
                     float* stdot, const int* flag, const int* cflags, int T, int units, cudaStream_t st) {
    return kw_dispatch<false>(K, V, mK, mDP, mV, mD, stats, h0, dfinal, dq32, stdot, flag, cflags, T, units, st);
}

cudaError_t dk_kwalk(int K, int V, const CUtensorMap& mQ, const CUtensorMap& mDP, const CUtensorMap& mD,
                     const CUtensorMap& mV, const float* stats, const float* dfinal, float* dk32, const int* flag,
                     const int* cflags, int T, int units, cudaStream_t st) {
    return kw_dispatch<true>(K, V, mQ, mDP, mD, mV, stats, dfinal, nullptr, dk32, nullptr, flag, cflags, T, units, st);
}

}  // namespace tc
}  // namespace gla
