// simt.cu -- fp32-arithmetic CUDA-core kernels for chunk-wise GLA (the "fp32 debug build").
//
// Every step of the method runs here in fp32 with exact per-element exponents (no tensor cores):
//   k_intra_P      : intra-chunk score matrix P per chunk via secondary chunking:
//                    off-diagonal sub-chunk pairs factorised with the key-sub-chunk-end normaliser
//                    (both factors <= 1), diagonal sub-chunk blocks with per-element exponent
//                    b_t - b_s <= 0 ("full-precision log space").
//   k_intra_dP     : dP = (dO V^T) (.) M  (causal incl. diagonal) for the backward.
//   k_fwd_state    : per (bh, V-tile): chunk-local cumsum, cross-chunk output Q (.) e^b H,
//                    intra output P V, state passing H <- e^Gamma H + (K (.) e^{Gamma-b})^T V.
//   k_bwd_dq       : per (bh, K-tile), forward walk recomputing H: dq (inter + intra); writes S_T rows.
//   k_bwd_dk       : per (bh, K-tile), reverse walk of dH: dk, d log alpha (global reverse cumsum of
//                    q.dq - k.dk plus rowsum(S_T (.) dS_T)), d_initial_state rows.
//   k_bwd_dv       : per (bh, V-tile), reverse walk of dH: dv.  Also serves gla_dstate_summary.
//   k_step         : one recurrent decode step.
//   k_combine      : H_out = e^{D} (.) H_in + S_loc.
// Layout [B,H,T,D] row-major; one (b,h) unit = "bh".  No atomics: fixed reduction order.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "prof.h"
#include "simt.h"

namespace gla {
namespace simt {

constexpr int NT = 256;      // threads per CTA
constexpr int KS = 24;       // channel slice for the intra kernels (3 x [MAXC][KS+1] fp32 static smem < 48 KB)
constexpr int VT_FWD = 32;   // V tile of k_fwd_state / k_bwd_dv
constexpr int KT_BWD = 32;   // K tile of k_bwd_dq / k_bwd_dk
constexpr int VS_BWD = 64;   // V slice staged per step in k_bwd_dq / k_bwd_dk
constexpr int MAXC = 128;
// GLA_SIMT_NOTILE=1: every SIMT kernel runs its scalar loops (the chunk-size sweep compares plans on equal code)
static int simt_tiles() {
    static const int v = getenv("GLA_SIMT_NOTILE") ? 0 : 1;
    return v;
}    // largest chunk C (the f4 chunk-size sweep runs C = 8 .. 128)

// ---------------------------------------------------------------------------------------------
// P[t][s] (s <= t) for one chunk.  grid (T/C, BH).  P written to Pws[bh][chunk][C][C] (fp32).
template <typename TQ, typename TG>
__global__ void __launch_bounds__(NT) k_intra_P(const TQ* __restrict__ q, const TQ* __restrict__ k,
                                                const TG* __restrict__ g, float* __restrict__ Pws,
                                                int T, int K, int C, int c, const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    __shared__ float sq[MAXC][KS + 1], sk[MAXC][KS + 1], sb[MAXC][KS + 1];
    const int chunk = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    const size_t base = ((size_t)bh * T + (size_t)chunk * C) * K;
    float acc[(MAXC * MAXC) / NT];
#pragma unroll
    for (int j = 0; j < (MAXC * MAXC) / NT; ++j) acc[j] = 0.f;
    for (int m0 = 0; m0 < K; m0 += KS) {
        const int ms = min(KS, K - m0);
        __syncthreads();
        for (int e = tid; e < C * KS; e += NT) {
            const int t = e / KS, m = e % KS;
            float qv = 0.f, kv = 0.f, gv = 0.f;
            if (m < ms) {
                qv = to_f(q[base + (size_t)t * K + m0 + m]);
                kv = to_f(k[base + (size_t)t * K + m0 + m]);
                gv = to_f(g[base + (size_t)t * K + m0 + m]);
            }
            sq[t][m] = qv; sk[t][m] = kv; sb[t][m] = gv;
        }
        __syncthreads();
        if (tid < KS) {                       // (a1) chunk-local inclusive cumsum, one column per thread
            float run = 0.f;
            for (int t = 0; t < C; ++t) { run += sb[t][tid]; sb[t][tid] = run; }
        }
        __syncthreads();
        int j = 0;
        for (int e = tid; e < C * C; e += NT, ++j) {
            const int t = e / C, s = e % C;
            if (s > t) continue;
            const int x = t / c, y = s / c;
            float a = 0.f;
            if (x == y) {                         // diagonal sub-chunk: exponent b_t - b_s <= 0
                for (int m = 0; m < ms; ++m) a += sq[t][m] * sk[s][m] * fexp(sb[t][m] - sb[s][m]);
            } else {                              // off-diagonal pair: normaliser e_y = b[(y+1)c - 1]
                const int ey = (y + 1) * c - 1;
                for (int m = 0; m < ms; ++m) {
                    const float e = sb[ey][m];
                    a += (sq[t][m] * fexp(sb[t][m] - e)) * (sk[s][m] * fexp(e - sb[s][m]));
                }
            }
            acc[j] += a;
        }
    }
    float* out = Pws + ((size_t)bh * (T / C) + chunk) * (size_t)C * C;
    int j = 0;
    for (int e = tid; e < C * C; e += NT, ++j) {
        const int t = e / C, s = e % C;
        out[e] = (s <= t) ? acc[j] : 0.f;
    }
}

// dP[t][s] = sum_v dO[t][v] V[s][v] for s <= t.  grid (T/C, BH).
template <typename TQ>
__global__ void __launch_bounds__(NT) k_intra_dP(const TQ* __restrict__ dO, const TQ* __restrict__ v,
                                                 float* __restrict__ dPws, int T, int V, int C, const int* __restrict__ run_if) {
    if (run_if && *run_if == 0) return;
    __shared__ float sd[MAXC][KS + 1], sv[MAXC][KS + 1];
    const int chunk = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    const size_t base = ((size_t)bh * T + (size_t)chunk * C) * V;
    float acc[(MAXC * MAXC) / NT];
#pragma unroll
    for (int j = 0; j < (MAXC * MAXC) / NT; ++j) acc[j] = 0.f;
    for (int c0 = 0; c0 < V; c0 += KS) {
        const int cs = min(KS, V - c0);
        __syncthreads();
        for (int e = tid; e < C * KS; e += NT) {
            const int t = e / KS, m = e % KS;
            sd[t][m] = m < cs ? to_f(dO[base + (size_t)t * V + c0 + m]) : 0.f;
            sv[t][m] = m < cs ? to_f(v[base + (size_t)t * V + c0 + m]) : 0.f;
        }
        __syncthreads();
        int j = 0;
        for (int e = tid; e < C * C; e += NT, ++j) {
            const int t = e / C, s = e % C;
            if (s > t) continue;
            float a = 0.f;
            for (int m = 0; m < cs; ++m) a += sd[t][m] * sv[s][m];
            acc[j] += a;
        }
    }
    float* out = dPws + ((size_t)bh * (T / C) + chunk) * (size_t)C * C;
    int j = 0;
    for (int e = tid; e < C * C; e += NT, ++j) {
        const int t = e / C, s = e % C;
        out[e] = (s <= t) ? acc[j] : 0.f;
    }
}

// Register-tiled loops of the V-tiled kernels (k_fwd_state, k_bwd_dv) for C = 64, K % 32 == 0: lane = value column
// j of the 32-wide tile; float4 loads along the channels (broadcast within a warp).  Fixed summation order.
//   rows:   a[r] = sum_m X[t][m] S[m][j]  for the 8 tokens t = warp + 8 r           (X [C][K], S [K][32])
//   update: S[m][j] = eS[m] S[m][j] + sum_s A[s][m] Y[s][j]  for the channels m = 4 (warp + 8 r) + u
__device__ __forceinline__ void rows_tile64(float (&a)[8], const float* X, const float* S, int K) {
    const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int m = 0; m < K; m += 4) {
        const float s0 = S[m * VT_FWD + j], s1 = S[(m + 1) * VT_FWD + j], s2 = S[(m + 2) * VT_FWD + j],
                    s3 = S[(m + 3) * VT_FWD + j];
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const float4 x = *reinterpret_cast<const float4*>(X + (w + 8 * r) * K + m);
            a[r] += x.x * s0 + x.y * s1 + x.z * s2 + x.w * s3;
        }
    }
}
__device__ __forceinline__ void update_vtile64(float* S, const float* eS, const float* A, const float* Y, int K, int C,
                                               float cd, bool has_cd) {
    const int j = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int m0 = 4 * w; m0 < K; m0 += 32) {   // 4 consecutive channels per pass
        float u[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) u[q] = eS[m0 + q] * S[(m0 + q) * VT_FWD + j];
        for (int s = 0; s < C; ++s) {
            const float y = Y[s * VT_FWD + j];
            const float4 a4 = *reinterpret_cast<const float4*>(A + s * K + m0);
            u[0] += a4.x * y; u[1] += a4.y * y; u[2] += a4.z * y; u[3] += a4.w * y;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) S[(m0 + q) * VT_FWD + j] = has_cd ? u[q] * cd : u[q];
    }
}

// ---------------------------------------------------------------------------------------------
// Shared-memory carve-up for the (bh, V-tile) kernels: qe,ke [C][K], H [K][VT], P [C][C], V [C][VT],
// expG [K].
__host__ __device__ inline size_t fwd_state_smem(int C, int K) {
    return sizeof(float) * ((size_t)2 * C * K + (size_t)K * VT_FWD + (size_t)C * C + (size_t)C * VT_FWD + K);
}

// grid (V/VT_FWD, BH).  mode 0: forward (out, optional final_state); mode 1: state summary
// (final_state only = S_loc, log_decay written by vtile 0).
template <typename TQ, typename TG>
__global__ void __launch_bounds__(NT) k_fwd_state(const TQ* __restrict__ q, const TQ* __restrict__ k,
                                                  const TQ* __restrict__ v, const TG* __restrict__ g,
                                                  const float* __restrict__ Pws, const float* __restrict__ h0,
                                                  TQ* __restrict__ out, float* __restrict__ final_state,
                                                  float* __restrict__ log_decay, int T, int K, int V, int C,
                                                  int mode, const float* __restrict__ colD = nullptr, int tile_ok = 1) {
    // colD (value-gate path, simt_beta.cu; NULL = 1): the state update is followed by a per-value-column decay
    // colD[bh][chunk][v], i.e. H <- colD (.)_col (e^Gamma H + (K e^{Gamma-b})^T V).
    extern __shared__ float smem[];
    float* qe = smem;                          // [C][K]   q (.) e^{b}
    float* ke = qe + C * K;                    // [C][K]   k (.) e^{Gamma - b}
    float* Hs = ke + C * K;                    // [K][VT]
    float* Ps = Hs + K * VT_FWD;               // [C][C]
    float* Vs = Ps + C * C;                    // [C][VT]
    float* eG = Vs + C * VT_FWD;               // [K]      e^{Gamma}
    const int vt = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    const int v0 = vt * VT_FWD;
    const int NC = T / C;
    const bool tiled = tile_ok && C == 64 && K % 32 == 0;
    for (int e = tid; e < K * VT_FWD; e += NT) {
        const int m = e / VT_FWD, j = e % VT_FWD;
        Hs[e] = (h0 && v0 + j < V) ? h0[((size_t)bh * K + m) * V + v0 + j] : 0.f;
    }
    for (int i = 0; i < NC; ++i) {
        const size_t rowK = ((size_t)bh * T + (size_t)i * C) * K;
        const size_t rowV = ((size_t)bh * T + (size_t)i * C) * V;
        __syncthreads();
        // (a1) chunk-local inclusive cumsum b, one channel per thread; build qe, ke.
        for (int m = tid; m < K; m += NT) {   // (unrolled: batches of independent loads, not one per token)
            float run = 0.f;
#pragma unroll 8
            for (int t = 0; t < C; ++t) {
                run += to_f(g[rowK + (size_t)t * K + m]);
                ke[t * K + m] = run;                                   // b_t (temporarily)
                if (mode == 0) qe[t * K + m] = to_f(q[rowK + (size_t)t * K + m]) * fexp(run);
            }
#pragma unroll 8
            for (int t = 0; t < C; ++t)
                ke[t * K + m] = to_f(k[rowK + (size_t)t * K + m]) * fexp(run - ke[t * K + m]);
            eG[m] = fexp(run);
        }
        for (int e = tid; e < C * VT_FWD; e += NT) {
            const int t = e / VT_FWD, j = e % VT_FWD;
            Vs[e] = (v0 + j < V) ? to_f(v[rowV + (size_t)t * V + v0 + j]) : 0.f;
        }
        if (mode == 0) {
            const float* Pc = Pws + ((size_t)bh * NC + i) * (size_t)C * C;
            for (int e = tid; e < C * C; e += NT) Ps[e] = Pc[e];
        }
        __syncthreads();
        if (mode == 0) {
            // o_t = (q_t (.) e^{b_t}) H_i + sum_s P_ts v_s
            const int j = tid % VT_FWD;
            if (tiled) {
                float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                rows_tile64(a, qe, Hs, K);
                const int w = tid / VT_FWD;
                for (int s = 0; s < C; ++s) {
                    const float vs = Vs[s * VT_FWD + j];
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (s <= w + 8 * r) a[r] += Ps[(w + 8 * r) * C + s] * vs;
                }
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (v0 + j < V) out[rowV + (size_t)(w + 8 * r) * V + v0 + j] = from_f<TQ>(a[r]);
            } else {
                for (int t = tid / VT_FWD; t < C; t += NT / VT_FWD) {
                    float a = 0.f;
                    for (int m = 0; m < K; ++m) a += qe[t * K + m] * Hs[m * VT_FWD + j];
                    for (int s = 0; s <= t; ++s) a += Ps[t * C + s] * Vs[s * VT_FWD + j];
                    if (v0 + j < V) out[rowV + (size_t)t * V + v0 + j] = from_f<TQ>(a);
                }
            }
            __syncthreads();
        }
        // H_{i+1} = e^{Gamma} (.) H_i + (K (.) e^{Gamma - b})^T V
        {
            const int j = tid % VT_FWD;
            const float cd = (colD && v0 + j < V) ? colD[((size_t)bh * NC + i) * V + v0 + j] : 1.f;
            if (tiled) {
                update_vtile64(Hs, eG, ke, Vs, K, C, cd, colD != nullptr);
            } else {
                for (int m = tid / VT_FWD; m < K; m += NT / VT_FWD) {
                    float a = eG[m] * Hs[m * VT_FWD + j];
                    for (int s = 0; s < C; ++s) a += ke[s * K + m] * Vs[s * VT_FWD + j];
                    Hs[m * VT_FWD + j] = colD ? a * cd : a;
                }
            }
        }
    }
    __syncthreads();
    if (final_state) {
        for (int e = tid; e < K * VT_FWD; e += NT) {
            const int m = e / VT_FWD, j = e % VT_FWD;
            if (v0 + j < V) final_state[((size_t)bh * K + m) * V + v0 + j] = Hs[e];
        }
    }
    if (mode == 1 && log_decay && vt == 0)
        for (int m = tid; m < K; m += NT) {
            // recompute in a fixed order (sum of chunk totals), identical for every m-owner
            float tot = 0.f;
            for (int i = 0; i < NC; ++i) {
                float run = 0.f;
                const size_t rowK = ((size_t)bh * T + (size_t)i * C) * K;
                for (int t = 0; t < C; ++t) run += to_f(g[rowK + (size_t)t * K + m]);
                tot += run;
            }
            log_decay[(size_t)bh * K + m] = tot;
        }
}

// ---------------------------------------------------------------------------------------------
// Backward, K-tiled kernels.  smem: H or dH [KT][V], qe/ke/b for the K-tile [C][KT] x3,
// dP [C][C], staged dO / V slices [C][VS].
__host__ __device__ inline size_t bwd_k_smem(int C, int V) {
    return sizeof(float) * ((size_t)KT_BWD * (V + 4) + (size_t)4 * C * KT_BWD + (size_t)C * C +
                            (size_t)2 * C * VS_BWD + KT_BWD);
}

// Register-tiled inner loops of the K-tiled backward kernels for the common plan C = 64 with V % 4 == 0 (the exact
// fallback of the tensor-core path always has C = 64): lane = channel m of the tile, the 8 warps split the tokens
// (inter) or the values (state update); float4 loads along the values.  Same sums as the scalar loops, in a
// different (still fixed) order.
//   inter:  acc[t][m] += scale(t, m) * sum_{j < cs} X[t][j] S[m][c0 + j]      (8 tokens t = warp + 8 r per thread)
//   update: S[m][c0 + j] = eS * S[m][c0 + j] + sum_s A[s][m] Y[s][j]          (8 values j = 8 warp + u per thread)
template <typename ScaleF>
__device__ __forceinline__ void inter_tile64(float* acc, const float* X, const float* S, int HV, int c0, int cs,
                                             ScaleF scale) {
    const int m = threadIdx.x & 31, w = threadIdx.x >> 5;
    float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const float* srow = S + m * HV + c0;
    for (int j = 0; j < cs; j += 4) {
        const float4 h = *reinterpret_cast<const float4*>(srow + j);
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            const float4 x = *reinterpret_cast<const float4*>(X + (w + 8 * r) * VS_BWD + j);
            a[r] += x.x * h.x + x.y * h.y + x.z * h.z + x.w * h.w;
        }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
        const int t = w + 8 * r;
        acc[t * KT_BWD + m] += a[r] * scale(t, m);
    }
}
__device__ __forceinline__ void update_tile64(float* S, const float* A, const float* Y, int HV, int c0, int cs, float eS,
                                              int C) {
    const int m = threadIdx.x & 31, j0 = 8 * (threadIdx.x >> 5);
    if (j0 >= cs) return;
    float* srow = S + m * HV + c0 + j0;
    float4 u0 = *reinterpret_cast<float4*>(srow), u1 = *reinterpret_cast<float4*>(srow + 4);
    u0.x *= eS; u0.y *= eS; u0.z *= eS; u0.w *= eS; u1.x *= eS; u1.y *= eS; u1.z *= eS; u1.w *= eS;
    for (int s = 0; s < C; ++s) {
        const float am = A[s * KT_BWD + m];
        const float4 y0 = *reinterpret_cast<const float4*>(Y + s * VS_BWD + j0);
        const float4 y1 = *reinterpret_cast<const float4*>(Y + s * VS_BWD + j0 + 4);
        u0.x += am * y0.x; u0.y += am * y0.y; u0.z += am * y0.z; u0.w += am * y0.w;
        u1.x += am * y1.x; u1.y += am * y1.y; u1.z += am * y1.z; u1.w += am * y1.w;
    }
    *reinterpret_cast<float4*>(srow) = u0;
    *reinterpret_cast<float4*>(srow + 4) = u1;
}

// grid (K/KT, BH).  Forward walk: dq_t = e^{b_t} (.) (dO_t H_i^T) + sum_{s<=t} dP_ts k_s e^{b_t - b_s}.
template <typename TQ, typename TG>
__global__ void __launch_bounds__(NT) k_bwd_dq(const TQ* __restrict__ q, const TQ* __restrict__ k,
                                               const TQ* __restrict__ v, const TG* __restrict__ g,
                                               const TQ* __restrict__ dO, const float* __restrict__ h0,
                                               const float* __restrict__ dPws, TQ* __restrict__ dq,
                                               float* __restrict__ dq32, float* __restrict__ ST,
                                               int T, int K, int V, int C, const int* __restrict__ run_if,
                                               const float* __restrict__ colD = nullptr, int tile_ok = 1) {
    if (run_if && *run_if == 0) return;
    extern __shared__ float smem[];
    const int HV = V + 4;                      // padded row stride (16-B rows; lanes = channels hit distinct banks)
    float* Hs = smem;                          // [KT][V + 1]
    float* sb = Hs + KT_BWD * HV;              // [C][KT] b
    float* sk = sb + C * KT_BWD;               // [C][KT] k
    float* ke = sk + C * KT_BWD;               // [C][KT] k e^{Gamma-b}
    float* acc = ke + C * KT_BWD;              // [C][KT] dq accumulator
    float* sdP = acc + C * KT_BWD;             // [C][C]
    float* sd = sdP + C * C;                   // [C][VS] dO slice
    float* sv = sd + C * VS_BWD;               // [C][VS] V slice
    float* eG = sv + C * VS_BWD;               // [KT]
    const int kt = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    const int m0 = kt * KT_BWD;
    const int NC = T / C;
    const bool tiled = tile_ok && C == 64 && V % 4 == 0;
    for (int e = tid; e < KT_BWD * V; e += NT) {
        const int m = e / V, j = e % V;
        Hs[m * HV + j] = (h0 && m0 + m < K) ? h0[((size_t)bh * K + m0 + m) * V + j] : 0.f;
    }
    for (int i = 0; i < NC; ++i) {
        const size_t rowK = ((size_t)bh * T + (size_t)i * C) * K;
        const size_t rowV = ((size_t)bh * T + (size_t)i * C) * V;
        __syncthreads();
        // log alpha and k of this chunk's channel tile staged by all threads (coalesced, independent loads), then
        // the chunk-local cumsum by one thread per channel from shared memory
        for (int e = tid; e < C * KT_BWD; e += NT) {
            const int t = e / KT_BWD, m = e % KT_BWD;
            const bool ok = m0 + m < K;
            sb[e] = ok ? to_f(g[rowK + (size_t)t * K + m0 + m]) : 0.f;
            sk[e] = ok ? to_f(k[rowK + (size_t)t * K + m0 + m]) : 0.f;
        }
        __syncthreads();
        if (tid < KT_BWD) {
            const int m = tid;
            float run = 0.f;
            for (int t = 0; t < C; ++t) {
                run += sb[t * KT_BWD + m];
                sb[t * KT_BWD + m] = run;
            }
            for (int t = 0; t < C; ++t) ke[t * KT_BWD + m] = sk[t * KT_BWD + m] * fexp(run - sb[t * KT_BWD + m]);
            eG[m] = fexp(run);
        }
        const float* dPc = dPws + ((size_t)bh * NC + i) * (size_t)C * C;
        for (int e = tid; e < C * C; e += NT) sdP[e] = dPc[e];
        for (int e = tid; e < C * KT_BWD; e += NT) acc[e] = 0.f;
        __syncthreads();
        // intra: sum_{s<=t} dP_ts k_s e^{b_t - b_s}  (per-element exponent <= 0)
        for (int e = tid; e < C * KT_BWD; e += NT) {
            const int t = e / KT_BWD, m = e % KT_BWD;
            float a = 0.f;
            const float bt = sb[t * KT_BWD + m];
            for (int s = 0; s <= t; ++s) a += sdP[t * C + s] * sk[s * KT_BWD + m] * fexp(bt - sb[s * KT_BWD + m]);
            acc[e] = a;
        }
        for (int c0 = 0; c0 < V; c0 += VS_BWD) {
            const int cs = min(VS_BWD, V - c0);
            __syncthreads();
            for (int e = tid; e < C * VS_BWD; e += NT) {
                const int t = e / VS_BWD, j = e % VS_BWD;
                sd[e] = j < cs ? to_f(dO[rowV + (size_t)t * V + c0 + j]) : 0.f;
                sv[e] = j < cs ? to_f(v[rowV + (size_t)t * V + c0 + j]) : 0.f;
            }
            __syncthreads();
            // inter: e^{b_t} (.) sum_v dO_tv H[m][v]  (H = H_i, before the update below)
            if (tiled)
                inter_tile64(acc, sd, Hs, HV, c0, cs, [&](int t, int m) { return fexp(sb[t * KT_BWD + m]); });
            else
                for (int e = tid; e < C * KT_BWD; e += NT) {
                    const int t = e / KT_BWD, m = e % KT_BWD;
                    float a = 0.f;
                    for (int j = 0; j < cs; ++j) a += sd[t * VS_BWD + j] * Hs[m * HV + c0 + j];
                    acc[e] += a * fexp(sb[t * KT_BWD + m]);
                }
            __syncthreads();
            // H_{i+1}[m][v] = e^{Gamma_m} H + sum_s ke[s][m] V[s][v]  for this V slice
            if (tiled && !colD)
                update_tile64(Hs, ke, sv, HV, c0, cs, eG[tid & 31], C);
            else
                for (int e = tid; e < KT_BWD * VS_BWD; e += NT) {
                    const int m = e / VS_BWD, j = e % VS_BWD;
                    if (j >= cs) continue;
                    float a = eG[m] * Hs[m * HV + c0 + j];
                    for (int s = 0; s < C; ++s) a += ke[s * KT_BWD + m] * sv[s * VS_BWD + j];
                    Hs[m * HV + c0 + j] = colD ? a * colD[((size_t)bh * NC + i) * V + c0 + j] : a;
                }
        }
        __syncthreads();
        for (int e = tid; e < C * KT_BWD; e += NT) {
            const int t = e / KT_BWD, m = e % KT_BWD;
            if (m0 + m < K) {
                dq[rowK + (size_t)t * K + m0 + m] = from_f<TQ>(acc[e]);
                dq32[rowK + (size_t)t * K + m0 + m] = acc[e];
            }
        }
    }
    __syncthreads();
    for (int e = tid; e < KT_BWD * V; e += NT) {
        const int m = e / V, j = e % V;
        if (m0 + m < K) ST[((size_t)bh * K + m0 + m) * V + j] = Hs[m * HV + j];
    }
}

// grid (K/KT, BH).  Reverse walk: dk_s = e^{Gamma-b_s} (.) (v_s dH_{i+1}^T) + sum_{t>=s} dP_ts q_t e^{b_t-b_s};
// d log alpha_t = sum_{s>=t} (q.dq - k.dk)_s + rowsum(S_T (.) dS_T);   dH_i = e^Gamma dH_{i+1} + (q e^b)^T dO.
template <typename TQ, typename TG>
__global__ void __launch_bounds__(NT) k_bwd_dk(const TQ* __restrict__ q, const TQ* __restrict__ k,
                                               const TQ* __restrict__ v, const TG* __restrict__ g,
                                               const TQ* __restrict__ dO, const float* __restrict__ dfinal,
                                               const float* __restrict__ dPws, const float* __restrict__ dq32,
                                               const float* __restrict__ ST, TQ* __restrict__ dk,
                                               float* __restrict__ dg, float* __restrict__ dh0,
                                               int T, int K, int V, int C, const int* __restrict__ run_if,
                                               const float* __restrict__ colD = nullptr, int tile_ok = 1) {
    if (run_if && *run_if == 0) return;
    extern __shared__ float smem[];
    const int HV = V + 4;                      // padded row stride (see k_bwd_dq)
    float* dH = smem;                          // [KT][V + 1]
    float* sb = dH + KT_BWD * HV;              // [C][KT] b
    float* sq = sb + C * KT_BWD;               // [C][KT] q
    float* qe = sq + C * KT_BWD;               // [C][KT] q e^{b}
    float* acc = qe + C * KT_BWD;              // [C][KT] dk accumulator
    float* sdP = acc + C * KT_BWD;             // [C][C]
    float* sd = sdP + C * C;                   // [C][VS] dO slice
    float* sv = sd + C * VS_BWD;               // [C][VS] V slice
    float* carry = sv + C * VS_BWD;            // [KT] running sum for d log alpha
    const int kt = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    const int m0 = kt * KT_BWD;
    const int NC = T / C;
    const bool tiled = tile_ok && C == 64 && V % 4 == 0;
    for (int e = tid; e < KT_BWD * V; e += NT) {
        const int m = e / V, j = e % V;
        dH[m * HV + j] = (dfinal && m0 + m < K) ? dfinal[((size_t)bh * K + m0 + m) * V + j] : 0.f;
    }
    __syncthreads();
    // carry init: rowsum(S_T (.) dS_T) -- the final-state term of d log alpha (R6)
    if (tid < KT_BWD) {
        float a = 0.f;
        if (m0 + tid < K)
            for (int j = 0; j < V; ++j) a += ST[((size_t)bh * K + m0 + tid) * V + j] * dH[tid * HV + j];
        carry[tid] = a;
    }
    for (int i = NC - 1; i >= 0; --i) {
        const size_t rowK = ((size_t)bh * T + (size_t)i * C) * K;
        const size_t rowV = ((size_t)bh * T + (size_t)i * C) * V;
        __syncthreads();
        if (colD)   // adjoint of the column decay that followed chunk i's update: dH_{i+1} <- colD_i (.)_col dH_{i+1}
            for (int e = tid; e < KT_BWD * V; e += NT) dH[(e / V) * HV + e % V] *= colD[((size_t)bh * NC + i) * V + e % V];
        for (int e = tid; e < C * KT_BWD; e += NT) {   // staged as in k_bwd_dq
            const int t = e / KT_BWD, m = e % KT_BWD;
            const bool ok = m0 + m < K;
            sb[e] = ok ? to_f(g[rowK + (size_t)t * K + m0 + m]) : 0.f;
            sq[e] = ok ? to_f(q[rowK + (size_t)t * K + m0 + m]) : 0.f;
        }
        __syncthreads();
        if (tid < KT_BWD) {
            const int m = tid;
            float run = 0.f;
            for (int t = 0; t < C; ++t) {
                run += sb[t * KT_BWD + m];
                sb[t * KT_BWD + m] = run;
                qe[t * KT_BWD + m] = sq[t * KT_BWD + m] * fexp(run);
            }
        }
        const float* dPc = dPws + ((size_t)bh * NC + i) * (size_t)C * C;
        for (int e = tid; e < C * C; e += NT) sdP[e] = dPc[e];
        __syncthreads();
        // intra: sum_{t>=s} dP_ts q_t e^{b_t - b_s}
        for (int e = tid; e < C * KT_BWD; e += NT) {
            const int s = e / KT_BWD, m = e % KT_BWD;
            float a = 0.f;
            const float bs = sb[s * KT_BWD + m];
            for (int t = s; t < C; ++t) a += sdP[t * C + s] * sq[t * KT_BWD + m] * fexp(sb[t * KT_BWD + m] - bs);
            acc[e] = a;
        }
        for (int c0 = 0; c0 < V; c0 += VS_BWD) {
            const int cs = min(VS_BWD, V - c0);
            __syncthreads();
            for (int e = tid; e < C * VS_BWD; e += NT) {
                const int t = e / VS_BWD, j = e % VS_BWD;
                sd[e] = j < cs ? to_f(dO[rowV + (size_t)t * V + c0 + j]) : 0.f;
                sv[e] = j < cs ? to_f(v[rowV + (size_t)t * V + c0 + j]) : 0.f;
            }
            __syncthreads();
            // inter: e^{Gamma - b_s} (.) sum_v V_sv dH_{i+1}[m][v]
            if (tiled)
                inter_tile64(acc, sv, dH, HV, c0, cs, [&](int t, int m) {
                    return fexp(sb[(C - 1) * KT_BWD + m] - sb[t * KT_BWD + m]);
                });
            else
                for (int e = tid; e < C * KT_BWD; e += NT) {
                    const int s = e / KT_BWD, m = e % KT_BWD;
                    float a = 0.f;
                    for (int j = 0; j < cs; ++j) a += sv[s * VS_BWD + j] * dH[m * HV + c0 + j];
                    acc[e] += a * fexp(sb[(C - 1) * KT_BWD + m] - sb[s * KT_BWD + m]);
                }
            __syncthreads();
            // dH_i = e^{Gamma} dH_{i+1} + (q e^b)^T dO   for this V slice
            if (tiled)
                update_tile64(dH, qe, sd, HV, c0, cs, fexp(sb[(C - 1) * KT_BWD + (tid & 31)]), C);
            else
                for (int e = tid; e < KT_BWD * VS_BWD; e += NT) {
                    const int m = e / VS_BWD, j = e % VS_BWD;
                    if (j >= cs) continue;
                    float a = fexp(sb[(C - 1) * KT_BWD + m]) * dH[m * HV + c0 + j];
                    for (int t = 0; t < C; ++t) a += qe[t * KT_BWD + m] * sd[t * VS_BWD + j];
                    dH[m * HV + c0 + j] = a;
                }
        }
        __syncthreads();
        for (int e = tid; e < C * KT_BWD; e += NT) {
            const int t = e / KT_BWD, m = e % KT_BWD;
            if (m0 + m < K) dk[rowK + (size_t)t * K + m0 + m] = from_f<TQ>(acc[e]);
        }
        // d log alpha: reverse cumsum within the chunk of x = q.dq - k.dk, plus the carry
        if (tid < KT_BWD && m0 + tid < K) {
            const int m = tid;
            float run = carry[m];
            for (int t = C - 1; t >= 0; --t) {
                const size_t ix = rowK + (size_t)t * K + m0 + m;
                const float x = sq[t * KT_BWD + m] * dq32[ix] - to_f(k[ix]) * acc[t * KT_BWD + m];
                run += x;
                dg[ix] = run;
            }
            carry[m] = run;
        }
    }
    __syncthreads();
    if (dh0)
        for (int e = tid; e < KT_BWD * V; e += NT) {
            const int m = e / V, j = e % V;
            if (m0 + m < K) dh0[((size_t)bh * K + m0 + m) * V + j] = dH[m * HV + j];
        }
}

// grid (V/VT, BH).  Reverse walk: dv_s = sum_{t>=s} P_ts dO_t + (k_s e^{Gamma - b_s}) dH_{i+1}.
// mode 0: dv; mode 1: dstate summary only (dH_0 with dfinal = 0 written to dh0).
template <typename TQ, typename TG>
__global__ void __launch_bounds__(NT) k_bwd_dv(const TQ* __restrict__ q, const TQ* __restrict__ k,
                                               const TG* __restrict__ g, const TQ* __restrict__ dO,
                                               const float* __restrict__ dfinal, const float* __restrict__ Pws,
                                               TQ* __restrict__ dv, float* __restrict__ dh0,
                                               int T, int K, int V, int C, int mode, const int* __restrict__ run_if,
                                               const float* __restrict__ colD = nullptr, int tile_ok = 1) {
    if (run_if && *run_if == 0) return;
    extern __shared__ float smem[];
    float* qe = smem;                          // [C][K] q e^{b}
    float* ke = qe + C * K;                    // [C][K] k e^{Gamma-b}
    float* dH = ke + C * K;                    // [K][VT]
    float* Ps = dH + K * VT_FWD;               // [C][C]
    float* sd = Ps + C * C;                    // [C][VT]
    float* eG = sd + C * VT_FWD;               // [K]
    const int vt = blockIdx.x, bh = blockIdx.y, tid = threadIdx.x;
    const int v0 = vt * VT_FWD;
    const int NC = T / C;
    const bool tiled = tile_ok && C == 64 && K % 32 == 0;
    for (int e = tid; e < K * VT_FWD; e += NT) {
        const int m = e / VT_FWD, j = e % VT_FWD;
        dH[e] = (dfinal && v0 + j < V) ? dfinal[((size_t)bh * K + m) * V + v0 + j] : 0.f;
    }
    for (int i = NC - 1; i >= 0; --i) {
        const size_t rowK = ((size_t)bh * T + (size_t)i * C) * K;
        const size_t rowV = ((size_t)bh * T + (size_t)i * C) * V;
        __syncthreads();
        if (colD)   // adjoint of the column decay after chunk i (see k_bwd_dk)
            for (int e = tid; e < K * VT_FWD; e += NT)
                if (v0 + e % VT_FWD < V) dH[e] *= colD[((size_t)bh * NC + i) * V + v0 + e % VT_FWD];
        for (int m = tid; m < K; m += NT) {   // (unrolled as in k_fwd_state)
            float run = 0.f;
#pragma unroll 8
            for (int t = 0; t < C; ++t) {
                run += to_f(g[rowK + (size_t)t * K + m]);
                ke[t * K + m] = run;
                qe[t * K + m] = to_f(q[rowK + (size_t)t * K + m]) * fexp(run);
            }
#pragma unroll 8
            for (int t = 0; t < C; ++t)
                ke[t * K + m] = to_f(k[rowK + (size_t)t * K + m]) * fexp(run - ke[t * K + m]);
            eG[m] = fexp(run);
        }
        for (int e = tid; e < C * VT_FWD; e += NT) {
            const int t = e / VT_FWD, j = e % VT_FWD;
            sd[e] = (v0 + j < V) ? to_f(dO[rowV + (size_t)t * V + v0 + j]) : 0.f;
        }
        if (mode == 0) {
            const float* Pc = Pws + ((size_t)bh * NC + i) * (size_t)C * C;
            for (int e = tid; e < C * C; e += NT) Ps[e] = Pc[e];
        }
        __syncthreads();
        if (mode == 0) {
            const int j = tid % VT_FWD;
            if (tiled) {
                float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                const int w = tid / VT_FWD;
                for (int t = 0; t < C; ++t) {
                    const float x = sd[t * VT_FWD + j];
#pragma unroll
                    for (int r = 0; r < 8; ++r)
                        if (t >= w + 8 * r) a[r] += Ps[t * C + w + 8 * r] * x;
                }
                rows_tile64(a, ke, dH, K);
#pragma unroll
                for (int r = 0; r < 8; ++r)
                    if (v0 + j < V) dv[rowV + (size_t)(w + 8 * r) * V + v0 + j] = from_f<TQ>(a[r]);
            } else {
                for (int s = tid / VT_FWD; s < C; s += NT / VT_FWD) {
                    float a = 0.f;
                    for (int t = s; t < C; ++t) a += Ps[t * C + s] * sd[t * VT_FWD + j];
                    for (int m = 0; m < K; ++m) a += ke[s * K + m] * dH[m * VT_FWD + j];
                    if (v0 + j < V) dv[rowV + (size_t)s * V + v0 + j] = from_f<TQ>(a);
                }
            }
            __syncthreads();
        }
        if (tiled) {
            update_vtile64(dH, eG, qe, sd, K, C, 1.f, false);
        } else {
            const int j = tid % VT_FWD;
            for (int m = tid / VT_FWD; m < K; m += NT / VT_FWD) {
                float a = eG[m] * dH[m * VT_FWD + j];
                for (int t = 0; t < C; ++t) a += qe[t * K + m] * sd[t * VT_FWD + j];
                dH[m * VT_FWD + j] = a;
            }
        }
    }
    __syncthreads();
    if (dh0)
        for (int e = tid; e < K * VT_FWD; e += NT) {
            const int m = e / VT_FWD, j = e % VT_FWD;
            if (v0 + j < V) dh0[((size_t)bh * K + m) * V + v0 + j] = dH[e];
        }
}

// ---------------------------------------------------------------------------------------------
constexpr int MAXK_STEP = 1024;
// Decode step.  grid (ceil(V / (4 CQ)), BH), CQ x RG threads = CQ column-quads x RG row groups; every thread
// streams its K / RG state rows (float4 read-modify-write, rows of a warp contiguous), o reduced over the row
// groups in shared memory (fixed order).  Small batches use narrow tiles (CQ = 8, RG = 16) to spread the state
// over more SMs (CQ = 4, RG = 32 when even those leave SMs idle); large batches the wide ones (CQ = 32, RG = 8).
template <typename TQ, typename TG, int CQ, int RG>
__global__ void __launch_bounds__(CQ * RG) k_step(const TQ* __restrict__ q, const TQ* __restrict__ k,
                                                  const TQ* __restrict__ v, const TG* __restrict__ g,
                                                  float* __restrict__ state, TQ* __restrict__ out, int K, int V) {
    __shared__ float red[RG][4 * CQ];
    __shared__ float sa[MAXK_STEP], sk[MAXK_STEP], sq[MAXK_STEP];   // alpha, k, q of this unit (staged once)
    const int bh = blockIdx.y, tid = threadIdx.x;
    const int col = blockIdx.x * 4 * CQ + (tid % CQ) * 4;
    const int rg = tid / CQ;
    for (int m = tid; m < K; m += CQ * RG) {
        sa[m] = fexp(to_f(g[(size_t)bh * K + m]));
        sk[m] = to_f(k[(size_t)bh * K + m]);
        sq[m] = to_f(q[(size_t)bh * K + m]);
    }
    float o[4] = {0.f, 0.f, 0.f, 0.f};
    float vv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) vv[u] = (col + u < V) ? to_f(v[(size_t)bh * V + col + u]) : 0.f;
    const bool vec = col + 3 < V && (V % 4) == 0;
    __syncthreads();
    if (vec) {
        // NB rows per batch: all loads first, then the updates and stores (the rows of one thread never alias, but
        // the compiler cannot know that: without the batching every load waited for the previous row's store)
        constexpr int NB = 8;
        float* base = state + (size_t)bh * K * V + col;
        for (int m0 = rg; m0 < K; m0 += RG * NB) {
            float4 s4[NB];
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int m = m0 + u * RG;
                if (m < K) s4[u] = *reinterpret_cast<const float4*>(base + (size_t)m * V);
            }
#pragma unroll
            for (int u = 0; u < NB; ++u) {
                const int m = m0 + u * RG;
                if (m < K) {
                    const float a = sa[m], km = sk[m], qm = sq[m];
                    float4 x = s4[u];
                    x.x = a * x.x + km * vv[0]; x.y = a * x.y + km * vv[1];
                    x.z = a * x.z + km * vv[2]; x.w = a * x.w + km * vv[3];
                    *reinterpret_cast<float4*>(base + (size_t)m * V) = x;
                    o[0] += qm * x.x; o[1] += qm * x.y; o[2] += qm * x.z; o[3] += qm * x.w;
                }
            }
        }
    } else
    for (int m = rg; m < K; m += RG) {
        const float a = sa[m], km = sk[m], qm = sq[m];
        float* row = state + ((size_t)bh * K + m) * V;
        {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (col + u < V) {
                    const float sv = a * row[col + u] + km * vv[u];
                    row[col + u] = sv;
                    o[u] += qm * sv;
                }
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) red[rg][(tid % CQ) * 4 + u] = o[u];
    __syncthreads();
    if (tid < 4 * CQ) {
        float acc = 0.f;
        for (int r = 0; r < RG; ++r) acc += red[r][tid];
        const int c = blockIdx.x * 4 * CQ + tid;
        if (c < V) out[(size_t)bh * V + c] = from_f<TQ>(acc);
    }
}

__global__ void k_combine(const float* __restrict__ Hin, const float* __restrict__ D, const float* __restrict__ S,
                          float* __restrict__ Hout, int BH, int K, int V) {
    const size_t n = (size_t)BH * K * V;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const size_t row = e / V;   // (bh, m)
        Hout[e] = fexp(D[row]) * Hin[e] + S[e];
    }
}

// ---------------------------------------------------------------------------------------------
// Launchers.
template <typename F>
static cudaError_t set_smem(F f, size_t bytes) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

template <typename TQ, typename TG>
static cudaError_t fwd_impl(const Problem& p, cudaStream_t st) {
    const int BH = p.B * p.H, NC = p.T / p.C;
    float* Pws = (float*)p.ws;
    const TQ* q = (const TQ*)p.q; const TQ* k = (const TQ*)p.k; const TQ* v = (const TQ*)p.v;
    const TG* g = (const TG*)p.g;
    if (p.mode == 0) {
        {
            GLA_PROF("simt::k_intra_P", st);
            k_intra_P<TQ, TG><<<dim3(NC, BH), NT, 0, st>>>(q, k, g, Pws, p.T, p.K, p.C, p.c, nullptr);
        }
    }
    const size_t sm = fwd_state_smem(p.C, p.K);
    cudaError_t e = set_smem(k_fwd_state<TQ, TG>, sm);
    if (e != cudaSuccess) return e;
    {
        GLA_PROF("simt::k_fwd_state", st);
        k_fwd_state<TQ, TG><<<dim3(cdiv(p.V, VT_FWD), BH), NT, sm, st>>>(q, k, v, g, Pws, p.h0, (TQ*)p.out,
                                                                        p.final_state, p.log_decay, p.T, p.K,
                                                                        p.V, p.C, p.mode, p.colD, simt_tiles());
    }
    return cudaGetLastError();
}

// Arguments of the exact fallback backward (device-side launch of the five kernels below).
template <typename TQ, typename TG>
struct BwdArgs {
    const TQ *q, *k, *v; const TG* g; const TQ* dO; const float *h0, *dfinal;
    float *Pws, *dPws, *dq32, *ST; TQ *dq, *dk, *dv; float *dg, *dh0;
    int T, K, V, C, c, BH, NC; size_t smk, smv;
};
// Gate for the tensor-core backward's exact fallback: when the device flag is set (a chunk failed the
// factorisation guard, R9) it tail-launches the fp32 CUDA-core backward, which then runs after this
// grid in launch order and overwrites every gradient; otherwise it costs one one-warp launch.
template <typename TQ, typename TG>
__global__ void k_bwd_gate(BwdArgs<TQ, TG> a, const int* __restrict__ flag) {
    if (threadIdx.x != 0 || *flag == 0) return;
    k_intra_P<TQ, TG><<<dim3(a.NC, a.BH), NT, 0, cudaStreamTailLaunch>>>(a.q, a.k, a.g, a.Pws, a.T, a.K, a.C, a.c, nullptr);
    k_intra_dP<TQ><<<dim3(a.NC, a.BH), NT, 0, cudaStreamTailLaunch>>>(a.dO, a.v, a.dPws, a.T, a.V, a.C, nullptr);
    k_bwd_dq<TQ, TG><<<dim3(cdiv(a.K, KT_BWD), a.BH), NT, a.smk, cudaStreamTailLaunch>>>(
        a.q, a.k, a.v, a.g, a.dO, a.h0, a.dPws, a.dq, a.dq32, a.ST, a.T, a.K, a.V, a.C, nullptr);
    k_bwd_dk<TQ, TG><<<dim3(cdiv(a.K, KT_BWD), a.BH), NT, a.smk, cudaStreamTailLaunch>>>(
        a.q, a.k, a.v, a.g, a.dO, a.dfinal, a.dPws, a.dq32, a.ST, a.dk, a.dg, a.dh0, a.T, a.K, a.V, a.C, nullptr);
    k_bwd_dv<TQ, TG><<<dim3(cdiv(a.V, VT_FWD), a.BH), NT, a.smv, cudaStreamTailLaunch>>>(
        a.q, a.k, a.g, a.dO, a.dfinal, a.Pws, a.dv, nullptr, a.T, a.K, a.V, a.C, 0, nullptr);
}

template <typename TQ, typename TG>
static cudaError_t bwd_impl(const BwdProblem& p, cudaStream_t st) {
    const int BH = p.B * p.H, NC = p.T / p.C;
    const size_t nP = (size_t)BH * p.T * p.C;
    float* Pws = (float*)p.ws;
    float* dPws = Pws + nP;
    float* dq32 = dPws + nP;
    float* ST = dq32 + (size_t)BH * p.T * p.K;
    const TQ* q = (const TQ*)p.q; const TQ* k = (const TQ*)p.k; const TQ* v = (const TQ*)p.v;
    const TG* g = (const TG*)p.g; const TQ* dO = (const TQ*)p.dO;
    if (p.mode == 1) {   // dstate summary: dH_0 with dfinal = 0
        const size_t sm = fwd_state_smem(p.C, p.K);
        cudaError_t e = set_smem(k_bwd_dv<TQ, TG>, sm);
        if (e != cudaSuccess) return e;
        {
            GLA_PROF("simt::k_bwd_dv", st);
            k_bwd_dv<TQ, TG><<<dim3(cdiv(p.V, VT_FWD), BH), NT, sm, st>>>(q, k, g, dO, nullptr, nullptr, nullptr,
                                                                         p.dh0, p.T, p.K, p.V, p.C, 1, nullptr);
        }
        return cudaGetLastError();
    }
    const size_t smk = bwd_k_smem(p.C, p.V);
    cudaError_t e = set_smem(k_bwd_dq<TQ, TG>, smk);
    if (e != cudaSuccess) return e;
    e = set_smem(k_bwd_dk<TQ, TG>, smk);
    if (e != cudaSuccess) return e;
    const size_t smv = fwd_state_smem(p.C, p.K);
    e = set_smem(k_bwd_dv<TQ, TG>, smv);
    if (e != cudaSuccess) return e;
    BwdArgs<TQ, TG> a{q, k, v, g, dO, p.h0, p.dfinal, Pws, dPws, dq32, ST, (TQ*)p.dq, (TQ*)p.dk, (TQ*)p.dv, p.dg,
                      p.dh0, p.T, p.K, p.V, p.C, p.c, BH, NC, smk, smv};
    if (p.run_if) {   // gated exact fallback: one tiny launch; the five kernels are tail-launched only if flagged
        GLA_PROF("simt::bwd_gate", st);
        k_bwd_gate<TQ, TG><<<1, 32, 0, st>>>(a, p.run_if);
        return cudaGetLastError();
    }
    {
        GLA_PROF("simt::k_intra_P", st);
        k_intra_P<TQ, TG><<<dim3(NC, BH), NT, 0, st>>>(q, k, g, Pws, p.T, p.K, p.C, p.c, nullptr);
    }
    {
        GLA_PROF("simt::k_intra_dP", st);
        k_intra_dP<TQ><<<dim3(NC, BH), NT, 0, st>>>(dO, v, dPws, p.T, p.V, p.C, nullptr);
    }
    {
        GLA_PROF("simt::k_bwd_dq", st);
        k_bwd_dq<TQ, TG><<<dim3(cdiv(p.K, KT_BWD), BH), NT, smk, st>>>(q, k, v, g, dO, p.h0, dPws, (TQ*)p.dq, dq32,
                                                                      ST, p.T, p.K, p.V, p.C, nullptr, p.colD,
                                                                      simt_tiles());
    }
    {
        GLA_PROF("simt::k_bwd_dk", st);
        k_bwd_dk<TQ, TG><<<dim3(cdiv(p.K, KT_BWD), BH), NT, smk, st>>>(q, k, v, g, dO, p.dfinal, dPws, dq32, ST,
                                                                      (TQ*)p.dk, p.dg, p.dh0, p.T, p.K, p.V, p.C, nullptr,
                                                                      p.colD, simt_tiles());
    }
    {
        GLA_PROF("simt::k_bwd_dv", st);
        k_bwd_dv<TQ, TG><<<dim3(cdiv(p.V, VT_FWD), BH), NT, smv, st>>>(q, k, g, dO, p.dfinal, Pws, (TQ*)p.dv,
                                                                      nullptr, p.T, p.K, p.V, p.C, 0, nullptr, p.colD,
                                                                      simt_tiles());
    }
    return cudaGetLastError();
}

#define GLA_DISPATCH(QT, GT, FN, ...)                                                         \
    do {                                                                                      \
        if ((QT) == 1 && (GT) == 1) return FN<float, float>(__VA_ARGS__);                     \
        if ((QT) == 1 && (GT) == 0) return FN<float, __nv_bfloat16>(__VA_ARGS__);             \
        if ((QT) == 0 && (GT) == 1) return FN<__nv_bfloat16, float>(__VA_ARGS__);             \
        return FN<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__);                                 \
    } while (0)

cudaError_t fwd(const Problem& p, cudaStream_t st) { GLA_DISPATCH(p.qkv_dtype, p.gate_dtype, fwd_impl, p, st); }
cudaError_t bwd(const BwdProblem& p, cudaStream_t st) { GLA_DISPATCH(p.qkv_dtype, p.gate_dtype, bwd_impl, p, st); }

template <typename TQ, typename TG>
static cudaError_t step_impl(int BH, int K, int V, const void* q, const void* k, const void* v, const void* g,
                             float* state, void* out, cudaStream_t st) {
    {
        GLA_PROF("simt::k_step", st);
        // (measured: the 16-column tiles also for up to 4x148 units were equal at B = 16, slower beyond)
        if ((long)BH * cdiv(V, 32) <= 148 && K <= 8 * 32)   // very few units (B = 1 decode): 16-column tiles and
            // one batch of 8 rows per thread, so each thread's state traffic is one round trip to HBM
            k_step<TQ, TG, 4, 32><<<dim3(cdiv(V, 16), BH), 128, 0, st>>>((const TQ*)q, (const TQ*)k, (const TQ*)v,
                                                                       (const TG*)g, state, (TQ*)out, K, V);
        else if ((long)BH * cdiv(V, 128) < 2 * 148)   // few units: narrow tiles, more CTAs
            k_step<TQ, TG, 8, 16><<<dim3(cdiv(V, 32), BH), 128, 0, st>>>((const TQ*)q, (const TQ*)k, (const TQ*)v,
                                                                       (const TG*)g, state, (TQ*)out, K, V);
        else
            k_step<TQ, TG, 32, 8><<<dim3(cdiv(V, 128), BH), 256, 0, st>>>((const TQ*)q, (const TQ*)k, (const TQ*)v,
                                                                        (const TG*)g, state, (TQ*)out, K, V);
    }
    return cudaGetLastError();
}
cudaError_t step(int BH, int K, int V, int qt, int gt, const void* q, const void* k, const void* v,
                 const void* g, float* state, void* out, cudaStream_t st) {
    GLA_DISPATCH(qt, gt, step_impl, BH, K, V, q, k, v, g, state, out, st);
}

cudaError_t combine(int BH, int K, int V, const float* Hin, const float* D, const float* S, float* Hout,
                    cudaStream_t st) {
    const size_t n = (size_t)BH * K * V;
    const int blocks = (int)std::min<size_t>((n + 255) / 256, 148 * 16);
    {
        GLA_PROF("simt::k_combine", st);
        k_combine<<<blocks, 256, 0, st>>>(Hin, D, S, Hout, BH, K, V);
    }
    return cudaGetLastError();
}

bool plan_ok(int C, int K, int V) {
    return C >= 1 && C <= MAXC && fwd_state_smem(C, K) <= 232448 && bwd_k_smem(C, V) <= 232448;
}

size_t fwd_ws(int B, int H, int T, int K, int V, int C) { return sizeof(float) * (size_t)B * H * T * C; }
size_t bwd_ws(int B, int H, int T, int K, int V, int C) {
    return sizeof(float) * ((size_t)2 * B * H * T * C + (size_t)B * H * T * K + (size_t)B * H * K * V);
}

}  // namespace simt
}  // namespace gla
