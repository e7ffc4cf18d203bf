// layer.cu -- the elementwise parts of a full multi-head GLA layer around the chunk-wise core (
// P:298-307 multi-head GLA layer, P:321-326 low-rank gate):
//   q, k, v, r_pre, z_alpha = projections of x (cuBLAS GEMMs, outside this file)
//   log alpha = logsigmoid(z_alpha + b_alpha) / tau            (P:177 footnote: tau = 16)
//   O^h       = GLA core (q^h, k^h, v^h, alpha^h)              (the tensor-core kernels)
//   Z         = concat_h(LN(O^h)) (.) Swish(r_pre + b_r)      (per-head LayerNorm as in RetNet,
//                                                              per-channel affine ln_w, ln_b)
//   y         = Z W_O                                          (cuBLAS GEMM, outside)
// Layouts: projection output P [B*T][ldP] bf16 with column blocks [q (H*K) | k (H*K) | v (H*V) | r (H*V)],
// z_alpha [B*T][H*K] bf16; the core's tensors are [B,H,T,D] (the prep kernel transposes; the output kernel
// transposes back).  One warp per (row, head) in the row kernels; the parameter gradients are per-CTA fp32
// partials summed in a fixed order by k_sum_partials (deterministic, no atomics).
#include <cuda_bf16.h>

#include <initializer_list>

#include "common.cuh"
#include "prof.h"
#include "tc_build.cuh"

namespace gla {
namespace layer {

namespace {
__device__ __forceinline__ float logsigmoid(float z) { return fminf(z, 0.f) - log1pf(__expf(-fabsf(z))); }
// fast reciprocal (MUFU.RCP): the IEEE division was a third of out_bwd's stall samples; 1 / inf -> 0 for z -> -inf
__device__ __forceinline__ float sigmoid(float z) { return __fdividef(1.f, 1.f + __expf(-z)); }

__device__ __forceinline__ void ld8(const __nv_bfloat16* p, float (&x)[8]) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) { x[2 * i] = tc::bf16lo(w[i]); x[2 * i + 1] = tc::bf16hi(w[i]); }
}
__device__ __forceinline__ void ldf8(const float* p, float (&x)[8]) {   // 8 fp32 parameters, two 16-B loads
    const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p + 4));
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
}
// 8 parameters from shared memory (SP) or global memory
template <bool SP>
__device__ __forceinline__ void ldp8(const float* p, float (&x)[8]) {
    if (SP) {
        const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    } else {
        ldf8(p, x);
    }
}
// CTA-cooperative copy of the three n-float parameter vectors into shared memory [3][n] (n % 4 == 0), then a barrier
__device__ __forceinline__ void stage_params(float* s, const float* a, const float* b, const float* c, int n) {
    for (int i = threadIdx.x; i < 3 * n / 4; i += blockDim.x) {
        const int v = i / (n / 4), j = i - v * (n / 4);
        const float* src = v == 0 ? a : (v == 1 ? b : c);
        reinterpret_cast<float4*>(s)[i] = __ldg(reinterpret_cast<const float4*>(src) + j);
    }
    __syncthreads();
}
__device__ __forceinline__ void st8(__nv_bfloat16* p, const float (&x)[8]) {
    *reinterpret_cast<uint4*>(p) = make_uint4(tc::pack_bf16(x[0], x[1]), tc::pack_bf16(x[2], x[3]),
                                              tc::pack_bf16(x[4], x[5]), tc::pack_bf16(x[6], x[7]));
}
}  // namespace

// ---- forward prep: P, z_alpha -> q, k, v [B,H,T,.] (bf16), log alpha [B,H,T,K] (fp32) ---------------------------
// One thread per 8 consecutive elements of a row; the vector index space of a row is q | k | v | gate.
template <typename I>   // index type: 32-bit when the element count allows (cheaper divisions)
__global__ void k_prep(const __nv_bfloat16* __restrict__ P, int ldP, const __nv_bfloat16* __restrict__ Za,
                       const float* __restrict__ b_alpha, __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                       __nv_bfloat16* __restrict__ v, float* __restrict__ g, int B, int T, int H, int K, int V,
                       float inv_tau) {
    const int HK = H * K, HV = H * V, nvec = (3 * HK + HV) / 8;
    const I total = (I)B * T * nvec;
    for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
        const I row = i / nvec;                          // b * T + t
        const int c = 8 * (int)(i - row * nvec);
        const int b = (int)(row / T), t = (int)(row - (I)b * T);
        float x[8];
        if (c < 2 * HK + HV) {                           // q | k | v: transpose to [B,H,T,D]
            ld8(P + row * ldP + c, x);
            const bool isv = c >= 2 * HK;
            const int cc = isv ? c - 2 * HK : c % HK, D = isv ? V : K;
            const int h = cc / D, e = cc % D;
            __nv_bfloat16* dst = isv ? v : (c < HK ? q : k);
            st8(dst + (((size_t)b * H + h) * T + t) * D + e, x);
        } else {                                         // gate: log alpha = logsigmoid(z + b_alpha) / tau
            const int cc = c - 2 * HK - HV, h = cc / K, e = cc % K;
            ld8(Za + row * HK + cc, x);
            float y[8], ba[8];
            ldf8(b_alpha + cc, ba);
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = logsigmoid(x[j] + ba[j]) * inv_tau;
            float4* o = reinterpret_cast<float4*>(g + (((size_t)b * H + h) * T + t) * K + e);
            o[0] = make_float4(y[0], y[1], y[2], y[3]);
            o[1] = make_float4(y[4], y[5], y[6], y[7]);
        }
    }
}

// ---- forward output: Z = LN_h(O) * ln_w + ln_b, times Swish(r_pre + b_r); saves mean, rstd per (row, head) -----
// One warp per (row, head): lane l owns the 8-element chunks l, l + 32, ... of the head's V values.
// SP: the per-column parameters (b_r, ln_w, ln_b: 3 H V floats) are staged once per CTA in shared memory (their
// global loads sat on every item's critical path).
template <int NCH, bool SP>   // chunks of 8 per lane: V = 256 * NCH
__global__ void k_out(const __nv_bfloat16* __restrict__ O, const __nv_bfloat16* __restrict__ P, int ldP, int r_off,
                      const float* __restrict__ b_r, const float* __restrict__ ln_w, const float* __restrict__ ln_b,
                      __nv_bfloat16* __restrict__ Z, float* __restrict__ mean_out, float* __restrict__ rstd_out,
                      int B, int T, int H, int V, float eps) {
    extern __shared__ float4 sparam4[];
    float* sparam = reinterpret_cast<float*>(sparam4);
    if (SP) {
        stage_params(sparam, b_r, ln_w, ln_b, H * V);
        b_r = sparam; ln_w = sparam + H * V; ln_b = sparam + 2 * H * V;
    }
    const int lane = threadIdx.x & 31;
    const int nw = B * T * H;   // (row, head) items; B*T*H < 2^31 (checked by the caller's shapes)
    for (int w = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5); w < nw; w += (int)((gridDim.x * blockDim.x) >> 5)) {
        const int row = w / H, h = w - row * H, b = row / T, t = row - b * T;
        const __nv_bfloat16* o = O + (((size_t)b * H + h) * T + t) * V;
        float x[NCH][8], rp[NCH][8], s = 0.f;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {   // both rows' loads issued before any use (one memory latency per item)
            ld8(o + 8 * (lane + 32 * c), x[c]);
            ld8(P + (size_t)row * ldP + r_off + h * V + 8 * (lane + 32 * c), rp[c]);
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int j = 0; j < 8; ++j) s += x[c][j];
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        const float mu = s / V;
        float q2 = 0.f;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
#pragma unroll
            for (int j = 0; j < 8; ++j) { const float d = x[c][j] - mu; q2 += d * d; }
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) q2 += __shfl_xor_sync(0xffffffffu, q2, m);
        const float rs = rsqrtf(q2 / V + eps);
        if (lane == 0) { mean_out[w] = mu; rstd_out[w] = rs; }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int e = 8 * (lane + 32 * c), col = h * V + e;
            float z[8], br[8], lw[8], lb[8];
            ldp8<SP>(b_r + col, br);
            ldp8<SP>(ln_w + col, lw);
            ldp8<SP>(ln_b + col, lb);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float r = rp[c][j] + br[j];
                z[j] = ((x[c][j] - mu) * rs * lw[j] + lb[j]) * (r * sigmoid(r));
            }
            st8(Z + (size_t)row * (H * V) + col, z);
        }
    }
}

// ---- backward of the output: dZ -> dO [B,H,T,V] (bf16), d r_pre into dP's r block (bf16), parameter partials ---
// part[3][gridDim.x][H*V]: d ln_w, d ln_b, d b_r, accumulated over this CTA's rows in a fixed order.
template <int NCH, bool SP>
__global__ void k_out_bwd(const __nv_bfloat16* __restrict__ dZ, const __nv_bfloat16* __restrict__ O,
                          const __nv_bfloat16* __restrict__ P, int ldP, int r_off, const float* __restrict__ b_r,
                          const float* __restrict__ ln_w, const float* __restrict__ ln_b,
                          const float* __restrict__ mean_in, const float* __restrict__ rstd_in,
                          __nv_bfloat16* __restrict__ dO, __nv_bfloat16* __restrict__ dP, float* __restrict__ part,
                          int B, int T, int H, int V, int rows_per_cta) {
    // blockDim = 32 * H: warp h handles head h of each of this CTA's rows, the next row's loads in flight while
    // the current row is computed (the kernel is latency-bound otherwise: one row of loads per warp at a time).
    extern __shared__ float4 sparam4[];
    float* sparam = reinterpret_cast<float*>(sparam4);
    if (SP) {   // per-column parameters staged once per CTA (see k_out)
        stage_params(sparam, b_r, ln_w, ln_b, H * V);
        b_r = sparam; ln_w = sparam + H * V; ln_b = sparam + 2 * H * V;
    }
    const int lane = threadIdx.x & 31, h = threadIdx.x >> 5;
    const size_t nrows = (size_t)B * T, HV = (size_t)H * V;
    float aw[NCH][8] = {}, ab[NCH][8] = {}, ar[NCH][8] = {};
    const size_t r0 = (size_t)blockIdx.x * rows_per_cta, r1 = min(nrows, r0 + rows_per_cta);
    uint4 X[NCH], R[NCH], D[NCH];
    float MU = 0.f, RS = 0.f;
    auto load = [&](size_t row) {
        const int b = (int)row / T, t = (int)row - b * T;   // (32-bit: B * T < 2^31)
        const __nv_bfloat16* o = O + (((size_t)b * H + h) * T + t) * V;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int e = 8 * (lane + 32 * c), col = h * V + e;
            X[c] = *reinterpret_cast<const uint4*>(o + e);
            R[c] = *reinterpret_cast<const uint4*>(P + row * ldP + r_off + col);
            D[c] = *reinterpret_cast<const uint4*>(dZ + row * HV + col);
        }
        MU = mean_in[row * H + h];
        RS = rstd_in[row * H + h];
    };
    if (r0 < r1) load(r0);
    for (size_t row = r0; row < r1; ++row) {
        uint4 Xc[NCH], Rc[NCH], Dc[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) { Xc[c] = X[c]; Rc[c] = R[c]; Dc[c] = D[c]; }
        const float mu = MU, rs = RS;
        if (row + 1 < r1) load(row + 1);
        const int b = (int)row / T, t = (int)row - b * T;
        float n[NCH][8], dn[NCH][8], s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int e = 8 * (lane + 32 * c), col = h * V + e;
            const uint32_t xw[4] = {Xc[c].x, Xc[c].y, Xc[c].z, Xc[c].w}, rw[4] = {Rc[c].x, Rc[c].y, Rc[c].z, Rc[c].w},
                           dw[4] = {Dc[c].x, Dc[c].y, Dc[c].z, Dc[c].w};
            float drp[8], br[8], lw[8], lb[8];
            ldp8<SP>(b_r + col, br);
            ldp8<SP>(ln_w + col, lw);
            ldp8<SP>(ln_b + col, lb);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float xj = (j & 1) ? tc::bf16hi(xw[j >> 1]) : tc::bf16lo(xw[j >> 1]);
                const float rj = (j & 1) ? tc::bf16hi(rw[j >> 1]) : tc::bf16lo(rw[j >> 1]);
                const float dzj = (j & 1) ? tc::bf16hi(dw[j >> 1]) : tc::bf16lo(dw[j >> 1]);
                const float r = rj + br[j], sg = sigmoid(r), sw = r * sg;
                n[c][j] = (xj - mu) * rs;
                const float a = n[c][j] * lw[j] + lb[j];
                const float da = dzj * sw;                            // d(LN output after affine)
                drp[j] = dzj * a * sg * (1.f + r * (1.f - sg));       // Swish'(r) = s (1 + r (1 - s))
                aw[c][j] += da * n[c][j];
                ab[c][j] += da;
                ar[c][j] += drp[j];
                dn[c][j] = da * lw[j];
                s1 += dn[c][j];
                s2 += dn[c][j] * n[c][j];
            }
            st8(dP + row * ldP + r_off + col, drp);
        }
#pragma unroll
        for (int m = 16; m > 0; m >>= 1) {
            s1 += __shfl_xor_sync(0xffffffffu, s1, m);
            s2 += __shfl_xor_sync(0xffffffffu, s2, m);
        }
        s1 /= V;
        s2 /= V;
        __nv_bfloat16* d = dO + (((size_t)b * H + h) * T + t) * V;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            float y[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = rs * (dn[c][j] - s1 - n[c][j] * s2);
            st8(d + 8 * (lane + 32 * c), y);
        }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const int col = h * V + 8 * (lane + 32 * c);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            part[((size_t)0 * gridDim.x + blockIdx.x) * HV + col + j] = aw[c][j];
            part[((size_t)1 * gridDim.x + blockIdx.x) * HV + col + j] = ab[c][j];
            part[((size_t)2 * gridDim.x + blockIdx.x) * HV + col + j] = ar[c][j];
        }
    }
}

// ---- backward of the prep: dq, dk, dv, d log alpha -> dP's q | k | v blocks, d z_alpha, d b_alpha partials -------
template <typename I>
__global__ void k_prep_bwd(const __nv_bfloat16* __restrict__ dq, const __nv_bfloat16* __restrict__ dk,
                           const __nv_bfloat16* __restrict__ dv, const float* __restrict__ dg,
                           const __nv_bfloat16* __restrict__ Za, const float* __restrict__ b_alpha,
                           __nv_bfloat16* __restrict__ dP, int ldP, __nv_bfloat16* __restrict__ dZa,
                           int B, int T, int H, int K, int V, float inv_tau) {
    const int HK = H * K, HV = H * V, nvec = (3 * HK + HV) / 8;
    const I total = (I)B * T * nvec;
    for (I i = (I)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (I)gridDim.x * blockDim.x) {
        const I row = i / nvec;
        const int c = 8 * (int)(i - row * nvec);
        const int b = (int)(row / T), t = (int)(row - (I)b * T);
        float x[8];
        if (c < 2 * HK + HV) {
            const bool isv = c >= 2 * HK;
            const int cc = isv ? c - 2 * HK : c % HK, D = isv ? V : K;
            const int h = cc / D, e = cc % D;
            const __nv_bfloat16* src = isv ? dv : (c < HK ? dq : dk);
            ld8(src + (((size_t)b * H + h) * T + t) * D + e, x);
            st8(dP + row * ldP + c, x);
        } else {                                         // d z = d log alpha * sigmoid(-(z + b)) / tau
            const int cc = c - 2 * HK - HV, h = cc / K, e = cc % K;
            ld8(Za + row * HK + cc, x);
            const float4* gi = reinterpret_cast<const float4*>(dg + (((size_t)b * H + h) * T + t) * K + e);
            const float4 g0 = gi[0], g1 = gi[1];
            const float gg[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
            float y[8], ba[8];
            ldf8(b_alpha + cc, ba);
#pragma unroll
            for (int j = 0; j < 8; ++j) y[j] = gg[j] * sigmoid(-(x[j] + ba[j])) * inv_tau;
            st8(dZa + row * HK + cc, y);
        }
    }
}

// out[j] = sum_i part[i][j] over n partials, in order i = 0, 1, ... (deterministic).
__global__ void k_sum_partials(const float* __restrict__ part, float* __restrict__ out, int n, int len) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= len) return;
    float s = 0.f;
    for (int i = 0; i < n; ++i) s += part[(size_t)i * len + j];
    out[j] = s;
}

// d b_alpha partials: column sums of d z_alpha = d log alpha * sigmoid(-(z + b)) / tau over fixed row blocks,
// recomputed in fp32 from d log alpha (not from the bf16-rounded d z_alpha); one CTA per (row block, 256 columns).
__global__ void k_dbalpha_part(const float* __restrict__ dg, const __nv_bfloat16* __restrict__ Za,
                               const float* __restrict__ b_alpha, float* __restrict__ part, int T, int H, int K,
                               size_t nrows, int rows_per_cta, float inv_tau) {
    const int HK = H * K, col = blockIdx.y * blockDim.x + threadIdx.x;
    if (col >= HK) return;
    const int h = col / K, e = col % K;
    const float bb = b_alpha[col];
    const size_t r0 = (size_t)blockIdx.x * rows_per_cta, r1 = min(nrows, r0 + rows_per_cta);
    float s = 0.f;
    size_t b = r0 / T, t = r0 % T;   // (advanced incrementally: no 64-bit division per row)
    for (size_t r = r0; r < r1; ++r) {
        s += dg[((b * H + h) * T + t) * K + e] * sigmoid(-(__bfloat162float(Za[r * HK + col]) + bb)) * inv_tau;
        if (++t == (size_t)T) { t = 0; ++b; }
    }
    part[(size_t)blockIdx.x * HK + col] = s;
}

}  // namespace layer
}  // namespace gla

// ---------------------------------------------------------------------------------------------------------------
// C ABI (include/gla.h "GLA layer")
#include "../../include/gla.h"

namespace gla { void set_last_cuda(int e); }   // api.cu (gla_last_cuda_error)
namespace {
int lstatus(cudaError_t e) { return e == cudaSuccess ? GLA_OK : (gla::set_last_cuda((int)e), GLA_ERR_CUDA); }
bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
int grid_for(size_t work, int threads) {
    const size_t g = (work + threads - 1) / threads;
    return (int)(g < 148 * 32 ? (g > 0 ? g : 1) : 148 * 32);
}
int layer_shape_ok(int B, int T, int H, int K, int V, int ldP) {
    if (B < 0 || T < 0 || H <= 0 || K <= 0 || V <= 0) return GLA_ERR_SHAPE;
    if (K % 8 || V % 256 || V > 1024 || H > 32 || ldP < 2 * H * K + 2 * H * V || ldP % 8) return GLA_ERR_SHAPE;
    return GLA_OK;
}
}  // namespace

extern "C" {

int gla_layer_prep(int B, int T, int H, int K, int V, float tau, const void* P, int ldP, const void* z_alpha,
                   const float* b_alpha, void* q, void* k, void* v, float* log_alpha, void* stream) {
    int s = layer_shape_ok(B, T, H, K, V, ldP);
    if (s) return s;
    if (!(tau > 0.f)) return GLA_ERR_SHAPE;
    for (const void* p : std::initializer_list<const void*>{P, z_alpha, (const void*)b_alpha, q, k, v, (const void*)log_alpha}) {
        if (!p) return GLA_ERR_NULL;
        if (!al16(p)) return GLA_ERR_ALIGN;
    }
    if ((size_t)B * T == 0) return GLA_OK;
    const size_t work = (size_t)B * T * (3 * H * K + H * V) / 8;
    GLA_PROF("layer::prep", (cudaStream_t)stream);
    if (work < (1u << 31))
        gla::layer::k_prep<unsigned><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(
            (const __nv_bfloat16*)P, ldP, (const __nv_bfloat16*)z_alpha, b_alpha, (__nv_bfloat16*)q, (__nv_bfloat16*)k,
            (__nv_bfloat16*)v, log_alpha, B, T, H, K, V, 1.f / tau);
    else
        gla::layer::k_prep<size_t><<<grid_for(work, 256), 256, 0, (cudaStream_t)stream>>>(
            (const __nv_bfloat16*)P, ldP, (const __nv_bfloat16*)z_alpha, b_alpha, (__nv_bfloat16*)q, (__nv_bfloat16*)k,
            (__nv_bfloat16*)v, log_alpha, B, T, H, K, V, 1.f / tau);
    return lstatus(cudaGetLastError());
}

int gla_layer_out(int B, int T, int H, int V, const void* O, const void* P, int ldP, int r_off, const float* b_r,
                  const float* ln_w, const float* ln_b, float eps, void* Z, float* mean, float* rstd, void* stream) {
    if (B < 0 || T < 0 || H <= 0 || H > 32 || V % 256 || V > 1024 || r_off % 8 || ldP % 8 || r_off + H * V > ldP)
        return GLA_ERR_SHAPE;
    for (const void* p : std::initializer_list<const void*>{O, P, (const void*)b_r, (const void*)ln_w, (const void*)ln_b, Z, (const void*)mean,
                          (const void*)rstd}) {
        if (!p) return GLA_ERR_NULL;
        if (!al16(p)) return GLA_ERR_ALIGN;
    }
    if ((size_t)B * T == 0) return GLA_OK;
    const size_t warps = (size_t)B * T * H;
    cudaStream_t st = (cudaStream_t)stream;
    GLA_PROF("layer::out", st);
    // parameters in shared memory when they fit the default 48 KB (then a persistent grid of 4 CTAs per SM, so
    // the per-CTA staging stays small against the data)
    const size_t spb = (size_t)3 * H * V * sizeof(float);
    const bool sp = spb <= 48 * 1024;
    const int grid0 = grid_for(warps * 32, 256), grid = sp && grid0 > 148 * 4 ? 148 * 4 : grid0;
#define GLA_OUT(N) (sp ? gla::layer::k_out<N, true> : gla::layer::k_out<N, false>)<<<grid, 256, sp ? spb : 0, st>>>( \
        (const __nv_bfloat16*)O, (const __nv_bfloat16*)P, ldP, \
        r_off, b_r, ln_w, ln_b, (__nv_bfloat16*)Z, mean, rstd, B, T, H, V, eps)
    switch (V / 256) {
        case 1: GLA_OUT(1); break;
        case 2: GLA_OUT(2); break;
        case 3: GLA_OUT(3); break;
        default: GLA_OUT(4); break;
    }
#undef GLA_OUT
    return lstatus(cudaGetLastError());
}

size_t gla_layer_bwd_workspace_size(int B, int T, int H, int K, int V) {
    (void)K;
    const size_t rows = (size_t)B * T;
    const size_t nblk = rows < 148 * 4 ? (rows > 0 ? rows : 1) : 148 * 4;
    const size_t nb2 = rows < 148 ? (rows > 0 ? rows : 1) : 148;
    return (3 * nblk * (size_t)H * V + nb2 * (size_t)H * K) * sizeof(float) + 256;
}

int gla_layer_out_bwd(int B, int T, int H, int V, const void* dZ, const void* O, const void* P, int ldP, int r_off,
                      const float* b_r, const float* ln_w, const float* ln_b, const float* mean, const float* rstd,
                      void* dO, void* dP, float* d_ln_w, float* d_ln_b, float* d_b_r, void* workspace,
                      size_t workspace_bytes, void* stream) {
    if (B < 0 || T < 0 || H <= 0 || H > 32 || V % 256 || V > 1024 || r_off % 8 || ldP % 8 || r_off + H * V > ldP)
        return GLA_ERR_SHAPE;
    for (const void* p : std::initializer_list<const void*>{dZ, O, P, (const void*)b_r, (const void*)ln_w, (const void*)ln_b, (const void*)mean,
                          (const void*)rstd, dO, dP, (const void*)d_ln_w, (const void*)d_ln_b, (const void*)d_b_r,
                          (const void*)workspace}) {
        if (!p) return GLA_ERR_NULL;
        if (!al16(p)) return GLA_ERR_ALIGN;
    }
    if (workspace_bytes < gla_layer_bwd_workspace_size(B, T, H, 8, V)) return GLA_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t rows = (size_t)B * T, HV = (size_t)H * V;
    if (rows == 0) {
        for (float* o : std::initializer_list<float*>{d_ln_w, d_ln_b, d_b_r})
            if (int r = lstatus(cudaMemsetAsync(o, 0, HV * 4, st))) return r;
        return GLA_OK;
    }
    const int nblk = (int)(rows < 148 * 4 ? rows : 148 * 4);
    const int rpc = (int)((rows + nblk - 1) / nblk);
    float* part = (float*)workspace;
    {
        GLA_PROF("layer::out_bwd", st);
        const size_t spb = (size_t)3 * H * V * sizeof(float);
        const bool sp = spb <= 48 * 1024;
#define GLA_OUTB(N) (sp ? gla::layer::k_out_bwd<N, true> : gla::layer::k_out_bwd<N, false>)<<<nblk, 32 * H, sp ? spb : 0, st>>>((const __nv_bfloat16*)dZ, \
        (const __nv_bfloat16*)O, (const __nv_bfloat16*)P, ldP, r_off, b_r, ln_w, ln_b, mean, rstd, \
        (__nv_bfloat16*)dO, (__nv_bfloat16*)dP, part, B, T, H, V, rpc)
        switch (V / 256) {
            case 1: GLA_OUTB(1); break;
            case 2: GLA_OUTB(2); break;
            case 3: GLA_OUTB(3); break;
            default: GLA_OUTB(4); break;
        }
#undef GLA_OUTB
    }
    float* outs[3] = {d_ln_w, d_ln_b, d_b_r};
    for (int i = 0; i < 3; ++i)
        gla::layer::k_sum_partials<<<(int)((HV + 255) / 256), 256, 0, st>>>(part + (size_t)i * nblk * HV, outs[i], nblk,
                                                                          (int)HV);
    return lstatus(cudaGetLastError());
}

int gla_layer_prep_bwd(int B, int T, int H, int K, int V, float tau, const void* dq, const void* dk, const void* dv,
                       const float* d_log_alpha, const void* z_alpha, const float* b_alpha, void* dP, int ldP,
                       void* d_z_alpha, float* d_b_alpha, void* workspace, size_t workspace_bytes, void* stream) {
    int s = layer_shape_ok(B, T, H, K, V, ldP);
    if (s) return s;
    if (!(tau > 0.f)) return GLA_ERR_SHAPE;
    for (const void* p : std::initializer_list<const void*>{dq, dk, dv, (const void*)d_log_alpha, z_alpha, (const void*)b_alpha, dP, d_z_alpha,
                          (const void*)d_b_alpha, (const void*)workspace}) {
        if (!p) return GLA_ERR_NULL;
        if (!al16(p)) return GLA_ERR_ALIGN;
    }
    if (workspace_bytes < gla_layer_bwd_workspace_size(B, T, H, K, V)) return GLA_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t rows = (size_t)B * T;
    const int HK = H * K;
    if (rows == 0) return lstatus(cudaMemsetAsync(d_b_alpha, 0, (size_t)HK * 4, st));
    const size_t work = rows * (3 * H * K + H * V) / 8;
    {
        GLA_PROF("layer::prep_bwd", st);
        if (work < (1u << 31))
            gla::layer::k_prep_bwd<unsigned><<<grid_for(work, 256), 256, 0, st>>>(
                (const __nv_bfloat16*)dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)dv, d_log_alpha,
                (const __nv_bfloat16*)z_alpha, b_alpha, (__nv_bfloat16*)dP, ldP, (__nv_bfloat16*)d_z_alpha, B, T, H, K,
                V, 1.f / tau);
        else
            gla::layer::k_prep_bwd<size_t><<<grid_for(work, 256), 256, 0, st>>>(
                (const __nv_bfloat16*)dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)dv, d_log_alpha,
                (const __nv_bfloat16*)z_alpha, b_alpha, (__nv_bfloat16*)dP, ldP, (__nv_bfloat16*)d_z_alpha, B, T, H, K,
                V, 1.f / tau);
    }
    const int nb2 = (int)(rows < 148 ? rows : 148);
    const int rpc = (int)((rows + nb2 - 1) / nb2);
    float* part = (float*)workspace;
    gla::layer::k_dbalpha_part<<<dim3(nb2, (HK + 255) / 256), 256, 0, st>>>(
        d_log_alpha, (const __nv_bfloat16*)z_alpha, b_alpha, part, T, H, K, rows, rpc, 1.f / tau);
    gla::layer::k_sum_partials<<<(HK + 255) / 256, 256, 0, st>>>(part, d_b_alpha, nb2, HK);
    return lstatus(cudaGetLastError());
}

}  // extern "C"
