// simt_beta.cu -- the general outer-product gate G_t = alpha_t^T beta_t on the fp32 CUDA-core path.
//
// The value-side gate enters the chunk-wise algorithm through the paper's own rescaling (Eq. gla_QKV2, P:224-227:
// V~ = V / B, O = O~ (.) B, B_t = prod_{j<=t} beta_j), applied chunk by chunk with a per-chunk, per-value-column
// normaliser so that every factor stays in range (the same device the paper's secondary chunking uses on the
// key side).  Per chunk i (rows [iC, iC+C)), value column v, with c_t = chunk-local inclusive cumsum
// of log beta, r_i = c at the chunk's middle row, Delta_i = c at its last row (r_{T/C} := 0):
//     v~_t = v_t e^{r_i - c_t},   E_t = e^{c_t - r_i},   H'_i = S_{iC} (.)_col e^{r_i}
// then the alpha-only chunk-wise recurrence of simt.cu runs unchanged on (q, k, v~, log alpha) except that each
// chunk's state update is followed by the column decay colD_i = e^{Delta_i - r_i + r_{i+1}} (<= 1):
//     H'_{i+1} = colD_i (.)_col ( diag(e^{Gamma_i}) H'_i + (K_i (.) e^{Gamma_i - b})^T V~_i ),
//     o_t = E_t (.) o~_t,   final_state = H'_{T/C},   H'_0 = h0 (.)_col e^{r_0}.
// (Unfold: o_t = sum_s [q_t (.) e^{b_t - b_s} k_s] (v_s (.) e^{c_t - c_s}) + cross-chunk terms with the state's
// column factor e^{LB}: exactly the recurrence S_t = G_t (.) S_{t-1} + k_t^T v_t of P:188.)
// Backward: the alpha-only backward on (q, k, v~, log alpha, dO~ = E (.) dO) with the same column decays gives dq,
// dk, d log alpha (its identity is untouched: alpha enters only through q e^{LA}, k e^{-LA}), dv~ and dH'_0; then
// dv = dv~ (.) e^{r - c}, d_initial_state = dH'_0 (.)_col e^{r_0}, and, by the symmetric identity on the value side
// (o depends on (v, log beta) only through v (.) e^{-LB} and the output factor e^{LB}),
//     d log beta_t = sum_{s >= t} (o_s (.) do_s - v_s (.) dv_s) + colsum(S_T (.) dS_T)     (pinned in the oracle tests)
// Range: the factors e^{+-(c - r)} are bounded by the half-chunk log decay of beta, which must stay below ~60
// (fp32); with the paper's gates (logsigmoid / 16) it is ~2 at C = 64.
// Everything runs in fp32 (bf16 inputs are widened exactly); fixed reduction orders, no atomics.
#include <algorithm>

#include "common.cuh"
#include "prof.h"
#include "simt.h"

namespace gla {
namespace simt {

namespace {
constexpr int NTB = 256;
inline int cdivb(size_t a, int b) { return (int)((a + b - 1) / b); }

template <typename T>
__global__ void k_widen(const T* __restrict__ x, float* __restrict__ y, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] = to_f(x[i]);
}

// One thread per (bh, value column v): walks the chunks in order (loads coalesced across v).
template <typename TQ, typename TG>
__global__ void k_beta_prep(const TQ* __restrict__ v, const TG* __restrict__ lb, const float* __restrict__ h0,
                            float* __restrict__ vt, float* __restrict__ E, float* __restrict__ colD,
                            float* __restrict__ h0p, float* __restrict__ r0, int BH, int T, int K, int V, int C) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)BH * V) return;
    const int bh = (int)(idx / V), j = (int)(idx % V), NC = T / C, mid = (C - 1) / 2;
    float r_prev = 0.f, D_prev = 0.f;
    for (int i = 0; i < NC; ++i) {
        const size_t row0 = (size_t)bh * T + (size_t)i * C;
        float c = 0.f, r = 0.f;
        for (int t = 0; t < C; ++t) {       // r = c at the middle row
            c += to_f(lb[(row0 + t) * V + j]);
            if (t == mid) r = c;
        }
        c = 0.f;
        for (int t = 0; t < C; ++t) {
            const size_t e = (row0 + t) * V + j;
            c += to_f(lb[e]);
            vt[e] = to_f(v[e]) * expf(r - c);
            E[e] = expf(c - r);
        }
        if (i > 0) colD[((size_t)bh * NC + i - 1) * V + j] = expf(D_prev - r_prev + r);
        else r0[idx] = r;
        r_prev = r;
        D_prev = c;
    }
    if (NC > 0) colD[((size_t)bh * NC + NC - 1) * V + j] = expf(D_prev - r_prev);
    if (h0p) {
        const float f = NC > 0 ? expf(r0[idx]) : 1.f;
        for (int m = 0; m < K; ++m) {
            const size_t e = ((size_t)bh * K + m) * V + j;
            h0p[e] = h0 ? h0[e] * f : 0.f;
        }
    }
}

// y = a (.) b (fp32), optionally also written rounded to TQ.
template <typename TQ>
__global__ void k_mul(const float* __restrict__ a, const float* __restrict__ b, float* __restrict__ y32,
                      TQ* __restrict__ y, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float x = a[i] * b[i];
        if (y32) y32[i] = x;
        if (y) y[i] = from_f<TQ>(x);
    }
}
template <typename TQ>
__global__ void k_mul_in(const float* __restrict__ a, const TQ* __restrict__ b, float* __restrict__ y, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] = a[i] * to_f(b[i]);
}
// dv = dv~ / E  (= dv~ (.) e^{r - c})
template <typename TQ>
__global__ void k_div(const float* __restrict__ a, const float* __restrict__ E, float* __restrict__ y32,
                      TQ* __restrict__ y, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const float x = a[i] / E[i];
        y32[i] = x;
        y[i] = from_f<TQ>(x);
    }
}
template <typename TQ>
__global__ void k_narrow(const float* __restrict__ x, TQ* __restrict__ y, size_t n) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        y[i] = from_f<TQ>(x[i]);
}
// d_initial_state = dH'_0 (.)_col e^{r_0}
__global__ void k_dh0_col(const float* __restrict__ dh0p, const float* __restrict__ r0, float* __restrict__ dh0,
                          int BH, int K, int V) {
    const size_t n = (size_t)BH * K * V;
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const size_t bh = i / ((size_t)K * V);
        dh0[i] = dh0p[i] * expf(r0[bh * V + i % V]);
    }
}
// d log beta_t = sum_{s>=t} (o_s do_s - v_s dv_s) + colsum(S_T (.) dS_T): one thread per (bh, v), reverse
// over the tokens (coalesced across v).
template <typename TQ>
__global__ void k_dlog_beta(const float* __restrict__ o32, const TQ* __restrict__ dO, const TQ* __restrict__ v,
                            const float* __restrict__ dv32, const float* __restrict__ ST,
                            const float* __restrict__ dfinal, float* __restrict__ dlb, int BH, int T, int K, int V) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)BH * V) return;
    const int bh = (int)(idx / V), j = (int)(idx % V);
    float run = 0.f;
    if (dfinal)
        for (int m = 0; m < K; ++m) {
            const size_t e = ((size_t)bh * K + m) * V + j;
            run += ST[e] * dfinal[e];
        }
    for (int t = T - 1; t >= 0; --t) {
        const size_t e = ((size_t)bh * T + t) * V + j;
        run += o32[e] * to_f(dO[e]) - to_f(v[e]) * dv32[e];
        dlb[e] = run;
    }
}
// Decode step with both gates: state <- (alpha^T beta) (.) state + k^T v; o = q state.  One thread per (bh, v).
template <typename TQ, typename TG>
__global__ void k_step_beta(const TQ* __restrict__ q, const TQ* __restrict__ k, const TQ* __restrict__ v,
                            const TG* __restrict__ la, const TG* __restrict__ lb, float* __restrict__ state,
                            TQ* __restrict__ out, int BH, int K, int V) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)BH * V) return;
    const int bh = (int)(idx / V), j = (int)(idx % V);
    const float b = expf(to_f(lb[idx])), vj = to_f(v[idx]);
    float o = 0.f;
    for (int m = 0; m < K; ++m) {
        const size_t e = ((size_t)bh * K + m) * V + j;
        const float s = expf(to_f(la[(size_t)bh * K + m])) * b * state[e] + to_f(k[(size_t)bh * K + m]) * vj;
        state[e] = s;
        o += to_f(q[(size_t)bh * K + m]) * s;
    }
    out[idx] = from_f<TQ>(o);
}

// Workspace carve-up (fp32 words).
struct BetaWs {
    float *q32, *k32, *vt, *E, *colD, *r0, *h0p, *o32, *dO32, *dq32, *dk32, *dvt, *dv32, *dh0p, *ST;
    void* inner;   // alpha-only scratch (fwd / bwd)
};
size_t beta_words(int B, int H, int T, int K, int V, int C) {
    const size_t BH = (size_t)B * H, rows = BH * T, NC = C > 0 ? T / C : 0;
    return 2 * rows * K + 2 * rows * V + BH * NC * V + BH * V + BH * K * V + rows * V + rows * V + 2 * rows * K +
           2 * rows * V + 2 * BH * K * V + 64;
}
BetaWs carve(void* ws, int B, int H, int T, int K, int V, int C) {
    const size_t BH = (size_t)B * H, rows = BH * T, NC = T / C;
    float* w = (float*)ws;
    BetaWs b{};
    auto take = [&](size_t n) { float* p = w; w += (n + 3) & ~size_t(3); return p; };
    b.q32 = take(rows * K); b.k32 = take(rows * K); b.vt = take(rows * V); b.E = take(rows * V);
    b.colD = take(BH * NC * V); b.r0 = take(BH * V); b.h0p = take(BH * K * V); b.o32 = take(rows * V);
    b.dO32 = take(rows * V); b.dq32 = take(rows * K); b.dk32 = take(rows * K); b.dvt = take(rows * V);
    b.dv32 = take(rows * V); b.dh0p = take(BH * K * V); b.ST = take(BH * K * V);
    b.inner = (void*)w;
    return b;
}
}  // namespace

size_t beta_ws(int B, int H, int T, int K, int V, int C) {
    const size_t inner = std::max(fwd_ws(B, H, T, K, V, C), bwd_ws(B, H, T, K, V, C));
    return beta_words(B, H, T, K, V, C) * sizeof(float) + inner + 256;
}

template <typename TQ, typename TG>
static cudaError_t beta_prologue(const BetaProblem& p, BetaWs& w, cudaStream_t st) {
    const int BH = p.B * p.H;
    const size_t rows = (size_t)BH * p.T, nK = rows * p.K;
    const int gb = (int)std::min<size_t>(cdivb(nK, NTB), 148 * 16);
    {
        GLA_PROF("simt::beta_prep", st);
        if (p.qkv_dtype == 0) {   // widen bf16 q, k once (exact)
            k_widen<TQ><<<gb, NTB, 0, st>>>((const TQ*)p.q, w.q32, nK);
            k_widen<TQ><<<gb, NTB, 0, st>>>((const TQ*)p.k, w.k32, nK);
        }
        k_beta_prep<TQ, TG><<<cdivb((size_t)BH * p.V, NTB), NTB, 0, st>>>(
            (const TQ*)p.v, (const TG*)p.lb, p.h0, w.vt, w.E, w.colD, w.h0p, w.r0, BH, p.T, p.K, p.V, p.C);
    }
    return cudaGetLastError();
}

static Problem inner_fwd(const BetaProblem& p, const BetaWs& w) {
    Problem f{};
    f.B = p.B; f.H = p.H; f.T = p.T; f.K = p.K; f.V = p.V; f.C = p.C; f.c = p.c;
    f.qkv_dtype = 1; f.gate_dtype = p.gate_dtype; f.mode = 0;
    f.q = p.qkv_dtype == 0 ? (const void*)w.q32 : p.q;
    f.k = p.qkv_dtype == 0 ? (const void*)w.k32 : p.k;
    f.v = w.vt; f.g = p.g; f.h0 = w.h0p; f.out = w.o32; f.ws = w.inner; f.colD = w.colD;
    return f;
}

template <typename TQ, typename TG>
static cudaError_t fwd_beta_impl(const BetaProblem& p, cudaStream_t st) {
    BetaWs w = carve(p.ws, p.B, p.H, p.T, p.K, p.V, p.C);
    cudaError_t e = beta_prologue<TQ, TG>(p, w, st);
    if (e != cudaSuccess) return e;
    Problem f = inner_fwd(p, w);
    f.final_state = p.final_state;
    if ((e = fwd(f, st)) != cudaSuccess) return e;
    const size_t nV = (size_t)p.B * p.H * p.T * p.V;
    {
        GLA_PROF("simt::beta_out", st);
        k_mul<TQ><<<(int)std::min<size_t>(cdivb(nV, NTB), 148 * 16), NTB, 0, st>>>(w.E, w.o32, nullptr, (TQ*)p.out, nV);
    }
    return cudaGetLastError();
}

template <typename TQ, typename TG>
static cudaError_t bwd_beta_impl(const BetaBwdProblem& p, cudaStream_t st) {
    const BetaProblem& fp = p.f;
    BetaWs w = carve(fp.ws, fp.B, fp.H, fp.T, fp.K, fp.V, fp.C);
    cudaError_t e = beta_prologue<TQ, TG>(fp, w, st);
    if (e != cudaSuccess) return e;
    const int BH = fp.B * fp.H;
    const size_t rows = (size_t)BH * fp.T, nV = rows * fp.V, nK = rows * fp.K;
    const int gV = (int)std::min<size_t>(cdivb(nV, NTB), 148 * 16), gK = (int)std::min<size_t>(cdivb(nK, NTB), 148 * 16);
    // forward (o and S_T feed d log beta)
    Problem f = inner_fwd(fp, w);
    f.final_state = w.ST;
    if ((e = fwd(f, st)) != cudaSuccess) return e;
    {
        GLA_PROF("simt::beta_out", st);
        k_mul<TQ><<<gV, NTB, 0, st>>>(w.E, w.o32, w.o32, (TQ*)nullptr, nV);    // o = E (.) o~ (fp32, in place)
        k_mul_in<TQ><<<gV, NTB, 0, st>>>(w.E, (const TQ*)p.dO, w.dO32, nV);      // dO~ = E (.) dO
    }
    BwdProblem b{};
    b.B = fp.B; b.H = fp.H; b.T = fp.T; b.K = fp.K; b.V = fp.V; b.C = fp.C; b.c = fp.c;
    b.qkv_dtype = 1; b.gate_dtype = fp.gate_dtype; b.mode = 0;
    b.q = f.q; b.k = f.k; b.v = w.vt; b.g = fp.g; b.dO = w.dO32; b.h0 = w.h0p; b.dfinal = p.dfinal;
    b.dq = w.dq32; b.dk = w.dk32; b.dv = w.dvt; b.dg = p.dg; b.dh0 = w.dh0p; b.ws = w.inner; b.colD = w.colD;
    if ((e = bwd(b, st)) != cudaSuccess) return e;
    {
        GLA_PROF("simt::beta_post", st);
        k_narrow<TQ><<<gK, NTB, 0, st>>>(w.dq32, (TQ*)p.dq, nK);
        k_narrow<TQ><<<gK, NTB, 0, st>>>(w.dk32, (TQ*)p.dk, nK);
        k_div<TQ><<<gV, NTB, 0, st>>>(w.dvt, w.E, w.dv32, (TQ*)p.dv, nV);
        if (p.dh0) {
            const size_t nS = (size_t)BH * fp.K * fp.V;
            k_dh0_col<<<(int)std::min<size_t>(cdivb(nS, NTB), 148 * 16), NTB, 0, st>>>(w.dh0p, w.r0, p.dh0, BH,
                                                                                      fp.K, fp.V);
        }
        k_dlog_beta<TQ><<<cdivb((size_t)BH * fp.V, NTB), NTB, 0, st>>>(w.o32, (const TQ*)p.dO, (const TQ*)fp.v,
                                                                      w.dv32, w.ST, p.dfinal, p.dlb, BH, fp.T,
                                                                      fp.K, fp.V);
    }
    return cudaGetLastError();
}

template <typename TQ, typename TG>
static cudaError_t step_beta_impl(int BH, int K, int V, const void* q, const void* k, const void* v,
                                  const void* la, const void* lb, float* state, void* out, cudaStream_t st) {
    {
        GLA_PROF("simt::k_step_beta", st);
        k_step_beta<TQ, TG><<<cdivb((size_t)BH * V, 128), 128, 0, st>>>((const TQ*)q, (const TQ*)k, (const TQ*)v,
                                                                     (const TG*)la, (const TG*)lb, state, (TQ*)out,
                                                                     BH, K, V);
    }
    return cudaGetLastError();
}

#define GLA_BDISPATCH(QT, GT, FN, ...)                                                        \
    do {                                                                                      \
        if ((QT) == 1 && (GT) == 1) return FN<float, float>(__VA_ARGS__);                     \
        if ((QT) == 1 && (GT) == 0) return FN<float, __nv_bfloat16>(__VA_ARGS__);             \
        if ((QT) == 0 && (GT) == 1) return FN<__nv_bfloat16, float>(__VA_ARGS__);             \
        return FN<__nv_bfloat16, __nv_bfloat16>(__VA_ARGS__);                                 \
    } while (0)

cudaError_t fwd_beta(const BetaProblem& p, cudaStream_t st) {
    GLA_BDISPATCH(p.qkv_dtype, p.gate_dtype, fwd_beta_impl, p, st);
}
cudaError_t bwd_beta(const BetaBwdProblem& p, cudaStream_t st) {
    GLA_BDISPATCH(p.f.qkv_dtype, p.f.gate_dtype, bwd_beta_impl, p, st);
}
cudaError_t step_beta(int BH, int K, int V, int qt, int gt, const void* q, const void* k, const void* v,
                      const void* la, const void* lb, float* state, void* out, cudaStream_t st) {
    GLA_BDISPATCH(qt, gt, step_beta_impl, BH, K, V, q, k, v, la, lb, state, out, st);
}

}  // namespace simt
}  // namespace gla
