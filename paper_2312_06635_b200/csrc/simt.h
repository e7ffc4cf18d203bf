// simt.h -- host-side interface of the fp32 SIMT kernels (simt.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

namespace gla {

struct Problem {           // forward / state summary
    int B, H, T, K, V, C, c, qkv_dtype, gate_dtype;
    int mode;              // 0 forward, 1 state summary
    const void *q, *k, *v, *g;
    const float* h0;
    void* out;
    float* final_state;
    float* log_decay;
    void* ws;
    const float* colD = nullptr;    // value-gate path only: per-(chunk, value column) state decay (simt_beta.cu)
};

struct BwdProblem {
    int B, H, T, K, V, C, c, qkv_dtype, gate_dtype;
    int mode;              // 0 backward, 1 dstate summary (dh0 only)
    const void *q, *k, *v, *g, *dO;
    const float *h0, *dfinal;
    void *dq, *dk, *dv;
    float *dg, *dh0;
    void* ws;
    const int* run_if;     // device flag: kernels return immediately when *run_if == 0 (nullptr = always run)
    const void* fwd_ws = nullptr;   // workspace of a preceding TC gla_chunk_fwd on the same q, k, log alpha
    const float* colD = nullptr;    // value-gate path only (see Problem)
};

// The general outer-product gate G_t = alpha_t^T beta_t, fp32 CUDA-core path (simt_beta.cu).
struct BetaProblem {
    int B, H, T, K, V, C, c, qkv_dtype, gate_dtype;
    const void *q, *k, *v, *g, *lb;   // lb: log beta [B,H,T,V] (gate_dtype)
    const float* h0;
    void* out;
    float* final_state;
    void* ws;
};
struct BetaBwdProblem {
    BetaProblem f;                    // forward inputs (out / final_state unused)
    const void* dO;
    const float* dfinal;
    void *dq, *dk, *dv;
    float *dg, *dlb, *dh0;
};

namespace simt {
cudaError_t fwd_beta(const BetaProblem& p, cudaStream_t st);
cudaError_t bwd_beta(const BetaBwdProblem& p, cudaStream_t st);
size_t beta_ws(int B, int H, int T, int K, int V, int C);
cudaError_t step_beta(int BH, int K, int V, int qt, int gt, const void* q, const void* k, const void* v,
                      const void* la, const void* lb, float* state, void* out, cudaStream_t st);
cudaError_t fwd(const Problem& p, cudaStream_t st);
cudaError_t bwd(const BwdProblem& p, cudaStream_t st);
cudaError_t step(int BH, int K, int V, int qkv_dtype, int gate_dtype, const void* q, const void* k,
                 const void* v, const void* g, float* state, void* out, cudaStream_t st);
cudaError_t combine(int BH, int K, int V, const float* Hin, const float* D, const float* S, float* Hout,
                    cudaStream_t st);
size_t fwd_ws(int B, int H, int T, int K, int V, int C);
// chunk plan the SIMT kernels can run: C <= 128 and their shared-memory tiles fit (227 KB per CTA)
bool plan_ok(int C, int K, int V);
size_t bwd_ws(int B, int H, int T, int K, int V, int C);
}  // namespace simt
}  // namespace gla
