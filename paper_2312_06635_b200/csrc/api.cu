// api.cu -- the C ABI of libgla.so (include/gla.h): validation, path selection, dispatch.
// No compute here: every step of the method runs in the kernels of simt.cu / tc_*.cu.
#include <cuda_runtime.h>

#include <map>
#include <mutex>

#include "../../include/gla.h"
#include "simt.h"
#include "tc.h"

namespace {

thread_local int g_last_cuda = 0;

int cuda_status(cudaError_t e) {
    if (e == cudaSuccess) return GLA_OK;
    g_last_cuda = (int)e;
    return GLA_ERR_CUDA;
}

bool aligned(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool ok_dtype(int d) { return d == GLA_BF16 || d == GLA_FP32; }

int check_desc(const gla_desc* d) {
    if (!d) return GLA_ERR_NULL;
    if (d->B < 0 || d->H < 0 || d->T < 0 || d->K <= 0 || d->V <= 0) return GLA_ERR_SHAPE;
    if (d->K > 256 || d->V > 1024) return GLA_ERR_SHAPE;
    if (!ok_dtype(d->qkv_dtype) || !ok_dtype(d->gate_dtype)) return GLA_ERR_DTYPE;
    if (d->chunk <= 0 || d->subchunk <= 0 || d->chunk > 128) return GLA_ERR_PLAN;
    if (d->T % d->chunk != 0 || d->chunk % d->subchunk != 0) return GLA_ERR_PLAN;
    if (d->path < GLA_PATH_AUTO || d->path > GLA_PATH_TC) return GLA_ERR_UNSUPPORTED;
    // chunks above 64 exist only on the SIMT kernels, within their shared-memory tiles
    if (d->chunk > 64 && (d->path == GLA_PATH_TC || !gla::simt::plan_ok(d->chunk, d->K, d->V))) return GLA_ERR_PLAN;
    return GLA_OK;
}

// Row strides must keep 16-byte alignment of every (b,h,t) row for the vectorised paths.
int check_ptrs(std::initializer_list<const void*> required, std::initializer_list<const void*> optional) {
    for (const void* p : required) {
        if (!p) return GLA_ERR_NULL;
        if (!aligned(p)) return GLA_ERR_ALIGN;
    }
    for (const void* p : optional)
        if (p && !aligned(p)) return GLA_ERR_ALIGN;
    return GLA_OK;
}

int resolve(const gla_desc* d) {
    if (d->path == GLA_PATH_SIMT) return GLA_PATH_SIMT;
    const bool tc_ok = gla::tc::supported(d->B, d->H, d->T, d->K, d->V, d->chunk, d->subchunk, d->qkv_dtype,
                                          d->gate_dtype);
    if (d->path == GLA_PATH_TC) return tc_ok ? GLA_PATH_TC : -1;
    return tc_ok ? GLA_PATH_TC : GLA_PATH_SIMT;
}

gla::Problem make_fwd(const gla_desc* d, int mode) {
    gla::Problem p{};
    p.B = d->B; p.H = d->H; p.T = d->T; p.K = d->K; p.V = d->V; p.C = d->chunk; p.c = d->subchunk;
    p.qkv_dtype = d->qkv_dtype; p.gate_dtype = d->gate_dtype; p.mode = mode;
    return p;
}

gla::BwdProblem make_bwd(const gla_desc* d, int mode) {
    gla::BwdProblem p{};
    p.B = d->B; p.H = d->H; p.T = d->T; p.K = d->K; p.V = d->V; p.C = d->chunk; p.c = d->subchunk;
    p.qkv_dtype = d->qkv_dtype; p.gate_dtype = d->gate_dtype; p.mode = mode;
    return p;
}

// T == 0: nothing to scan.  final_state = h0 (or 0); d_initial_state = d_final_state (or 0).
int copy_or_zero(float* dst, const float* src, size_t n, cudaStream_t st) {
    if (!dst) return GLA_OK;
    cudaError_t e = src ? cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st)
                        : cudaMemsetAsync(dst, 0, n * sizeof(float), st);
    return cuda_status(e);
}

// Saved-forward fingerprints (gla_chunk_bwd_saved): the backward reuses per-chunk operands of the forward that
// depend on q, k, log_alpha (Q~, K~, P, statistics) and, through the saved anchor / segment-entry states, on v and
// initial_state as well.  Every TC gla_chunk_fwd records which inputs filled its workspace; a saved backward
// whose inputs differ (another pointer, a different descriptor, h0 present in one call only) ignores the
// workspace and recomputes instead.  Host-side map keyed by the workspace pointer (mutex-protected).
struct FwdPrint {
    const void *q, *k, *v, *g;
    const float* h0;
    int B, H, T, K, V, C, c, qt, gt;
    bool operator==(const FwdPrint& o) const {
        return q == o.q && k == o.k && v == o.v && g == o.g && h0 == o.h0 && B == o.B && H == o.H && T == o.T &&
               K == o.K && V == o.V && C == o.C && c == o.c && qt == o.qt && gt == o.gt;
    }
};
std::mutex g_print_mu;
std::map<const void*, FwdPrint> g_prints;

FwdPrint make_print(const gla_desc* d, const void* q, const void* k, const void* v, const void* g, const float* h0) {
    return FwdPrint{q, k, v, g, h0, d->B, d->H, d->T, d->K, d->V, d->chunk, d->subchunk, d->qkv_dtype, d->gate_dtype};
}
void record_print(const void* ws, const FwdPrint& f) {
    std::lock_guard<std::mutex> lock(g_print_mu);
    if (g_prints.size() > 4096) g_prints.clear();   // bounded: stale entries only cost a recompute
    g_prints[ws] = f;
}
bool print_matches(const void* ws, const FwdPrint& f) {
    std::lock_guard<std::mutex> lock(g_print_mu);
    auto it = g_prints.find(ws);
    return it != g_prints.end() && it->second == f;
}

}  // namespace

namespace gla {
void set_last_cuda(int e) { g_last_cuda = e; }
}  // namespace gla

extern "C" {

int gla_version(void) { return 100; }

int gla_last_cuda_error(void) { return g_last_cuda; }

const char* gla_status_string(int s) {
    switch (s) {
        case GLA_OK: return "ok";
        case GLA_ERR_SHAPE: return "bad shape (B,H,T >= 0; 0 < K <= 256; 0 < V <= 1024)";
        case GLA_ERR_PLAN: return "bad chunk plan (chunk | T, subchunk | chunk, chunk <= 64)";
        case GLA_ERR_DTYPE: return "bad dtype code";
        case GLA_ERR_ALIGN: return "pointer not 16-byte aligned";
        case GLA_ERR_NULL: return "required pointer is NULL";
        case GLA_ERR_UNSUPPORTED: return "shape/dtype not supported by the requested path";
        case GLA_ERR_CUDA: return "CUDA error (see gla_last_cuda_error)";
        case GLA_ERR_WORKSPACE: return "workspace missing or too small";
        default: return "unknown status";
    }
}

int gla_resolve_path(const gla_desc* d) {
    int s = check_desc(d);
    if (s) return -s;
    return resolve(d);
}

size_t gla_fwd_workspace_size(const gla_desc* d) {
    if (check_desc(d)) return 0;
    if (resolve(d) == GLA_PATH_TC) return gla::tc::fwd_ws(d->B, d->H, d->T, d->K, d->V, d->chunk);
    return gla::simt::fwd_ws(d->B, d->H, d->T, d->K, d->V, d->chunk);
}

size_t gla_bwd_workspace_size(const gla_desc* d) {
    if (check_desc(d)) return 0;
    if (resolve(d) == GLA_PATH_TC) return gla::tc::bwd_ws(d->B, d->H, d->T, d->K, d->V, d->chunk);
    return gla::simt::bwd_ws(d->B, d->H, d->T, d->K, d->V, d->chunk);
}

int gla_chunk_fwd(const gla_desc* d, const void* q, const void* k, const void* v, const void* log_alpha,
                  const float* initial_state, void* out, float* final_state, void* workspace,
                  size_t workspace_bytes, void* stream) {
    int s = check_desc(d);
    if (s) return s;
    const int path = resolve(d);
    if (path < 0) return GLA_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if ((size_t)d->B * d->H == 0) return GLA_OK;
    if (d->T == 0) {   // empty sequence: only the state pointers matter
        s = check_ptrs({}, {initial_state, final_state});
        return s ? s : copy_or_zero(final_state, initial_state, (size_t)d->B * d->H * d->K * d->V, st);
    }
    s = check_ptrs({q, k, v, log_alpha, out}, {initial_state, final_state, workspace});
    if (s) return s;
    if (workspace_bytes < gla_fwd_workspace_size(d) || (!workspace && gla_fwd_workspace_size(d)))
        return GLA_ERR_WORKSPACE;
    gla::Problem p = make_fwd(d, 0);
    p.q = q; p.k = k; p.v = v; p.g = log_alpha; p.h0 = initial_state; p.out = out;
    p.final_state = final_state; p.ws = workspace;
    if (path == GLA_PATH_TC) record_print(workspace, make_print(d, q, k, v, log_alpha, initial_state));
    return cuda_status(path == GLA_PATH_TC ? gla::tc::fwd(p, st) : gla::simt::fwd(p, st));
}

int gla_chunk_bwd_saved(const gla_desc* d, const void* q, const void* k, const void* v, const void* log_alpha,
                  const float* initial_state, const void* d_out, const float* d_final_state, void* dq, void* dk,
                  void* dv, float* d_log_alpha, float* d_initial_state, void* workspace, size_t workspace_bytes,
                  const void* fwd_workspace, void* stream) {
    int s = check_desc(d);
    if (s) return s;
    const int path = resolve(d);
    if (path < 0) return GLA_ERR_UNSUPPORTED;
    cudaStream_t st = (cudaStream_t)stream;
    if ((size_t)d->B * d->H == 0) return GLA_OK;
    if (d->T == 0) {
        s = check_ptrs({}, {initial_state, d_final_state, d_initial_state});
        return s ? s : copy_or_zero(d_initial_state, d_final_state, (size_t)d->B * d->H * d->K * d->V, st);
    }
    s = check_ptrs({q, k, v, log_alpha, d_out, dq, dk, dv, d_log_alpha},
                   {initial_state, d_final_state, d_initial_state, workspace, fwd_workspace});
    if (s) return s;
    if (workspace_bytes < gla_bwd_workspace_size(d) || (!workspace && gla_bwd_workspace_size(d)))
        return GLA_ERR_WORKSPACE;
    gla::BwdProblem p = make_bwd(d, 0);
    p.q = q; p.k = k; p.v = v; p.g = log_alpha; p.dO = d_out; p.h0 = initial_state; p.dfinal = d_final_state;
    p.dq = dq; p.dk = dk; p.dv = dv; p.dg = d_log_alpha; p.dh0 = d_initial_state; p.ws = workspace;
    // reuse the forward's operands only if that workspace was filled by a forward on these very inputs
    p.fwd_ws = (fwd_workspace && print_matches(fwd_workspace, make_print(d, q, k, v, log_alpha, initial_state)))
                   ? fwd_workspace : nullptr;
    return cuda_status(path == GLA_PATH_TC ? gla::tc::bwd(p, st) : gla::simt::bwd(p, st));
}

int gla_chunk_bwd(const gla_desc* d, const void* q, const void* k, const void* v, const void* log_alpha,
                  const float* initial_state, const void* d_out, const float* d_final_state, void* dq, void* dk,
                  void* dv, float* d_log_alpha, float* d_initial_state, void* workspace, size_t workspace_bytes,
                  void* stream) {
    return gla_chunk_bwd_saved(d, q, k, v, log_alpha, initial_state, d_out, d_final_state, dq, dk, dv, d_log_alpha,
                               d_initial_state, workspace, workspace_bytes, nullptr, stream);
}

// ---- the general outer-product gate G_t = alpha_t^T beta_t: fp32 CUDA-core path (simt_beta.cu) ----
size_t gla_beta_workspace_size(const gla_desc* d) {
    if (check_desc(d)) return 0;
    return gla::simt::beta_ws(d->B, d->H, d->T, d->K, d->V, d->chunk);
}

namespace {
gla::BetaProblem make_beta(const gla_desc* d, const void* q, const void* k, const void* v, const void* la,
                           const void* lb, const float* h0, void* ws) {
    gla::BetaProblem p{};
    p.B = d->B; p.H = d->H; p.T = d->T; p.K = d->K; p.V = d->V; p.C = d->chunk; p.c = d->subchunk;
    p.qkv_dtype = d->qkv_dtype; p.gate_dtype = d->gate_dtype;
    p.q = q; p.k = k; p.v = v; p.g = la; p.lb = lb; p.h0 = h0; p.ws = ws;
    return p;
}
int check_beta(const gla_desc* d) {
    int s = check_desc(d);
    if (s) return s;
    return d->path == GLA_PATH_TC ? GLA_ERR_UNSUPPORTED : GLA_OK;   // the value gate runs on the SIMT kernels
}
}  // namespace

int gla_chunk_fwd_beta(const gla_desc* d, const void* q, const void* k, const void* v, const void* log_alpha,
                       const void* log_beta, const float* initial_state, void* out, float* final_state,
                       void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_beta(d);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((size_t)d->B * d->H == 0) return GLA_OK;
    if (d->T == 0) {
        s = check_ptrs({}, {initial_state, final_state});
        return s ? s : copy_or_zero(final_state, initial_state, (size_t)d->B * d->H * d->K * d->V, st);
    }
    s = check_ptrs({q, k, v, log_alpha, log_beta, out, workspace}, {initial_state, final_state});
    if (s) return s;
    if (workspace_bytes < gla_beta_workspace_size(d)) return GLA_ERR_WORKSPACE;
    gla::BetaProblem p = make_beta(d, q, k, v, log_alpha, log_beta, initial_state, workspace);
    p.out = out; p.final_state = final_state;
    return cuda_status(gla::simt::fwd_beta(p, st));
}

int gla_chunk_bwd_beta(const gla_desc* d, const void* q, const void* k, const void* v, const void* log_alpha,
                       const void* log_beta, const float* initial_state, const void* d_out,
                       const float* d_final_state, void* dq, void* dk, void* dv, float* d_log_alpha,
                       float* d_log_beta, float* d_initial_state, void* workspace, size_t workspace_bytes,
                       void* stream) {
    int s = check_beta(d);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((size_t)d->B * d->H == 0) return GLA_OK;
    if (d->T == 0) {
        s = check_ptrs({}, {initial_state, d_final_state, d_initial_state});
        return s ? s : copy_or_zero(d_initial_state, d_final_state, (size_t)d->B * d->H * d->K * d->V, st);
    }
    s = check_ptrs({q, k, v, log_alpha, log_beta, d_out, dq, dk, dv, d_log_alpha, d_log_beta, workspace},
                   {initial_state, d_final_state, d_initial_state});
    if (s) return s;
    if (workspace_bytes < gla_beta_workspace_size(d)) return GLA_ERR_WORKSPACE;
    gla::BetaBwdProblem p{};
    p.f = make_beta(d, q, k, v, log_alpha, log_beta, initial_state, workspace);
    p.dO = d_out; p.dfinal = d_final_state; p.dq = dq; p.dk = dk; p.dv = dv; p.dg = d_log_alpha;
    p.dlb = d_log_beta; p.dh0 = d_initial_state;
    return cuda_status(gla::simt::bwd_beta(p, st));
}

int gla_recurrent_step_beta(int B, int H, int K, int V, int dtype, int gate_dtype, const void* q_t,
                            const void* k_t, const void* v_t, const void* log_alpha_t, const void* log_beta_t,
                            float* state, void* out_t, void* stream) {
    if (B < 0 || H < 0 || K <= 0 || V <= 0) return GLA_ERR_SHAPE;
    if (!ok_dtype(dtype) || !ok_dtype(gate_dtype)) return GLA_ERR_DTYPE;
    int s = check_ptrs({q_t, k_t, v_t, log_alpha_t, log_beta_t, state, out_t}, {});
    if (s) return s;
    if ((size_t)B * H == 0) return GLA_OK;
    return cuda_status(gla::simt::step_beta(B * H, K, V, dtype, gate_dtype, q_t, k_t, v_t, log_alpha_t, log_beta_t,
                                            state, out_t, (cudaStream_t)stream));
}

int gla_recurrent_step(int B, int H, int K, int V, int dtype, int gate_dtype, const void* q_t, const void* k_t,
                       const void* v_t, const void* log_alpha_t, float* state, void* out_t, void* stream) {
    if (B < 0 || H < 0 || K <= 0 || V <= 0 || K > 1024) return GLA_ERR_SHAPE;   // (K <= 1024: staged in smem)
    if (!ok_dtype(dtype) || !ok_dtype(gate_dtype)) return GLA_ERR_DTYPE;
    int s = check_ptrs({q_t, k_t, v_t, log_alpha_t, state, out_t}, {});
    if (s) return s;
    if ((size_t)B * H == 0) return GLA_OK;
    return cuda_status(gla::simt::step(B * H, K, V, dtype, gate_dtype, q_t, k_t, v_t, log_alpha_t, state, out_t,
                                       (cudaStream_t)stream));
}

int gla_state_summary(const gla_desc* d, const void* k, const void* v, const void* log_alpha, float* S_loc,
                      float* log_decay, void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_desc(d);
    if (s) return s;
    s = check_ptrs({k, v, log_alpha, S_loc, log_decay}, {workspace});
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((size_t)d->B * d->H == 0) return GLA_OK;
    const size_t BHK = (size_t)d->B * d->H * d->K;
    if (d->T == 0) {
        s = copy_or_zero(S_loc, nullptr, BHK * d->V, st);
        return s ? s : copy_or_zero(log_decay, nullptr, BHK, st);
    }
    if (resolve(d) == GLA_PATH_TC && gla::tc::summary_tc_ok(d->K, d->V)) {
        // tensor-core contraction (prep + one k_seg_summary per unit); needs the forward's workspace
        if (workspace_bytes < gla_fwd_workspace_size(d) || !workspace) return GLA_ERR_WORKSPACE;
        gla::Problem p = make_fwd(d, 0);
        p.q = k; p.k = k; p.v = v; p.g = log_alpha; p.ws = workspace;
        return cuda_status(gla::tc::summary_tc(p, v, S_loc, log_decay, false, st));
    }
    gla::Problem p = make_fwd(d, 1);
    p.q = nullptr; p.k = k; p.v = v; p.g = log_alpha; p.h0 = nullptr; p.out = nullptr;
    p.final_state = S_loc; p.log_decay = log_decay; p.ws = workspace;
    return cuda_status(gla::simt::fwd(p, st));
}

int gla_dstate_summary(const gla_desc* d, const void* q, const void* d_out, const void* log_alpha, float* dh0_loc,
                       void* workspace, size_t workspace_bytes, void* stream) {
    int s = check_desc(d);
    if (s) return s;
    s = check_ptrs({q, d_out, log_alpha, dh0_loc}, {workspace});
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((size_t)d->B * d->H == 0) return GLA_OK;
    if (d->T == 0) return copy_or_zero(dh0_loc, nullptr, (size_t)d->B * d->H * d->K * d->V, st);
    if (resolve(d) == GLA_PATH_TC && gla::tc::summary_tc_ok(d->K, d->V)) {
        if (workspace_bytes < gla_fwd_workspace_size(d) || !workspace) return GLA_ERR_WORKSPACE;
        gla::Problem pf = make_fwd(d, 0);
        pf.q = q; pf.k = q; pf.v = d_out; pf.g = log_alpha; pf.ws = workspace;
        return cuda_status(gla::tc::summary_tc(pf, d_out, dh0_loc, nullptr, true, st));
    }
    gla::BwdProblem p = make_bwd(d, 1);
    p.q = q; p.k = q; p.g = log_alpha; p.dO = d_out; p.dh0 = dh0_loc; p.ws = workspace;
    return cuda_status(gla::simt::bwd(p, st));
}

int gla_state_combine(int BH, int K, int V, const float* H_in, const float* log_decay, const float* S_loc,
                      float* H_out, void* stream) {
    if (BH < 0 || K <= 0 || V <= 0) return GLA_ERR_SHAPE;
    int s = check_ptrs({H_in, log_decay, S_loc, H_out}, {});
    if (s) return s;
    if (BH == 0) return GLA_OK;
    return cuda_status(gla::simt::combine(BH, K, V, H_in, log_decay, S_loc, H_out, (cudaStream_t)stream));
}

}  // extern "C"
