/*
 * gla.h -- C ABI of libgla.so: chunk-wise Gated Linear Attention (arXiv 2312.06635) on B200 (sm_100a).
 *
 * Notation (PAPER.md = "P:<line>"): per (batch b, head h) unit, 0-based token t,
 *   q_t, k_t, log_alpha_t in R^K   (K = d_k' = d_k / H, per-head key dim)
 *   v_t, o_t in R^V                (V = d_v' = d_v / H)
 *   S_t = diag(exp(log_alpha_t)) S_{t-1} + k_t^T v_t,  o_t = q_t S_t        (beta == 1 per P:321)
 * The library computes this operator with the chunk-wise two-level algorithm: chunk size C
 * (`chunk`), sub-chunk size c (`subchunk`).  The result is the recurrence's (the method is exact);
 * `chunk`/`subchunk` change only the rounding and the speed.  On the SIMT path both are honoured as given.
 * On the tensor-core path C = 64 and `subchunk` must divide 64 but is otherwise ignored: the TC kernels form
 * the 64 x 64 intra-chunk score block with one per-chunk normaliser under a range guard (R8/R9).
 * A chunk that fails the guard (some channel's half-chunk log decay exceeds 60) takes the exact path for that
 * chunk only: P from the paper's per-sub-chunk-pair normalisers taken down to single tokens (six
 * levels, tensor cores, every factor <= 1), the walks in the r = 0 frame, and (gla_chunk_bwd_saved with K-tiled
 * walks: K in {128,256}, V in {256,512}) the exact intra-chunk backward terms in fp32 in the reduce.  The other
 * TC backward configurations (gla_chunk_bwd, or other V) still send the WHOLE backward call to the fp32
 * CUDA-core kernels when any chunk is flagged (correct, but ~40x slower: the "guard cliff").
 *
 * Conventions shared by every entry point
 *   - Layout: row-major, [B, H, T, K] for q/k/log_alpha/dq/dk/d_log_alpha, [B, H, T, V] for v/out/d_out/dv,
 *     [B, H, K, V] fp32 for every state (initial_state, final_state, S_loc, d_initial_state, ...).
 *     Every pointer must be 16-byte aligned and its tensor contiguous.
 *   - Pointers are DEVICE pointers owned by the caller (the library never allocates or frees device
 *     memory); `workspace` is caller-allocated scratch of at least the size the matching *_workspace_size
 *     function returns.  Inputs are never written.  Outputs are fully overwritten.
 *   - `stream` is a cudaStream_t (passed as void* so this header needs no CUDA include); every call is
 *     asynchronous on that stream.  Calls are thread-safe.  Process-wide state, all mutex-protected: a
 *     per-device attribute cache, the launch tracer (gla_profile_*), the saved-forward fingerprints of
 *     gla_chunk_bwd_saved, and one library-owned side stream per (device, caller stream) on which the TC
 *     backward runs its second walk concurrently (forked from and joined back into the caller's stream with
 *     events, so it is also safe inside CUDA-graph stream capture).
 *   - q is NOT scaled by 1/sqrt(d_k): the paper has o_t = q_t S_t; the caller pre-scales.
 *   - log_alpha must be finite and <= 0 (sigma in (0,1) gives log alpha < 0; 0 = linear attention).
 *   - Determinism: fixed reduction order, no atomics: identical inputs give bitwise-identical outputs.
 *   - Errors: validation failures return synchronously with NO kernel launched and NO output written;
 *     a launch failure returns GLA_ERR_CUDA (cudaGetLastError) -- see gla_last_cuda_error().  No C++
 *     exception crosses the ABI.
 */
#ifndef GLA_H
#define GLA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GLA_OK = 0,
    GLA_ERR_SHAPE = 1,        /* B,H,T < 0 or K,V <= 0, or K,V above the supported maximum            */
    GLA_ERR_PLAN = 2,         /* chunk does not divide T, subchunk does not divide chunk, or C/c unsupported (C > 128, or C > 64 beyond the SIMT tiles) ("split into non-overlapping chunks") */
    GLA_ERR_DTYPE = 3,        /* unknown dtype code                                                   */
    GLA_ERR_ALIGN = 4,        /* a pointer is not 16-byte aligned                                     */
    GLA_ERR_NULL = 5,         /* a required pointer is NULL                                           */
    GLA_ERR_UNSUPPORTED = 6,  /* requested path cannot run this shape (e.g. PATH_TC with K not in {64,128,256}) */
    GLA_ERR_CUDA = 7,         /* kernel launch / device query failed                                  */
    GLA_ERR_WORKSPACE = 8     /* workspace NULL or smaller than *_workspace_size()                    */
} gla_status;

typedef enum { GLA_BF16 = 0, GLA_FP32 = 1 } gla_dtype;

/* Which implementation runs.
 *   GLA_PATH_AUTO : tensor-core path (tcgen05/TMEM/TMA) when qkv_dtype == BF16 and the shape is supported,
 *                   otherwise the SIMT path.
 *   GLA_PATH_SIMT : fp32-arithmetic CUDA-core kernels (the "fp32 debug build": any C <= 128, c with c | C | T,
 *                   K <= 256, V <= 1024; parity 1e-5 vs the fp64 oracle with fp32 inputs).  C > 64 needs the
 *                   kernels' per-CTA tiles to fit in shared memory (e.g. C = 128 with K, V <= 128), else
 *                   GLA_ERR_PLAN.
 *   GLA_PATH_TC   : bf16 tensor-core kernels: qkv_dtype BF16, C = 64, c | 64 (ignored, see above),
 *                   K in {64,128,256}, V % 128 == 0.  The TC backward needs K in {128,256} and
 *                   V / 128 in {1,2,4,8}; other TC-forward shapes run the backward on the SIMT kernels. */
typedef enum { GLA_PATH_AUTO = 0, GLA_PATH_SIMT = 1, GLA_PATH_TC = 2 } gla_path;

typedef struct {
    int B, H, T, K, V;   /* batch, heads, tokens, per-head key dim, per-head value dim            */
    int chunk;           /* C: first-level chunk length; must divide T                      */
    int subchunk;        /* c: secondary-level sub-chunk length; must divide C         */
    int qkv_dtype;       /* gla_dtype of q, k, v, out, d_out, dq, dk, dv                           */
    int gate_dtype;      /* gla_dtype of log_alpha (d_log_alpha is always fp32)                     */
    int path;            /* gla_path                                                              */
} gla_desc;

/* Scratch needed by gla_chunk_fwd / gla_chunk_bwd / gla_state_summary for this descriptor (bytes). */
size_t gla_fwd_workspace_size(const gla_desc *d);
size_t gla_bwd_workspace_size(const gla_desc *d);

/*
 * gla_chunk_fwd -- forward pass, parts (1)-(3) of the method:
 *   (1) chunk-local log-space cumsum of log_alpha            (P:216 A_t = prod alpha_j)
 *   (2) inter-chunk state passing  S_[i+1] = diag(e^Gamma_i) S_[i] + (K_i (.) e^{Gamma_i - b})^T V_i,
 *       cross-chunk output (Q_i (.) e^{b}) S_[i]            (P:250-262 Eqs. gla_inter_chunk_recur, gla_inter_intra)
 *   (3) intra-chunk secondary chunking: off-diagonal sub-chunk blocks on bf16 tensor cores, diagonal
 *       blocks in fp32 log space                             (P:269-284 Eqs. gla-subchunk-compute-p/o)
 * in:  q, k [B,H,T,K] (qkv_dtype); v [B,H,T,V] (qkv_dtype); log_alpha [B,H,T,K] (gate_dtype);
 *      initial_state [B,H,K,V] fp32 or NULL (= zeros; P:88 footnote)
 * out: out [B,H,T,V] (qkv_dtype); final_state [B,H,K,V] fp32 = S_T, or NULL (not written)
 */
int gla_chunk_fwd(const gla_desc *d, const void *q, const void *k, const void *v, const void *log_alpha,
                  const float *initial_state, void *out, float *final_state,
                  void *workspace, size_t workspace_bytes, void *stream);

/*
 * gla_chunk_bwd -- part (4): gradients of  L = <out, d_out> + <final_state, d_final_state>
 * (the paper gives no backward; derivation in DESIGN.md "Backward").  Reverse state pass
 * dS_[i] = diag(e^Gamma_i) dS_[i+1] + (Q_i (.) e^{b})^T dO_i, intra-chunk blocks, and
 * d log alpha_t = sum_{s >= t} (q (.) dq - k (.) dk)_s + rowsum(S_T (.) dS_T).
 * in:  as gla_chunk_fwd, plus d_out [B,H,T,V] (qkv_dtype), d_final_state [B,H,K,V] fp32 or NULL (= 0)
 * out: dq, dk [B,H,T,K] and dv [B,H,T,V] (qkv_dtype); d_log_alpha [B,H,T,K] fp32 (always);
 *      d_initial_state [B,H,K,V] fp32 or NULL (not written)
 */
int gla_chunk_bwd(const gla_desc *d, const void *q, const void *k, const void *v, const void *log_alpha,
                  const float *initial_state, const void *d_out, const float *d_final_state,
                  void *dq, void *dk, void *dv, float *d_log_alpha, float *d_initial_state,
                  void *workspace, size_t workspace_bytes, void *stream);

/*
 * gla_chunk_bwd_saved -- gla_chunk_bwd reusing the per-chunk operands a preceding gla_chunk_fwd left in its
 * workspace (the "saved activations" of a training step): on the tensor-core path the backward then skips
 * recomputing the chunk-local cumsums, Q~, K~ and P = (Q~ K~^T) (.) M and only forms dP.
 * fwd_workspace: the workspace of a gla_chunk_fwd call with the same descriptor and the same q, k, v,
 *                log_alpha and initial_state (same pointers, same contents), not modified since (no ownership
 *                transfer; the caller keeps both buffers alive), or NULL (then identical to gla_chunk_bwd).
 *                The forward's saved data depend on all five inputs (Q~, K~, P and the chunk statistics on
 *                q, k, log_alpha; the saved anchor and segment-entry states also on v and initial_state).
 *                The library records which pointers filled each forward workspace; if they differ from this
 *                call's (or initial_state is present in one call only) the workspace is ignored and the
 *                backward recomputes.  Contents changed behind identical pointers cannot be detected.
 *                Ignored on the SIMT path.
 * Results are bitwise identical to gla_chunk_bwd's.  Other arguments, errors: as gla_chunk_bwd.
 */
int gla_chunk_bwd_saved(const gla_desc *d, const void *q, const void *k, const void *v, const void *log_alpha,
                        const float *initial_state, const void *d_out, const float *d_final_state,
                        void *dq, void *dk, void *dv, float *d_log_alpha, float *d_initial_state,
                        void *workspace, size_t workspace_bytes, const void *fwd_workspace, void *stream);

/*
 * gla_recurrent_step -- one decoding step of the recurrent form, for every (b,h):
 *   state <- diag(exp(log_alpha_t)) state + k_t^T v_t ;  out_t = q_t state
 * in:  q_t, k_t [B,H,K] and v_t [B,H,V] (dtype); log_alpha_t [B,H,K] (gate_dtype)
 * in/out: state [B,H,K,V] fp32 (updated in place)
 * out: out_t [B,H,V] (dtype)
 * errors: GLA_ERR_SHAPE also for K > 1024.
 */
int gla_recurrent_step(int B, int H, int K, int V, int dtype, int gate_dtype,
                       const void *q_t, const void *k_t, const void *v_t, const void *log_alpha_t,
                       float *state, void *out_t, void *stream);

/*
 * The general outer-product gate:  G_t = alpha_t^T beta_t,
 *   S_t = G_t (.) S_{t-1} + k_t^T v_t,  o_t = q_t S_t          (P:188-189 without the beta == 1 simplification)
 * with log_beta [B,H,T,V] (gate_dtype; finite, <= 0) the value-side gate.  Computed chunk-wise with the paper's
 * V~ = V / B, O = O~ (.) B rescaling (Eq. gla_QKV2) applied per chunk with a mid-chunk normaliser
 * (simt_beta.cu), on the fp32 CUDA-core kernels: GLA_PATH_TC returns GLA_ERR_UNSUPPORTED, AUTO / SIMT run it.
 * Range: the half-chunk log decay of beta must stay below ~60 (the paper's gates give ~2 at C = 64).
 * gla_chunk_fwd_beta / gla_chunk_bwd_beta: as gla_chunk_fwd / gla_chunk_bwd plus log_beta (in) and
 *   d_log_beta [B,H,T,V] fp32 (out) = sum_{s >= t} (o (.) do - v (.) dv)_s + colsum(S_T (.) dS_T).
 *   workspace: at least gla_beta_workspace_size(d) bytes (required, also for the forward).
 * gla_recurrent_step_beta: one decode step  state <- (alpha_t^T beta_t) (.) state + k_t^T v_t, out_t = q_t state
 *   (log_beta_t [B,H,V]).
 */
size_t gla_beta_workspace_size(const gla_desc *d);
int gla_chunk_fwd_beta(const gla_desc *d, const void *q, const void *k, const void *v, const void *log_alpha,
                       const void *log_beta, const float *initial_state, void *out, float *final_state,
                       void *workspace, size_t workspace_bytes, void *stream);
int gla_chunk_bwd_beta(const gla_desc *d, const void *q, const void *k, const void *v, const void *log_alpha,
                       const void *log_beta, const float *initial_state, const void *d_out,
                       const float *d_final_state, void *dq, void *dk, void *dv, float *d_log_alpha,
                       float *d_log_beta, float *d_initial_state, void *workspace, size_t workspace_bytes,
                       void *stream);
int gla_recurrent_step_beta(int B, int H, int K, int V, int dtype, int gate_dtype, const void *q_t,
                            const void *k_t, const void *v_t, const void *log_alpha_t, const void *log_beta_t,
                            float *state, void *out_t, void *stream);

/*
 * Segment / sequence-parallel helpers (chunk-level recurrence as a two-stage scan).
 * For a segment of T tokens with zero initial state:
 *   gla_state_summary:  S_loc = sum_t (k_t (.) e^{LA_T - LA_t})^T v_t  [B,H,K,V] fp32,
 *                       log_decay = LA_T = sum_t log_alpha_t           [B,H,K]   fp32
 *   gla_dstate_summary: dh0_loc = sum_t (q_t (.) e^{LA_t})^T d_out_t    [B,H,K,V] fp32
 *                       (the d_initial_state of the segment when d_final_state = 0)
 *   gla_state_combine:  H_out = diag(e^{log_decay}) H_in + S_loc        (BH = B*H units; H_out may alias H_in)
 * so that, for consecutive segments r, the state entering r+1 is combine(H_r, D_r, S_loc_r) and the
 * adjoint leaving r-1 is combine(dF_r, D_r, dh0_loc_r).
 * Paths: when the descriptor resolves to GLA_PATH_TC and K in {128,256}, V % 256 == 0, both summaries run on
 * the tensor cores (the forward's prep kernel, then one tcgen05 contraction per (b,h) unit) and need
 * `workspace` of at least gla_fwd_workspace_size(d) bytes (else GLA_ERR_WORKSPACE); otherwise they run the
 * fp32 CUDA-core kernels and workspace may be NULL.  In gla_dstate_summary the descriptor's V is d_out's.
 */
int gla_state_summary(const gla_desc *d, const void *k, const void *v, const void *log_alpha,
                      float *S_loc, float *log_decay, void *workspace, size_t workspace_bytes, void *stream);
int gla_dstate_summary(const gla_desc *d, const void *q, const void *d_out, const void *log_alpha,
                       float *dh0_loc, void *workspace, size_t workspace_bytes, void *stream);
int gla_state_combine(int BH, int K, int V, const float *H_in, const float *log_decay, const float *S_loc,
                      float *H_out, void *stream);

/*
 * GLA layer: the elementwise stages of a full multi-head GLA layer around the core
 * (P:298-307 multi-head GLA layer with per-head LayerNorm and Swish output gate; P:321-326 low-rank gate with
 * beta == 1; P:177 log-space temperature tau).  The projections x W are plain GEMMs done by the caller (cuBLAS).
 * All pointers are device pointers, 16-byte aligned; P is the projection output [B*T][ldP] bf16 with column
 * blocks q (H*K) | k (H*K) | v (H*V) | r (H*V) (ldP >= 2HK + 2HV, ldP % 8 == 0); z_alpha [B*T][H*K] bf16 is the
 * low-rank gate pre-activation x W1 W2; parameters are fp32.  Constraints: K % 8 == 0, V in {256,512,768,1024},
 * H <= 32.  Errors as the core's; workspace-taking calls need gla_layer_bwd_workspace_size() bytes.
 *
 * gla_layer_prep:  q, k [B,H,T,K], v [B,H,T,V] (bf16, transposed out of P) and
 *                  log_alpha [B,H,T,K] fp32 = logsigmoid(z_alpha + b_alpha) / tau.
 * gla_layer_out:   Z [B*T][H*V] bf16 = concat_h(LN(O^h) * ln_w + ln_b) (.) Swish(r + b_r), O [B,H,T,V] bf16 the
 *                  core's output, LN over each head's V values (eps); r = P[:, r_off : r_off + H*V].  Saves the
 *                  per-(row, head) mean and rstd [B*T*H] fp32 for the backward.
 * gla_layer_out_bwd: from dZ: dO [B,H,T,V] bf16 (the core's d_out), d r written into dP's r block (bf16), and
 *                  d ln_w, d ln_b, d b_r [H*V] fp32 (deterministic fixed-order reductions).
 * gla_layer_prep_bwd: from the core's dq, dk, dv (bf16) and d_log_alpha (fp32): dP's q | k | v blocks (bf16),
 *                  d z_alpha [B*T][H*K] bf16 and d b_alpha [H*K] fp32.
 */
size_t gla_layer_bwd_workspace_size(int B, int T, int H, int K, int V);
int gla_layer_prep(int B, int T, int H, int K, int V, float tau, const void *P, int ldP, const void *z_alpha,
                   const float *b_alpha, void *q, void *k, void *v, float *log_alpha, void *stream);
int gla_layer_out(int B, int T, int H, int V, const void *O, const void *P, int ldP, int r_off, const float *b_r,
                  const float *ln_w, const float *ln_b, float eps, void *Z, float *mean, float *rstd, void *stream);
int gla_layer_out_bwd(int B, int T, int H, int V, const void *dZ, const void *O, const void *P, int ldP, int r_off,
                      const float *b_r, const float *ln_w, const float *ln_b, const float *mean, const float *rstd,
                      void *dO, void *dP, float *d_ln_w, float *d_ln_b, float *d_b_r, void *workspace,
                      size_t workspace_bytes, void *stream);
int gla_layer_prep_bwd(int B, int T, int H, int K, int V, float tau, const void *dq, const void *dk, const void *dv,
                       const float *d_log_alpha, const void *z_alpha, const float *b_alpha, void *dP, int ldP,
                       void *d_z_alpha, float *d_b_alpha, void *workspace, size_t workspace_bytes, void *stream);

/*
 * Launch tracing (the library's own profiler, used by bench.py for the live roofline numbers).
 * When enabled, every kernel launch is bracketed by two cudaEvents recorded on its launching stream.
 * gla_profile_get aggregates by kernel name: fills names[i*64 .. i*64+63] (NUL-terminated), total_ms[i]
 * and launches[i] for i < cap; returns the number of distinct kernels.  It synchronizes on the events.
 */
void gla_profile_enable(int enable);
void gla_profile_reset(void);
int gla_profile_count(void);
int gla_profile_get(int cap, char *names, float *total_ms, int *launches);

/* Human-readable status text (static storage). */
const char *gla_status_string(int status);
/* cudaError_t of the last GLA_ERR_CUDA returned on the calling thread (0 if none). */
int gla_last_cuda_error(void);
/* Which path GLA_PATH_AUTO would pick for this descriptor (GLA_PATH_SIMT or GLA_PATH_TC). */
int gla_resolve_path(const gla_desc *d);
/* Library version: 100 * major + minor. */
int gla_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GLA_H */
