/*
 * gla_oracle.c -- fp64 CPU oracle for Gated Linear Attention (arXiv 2312.06635).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The CUDA product path
 * (paper_2312_06635_b200/) never links, imports or calls it, and shares no code with it.
 *
 * What it computes: the paper's RECURRENT form, with the value-side gate removed
 * (beta == 1, "we remove it (i.e., beta_t = 1)"), per (batch, head) independently
 * (multi-head GLA):
 *
 *     S_0 = h0 (zeros if absent)                       P:88 footnote ("initialize ... historical states")
 *     S_t = G_t (.) S_{t-1} + k_t^T v_t,               P:188 Eq. gla_recurrence
 *           G_t = alpha_t^T 1, alpha_t = exp(log_alpha_t)   P:171, P:177 (gates applied in log space)
 *     o_t = q_t S_t
 *     final_state = S_T
 *
 * The method is exact (the chunk-wise two-level form reaches the same result),
 * so this plain definition is the oracle.  Backward (the paper gives none),
 * reverse-mode of the recurrence above with adjoint dS:
 *
 *     dS = d_final_state (or 0)
 *     for t = T..1:  dS += q_t^T do_t
 *                    dq_t = S_t do_t^T,  dk_t = dS v_t^T,  dv_t = k_t dS
 *                    dlog_alpha_t = alpha_t (.) rowsum(dS (.) S_{t-1})
 *                    dS = diag(alpha_t) dS
 *     d_initial_state = dS
 *
 * States S_t are recomputed from checkpoints every ORACLE_CKPT steps (memory O(T/64 K V)).
 * All inputs and outputs are double; arithmetic is fp64; the summation order inside one
 * (b,h) unit is fixed (ascending index), so results are deterministic.  Threads split the
 * B*H units only.
 *
 * Layout: q, k, log_alpha [B,H,T,K]; v, o, d_out [B,H,T,V]; states [B,H,K,V]; row-major.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_CKPT 64

typedef struct {
    int B, H, T, K, V;
    const double *q, *k, *v, *g, *h0, *d_out, *d_final;
    double *o, *final_state, *dq, *dk, *dv, *dg, *dh0;
    int next_unit;          /* protected by mu */
    int error;
    pthread_mutex_t mu;
} job_t;

/* one recurrence step: S <- diag(exp(g_t)) S + k_t^T v_t */
static void step_state(double *S, const double *kt, const double *vt, const double *gt, int K, int V)
{
    for (int m = 0; m < K; ++m) {
        const double a = exp(gt[m]);
        const double km = kt[m];
        double *row = S + (size_t)m * V;
        for (int j = 0; j < V; ++j) row[j] = a * row[j] + km * vt[j];
    }
}

/* o_t = q_t S_t */
static void read_out(const double *S, const double *qt, double *ot, int K, int V)
{
    for (int j = 0; j < V; ++j) ot[j] = 0.0;
    for (int m = 0; m < K; ++m) {
        const double qm = qt[m];
        const double *row = S + (size_t)m * V;
        for (int j = 0; j < V; ++j) ot[j] += qm * row[j];
    }
}

static void fwd_unit(job_t *J, int u)
{
    const int T = J->T, K = J->K, V = J->V;
    const size_t KV = (size_t)K * V;
    const double *q = J->q + (size_t)u * T * K, *k = J->k + (size_t)u * T * K;
    const double *g = J->g + (size_t)u * T * K, *v = J->v + (size_t)u * T * V;
    double *S = (double *)malloc(KV * sizeof(double));
    if (!S) { J->error = 1; return; }
    if (J->h0) memcpy(S, J->h0 + u * KV, KV * sizeof(double));
    else memset(S, 0, KV * sizeof(double));
    for (int t = 0; t < T; ++t) {
        step_state(S, k + (size_t)t * K, v + (size_t)t * V, g + (size_t)t * K, K, V);
        if (J->o) read_out(S, q + (size_t)t * K, J->o + ((size_t)u * T + t) * V, K, V);
    }
    if (J->final_state) memcpy(J->final_state + u * KV, S, KV * sizeof(double));
    free(S);
}

static void bwd_unit(job_t *J, int u)
{
    const int T = J->T, K = J->K, V = J->V;
    const size_t KV = (size_t)K * V;
    const double *q = J->q + (size_t)u * T * K, *k = J->k + (size_t)u * T * K;
    const double *g = J->g + (size_t)u * T * K, *v = J->v + (size_t)u * T * V;
    const double *dO = J->d_out + (size_t)u * T * V;
    double *dq = J->dq + (size_t)u * T * K, *dk = J->dk + (size_t)u * T * K;
    double *dv = J->dv + (size_t)u * T * V, *dg = J->dg + (size_t)u * T * K;

    const int nseg = (T + ORACLE_CKPT - 1) / ORACLE_CKPT;
    double *ckpt = (double *)malloc((size_t)(nseg + 1) * KV * sizeof(double)); /* S at t = 64*j */
    double *seg = (double *)malloc((size_t)(ORACLE_CKPT + 1) * KV * sizeof(double));
    double *dS = (double *)malloc(KV * sizeof(double));
    if (!ckpt || !seg || !dS) { J->error = 1; free(ckpt); free(seg); free(dS); return; }

    /* forward sweep, keeping S_{64 j} */
    double *S = ckpt;
    if (J->h0) memcpy(S, J->h0 + u * KV, KV * sizeof(double));
    else memset(S, 0, KV * sizeof(double));
    for (int j = 0; j < nseg; ++j) {
        double *nxt = ckpt + (size_t)(j + 1) * KV;
        memcpy(nxt, ckpt + (size_t)j * KV, KV * sizeof(double));
        const int t1 = (j + 1) * ORACLE_CKPT < T ? (j + 1) * ORACLE_CKPT : T;
        for (int t = j * ORACLE_CKPT; t < t1; ++t)
            step_state(nxt, k + (size_t)t * K, v + (size_t)t * V, g + (size_t)t * K, K, V);
    }

    if (J->d_final) memcpy(dS, J->d_final + u * KV, KV * sizeof(double));
    else memset(dS, 0, KV * sizeof(double));

    for (int j = nseg - 1; j >= 0; --j) {
        const int t0 = j * ORACLE_CKPT;
        const int t1 = (j + 1) * ORACLE_CKPT < T ? (j + 1) * ORACLE_CKPT : T;
        /* seg[i] = S_{t0+i}  (0-based t: S after t0+i steps) */
        memcpy(seg, ckpt + (size_t)j * KV, KV * sizeof(double));
        for (int t = t0; t < t1; ++t) {
            memcpy(seg + (size_t)(t - t0 + 1) * KV, seg + (size_t)(t - t0) * KV, KV * sizeof(double));
            step_state(seg + (size_t)(t - t0 + 1) * KV, k + (size_t)t * K, v + (size_t)t * V,
                       g + (size_t)t * K, K, V);
        }
        for (int t = t1 - 1; t >= t0; --t) {
            const double *St = seg + (size_t)(t - t0 + 1) * KV;   /* S after token t */
            const double *Sp = seg + (size_t)(t - t0) * KV;       /* S before token t */
            const double *qt = q + (size_t)t * K, *kt = k + (size_t)t * K, *gt = g + (size_t)t * K;
            const double *vt = v + (size_t)t * V, *dot = dO + (size_t)t * V;
            /* dq_t = S_t do_t^T (uses S_t, the state that produced o_t) */
            for (int m = 0; m < K; ++m) {
                double acc = 0.0;
                const double *row = St + (size_t)m * V;
                for (int c = 0; c < V; ++c) acc += row[c] * dot[c];
                dq[(size_t)t * K + m] = acc;
            }
            /* dS_t = (carried) + q_t^T do_t */
            for (int m = 0; m < K; ++m) {
                double *row = dS + (size_t)m * V;
                const double qm = qt[m];
                for (int c = 0; c < V; ++c) row[c] += qm * dot[c];
            }
            for (int m = 0; m < K; ++m) {
                double acc_k = 0.0, acc_a = 0.0;
                const double *row = dS + (size_t)m * V, *prow = Sp + (size_t)m * V;
                for (int c = 0; c < V; ++c) { acc_k += row[c] * vt[c]; acc_a += row[c] * prow[c]; }
                dk[(size_t)t * K + m] = acc_k;
                dg[(size_t)t * K + m] = exp(gt[m]) * acc_a;   /* d log alpha = alpha * d alpha */
            }
            for (int c = 0; c < V; ++c) {
                double acc = 0.0;
                for (int m = 0; m < K; ++m) acc += dS[(size_t)m * V + c] * kt[m];
                dv[(size_t)t * V + c] = acc;
            }
            for (int m = 0; m < K; ++m) {
                const double a = exp(gt[m]);
                double *row = dS + (size_t)m * V;
                for (int c = 0; c < V; ++c) row[c] *= a;
            }
        }
    }
    if (J->dh0) memcpy(J->dh0 + u * KV, dS, KV * sizeof(double));
    free(ckpt); free(seg); free(dS);
}

typedef void (*unit_fn)(job_t *, int);
typedef struct { job_t *J; unit_fn fn; } worker_arg;

static void *worker(void *p)
{
    worker_arg *a = (worker_arg *)p;
    for (;;) {
        pthread_mutex_lock(&a->J->mu);
        const int u = a->J->next_unit++;
        pthread_mutex_unlock(&a->J->mu);
        if (u >= a->J->B * a->J->H) break;
        a->fn(a->J, u);
    }
    return NULL;
}

static int run(job_t *J, unit_fn fn, int nthreads)
{
    const int units = J->B * J->H;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > units) nthreads = units;
    J->next_unit = 0;
    J->error = 0;
    pthread_mutex_init(&J->mu, NULL);
    worker_arg a = {J, fn};
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, worker, &a);
    worker(&a);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&J->mu);
    return J->error;
}

static int bad_shape(int B, int H, int T, int K, int V)
{
    return B < 0 || H < 0 || T < 0 || K <= 0 || V <= 0;
}

int oracle_fwd(int B, int H, int T, int K, int V, const double *q, const double *k, const double *v,
               const double *log_alpha, const double *h0, double *o, double *final_state, int nthreads)
{
    if (bad_shape(B, H, T, K, V)) return 1;
    job_t J;
    memset(&J, 0, sizeof(J));
    J.B = B; J.H = H; J.T = T; J.K = K; J.V = V;
    J.q = q; J.k = k; J.v = v; J.g = log_alpha; J.h0 = h0; J.o = o; J.final_state = final_state;
    return run(&J, fwd_unit, nthreads);
}

int oracle_bwd(int B, int H, int T, int K, int V, const double *q, const double *k, const double *v,
               const double *log_alpha, const double *h0, const double *d_out, const double *d_final,
               double *dq, double *dk, double *dv, double *dlog_alpha, double *dh0, int nthreads)
{
    if (bad_shape(B, H, T, K, V)) return 1;
    job_t J;
    memset(&J, 0, sizeof(J));
    J.B = B; J.H = H; J.T = T; J.K = K; J.V = V;
    J.q = q; J.k = k; J.v = v; J.g = log_alpha; J.h0 = h0; J.d_out = d_out; J.d_final = d_final;
    J.dq = dq; J.dk = dk; J.dv = dv; J.dg = dlog_alpha; J.dh0 = dh0;
    return run(&J, bwd_unit, nthreads);
}

/* One decode step for every (b,h): S <- diag(exp(g)) S + k^T v; o = q S. */
int oracle_step(int B, int H, int K, int V, const double *q, const double *k, const double *v,
                const double *log_alpha, double *state, double *o)
{
    if (bad_shape(B, H, 1, K, V)) return 1;
    const size_t KV = (size_t)K * V;
    for (int u = 0; u < B * H; ++u) {
        step_state(state + u * KV, k + (size_t)u * K, v + (size_t)u * V, log_alpha + (size_t)u * K, K, V);
        read_out(state + u * KV, q + (size_t)u * K, o + (size_t)u * V, K, V);
    }
    return 0;
}
