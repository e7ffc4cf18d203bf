/*
 * gla_beta_oracle.c -- fp64 CPU oracle for GLA with BOTH gates (arXiv 2312.06635, the general form).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The CUDA product path never links, imports or calls it and
 * shares no code with it.
 *
 * What it computes: the paper's RECURRENT form with the outer-product gate of P:171,
 *
 *     G_t = alpha_t^T beta_t,  alpha_t = exp(log_alpha_t) in R^{d_k},  beta_t = exp(log_beta_t) in R^{d_v}
 *                                                        P:171 (gates applied in log space)
 *     S_0 = h0 (zeros if absent)                          P:88 footnote
 *     S_t = G_t (.) S_{t-1} + k_t^T v_t                   P:188 Eq. gla_recurrence
 *     o_t = q_t S_t
 *     final_state = S_T
 *
 * (gla_oracle.c is the beta == 1 special case, kept separate and unchanged.)  Backward: reverse mode
 * of the recurrence above (the paper gives none), adjoint dS of S_t:
 *
 *     dS = d_final_state (or 0)
 *     for t = T..1:  dS += q_t^T do_t
 *                    dq_t = S_t do_t^T,  dk_t = dS v_t^T,  dv_t = k_t dS
 *                    dlog_alpha_t[m] = sum_j G_t[m][j] S_{t-1}[m][j] dS[m][j]      (d/dlog alpha of G (.) S_{t-1})
 *                    dlog_beta_t[j]  = sum_m G_t[m][j] S_{t-1}[m][j] dS[m][j]
 *                    dS = G_t (.) dS
 *     d_initial_state = dS
 *
 * Plain loops in fp64, ascending summation order (deterministic), states recomputed from checkpoints every
 * 64 steps.  Layout: q, k, log_alpha [B,H,T,K]; v, log_beta, o, d_out [B,H,T,V]; states [B,H,K,V].
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define BETA_CKPT 64

typedef struct {
    int B, H, T, K, V;
    const double *q, *k, *v, *ga, *gb, *h0, *d_out, *d_final;
    double *o, *final_state, *dq, *dk, *dv, *dga, *dgb, *dh0;
    int next_unit, error;
    pthread_mutex_t mu;
} bjob_t;

/* S <- (alpha^T beta) (.) S + k^T v */
static void bstep(double *S, const double *kt, const double *vt, const double *gat, const double *gbt, int K, int V)
{
    for (int m = 0; m < K; ++m) {
        const double a = exp(gat[m]), km = kt[m];
        double *row = S + (size_t)m * V;
        for (int j = 0; j < V; ++j) row[j] = a * exp(gbt[j]) * row[j] + km * vt[j];
    }
}

/* o_t = q_t S_t */
static void bread(const double *S, const double *qt, double *ot, int K, int V)
{
    for (int j = 0; j < V; ++j) ot[j] = 0.0;
    for (int m = 0; m < K; ++m)
        for (int j = 0; j < V; ++j) ot[j] += qt[m] * S[(size_t)m * V + j];
}

static void bfwd_unit(bjob_t *J, int u)
{
    const int T = J->T, K = J->K, V = J->V;
    const size_t KV = (size_t)K * V;
    const double *q = J->q + (size_t)u * T * K, *k = J->k + (size_t)u * T * K, *ga = J->ga + (size_t)u * T * K;
    const double *v = J->v + (size_t)u * T * V, *gb = J->gb + (size_t)u * T * V;
    double *S = (double *)malloc(KV * sizeof(double));
    if (!S) { J->error = 1; return; }
    if (J->h0) memcpy(S, J->h0 + u * KV, KV * sizeof(double));
    else memset(S, 0, KV * sizeof(double));
    for (int t = 0; t < T; ++t) {
        bstep(S, k + (size_t)t * K, v + (size_t)t * V, ga + (size_t)t * K, gb + (size_t)t * V, K, V);
        if (J->o) bread(S, q + (size_t)t * K, J->o + ((size_t)u * T + t) * V, K, V);
    }
    if (J->final_state) memcpy(J->final_state + u * KV, S, KV * sizeof(double));
    free(S);
}

static void bbwd_unit(bjob_t *J, int u)
{
    const int T = J->T, K = J->K, V = J->V;
    const size_t KV = (size_t)K * V;
    const double *q = J->q + (size_t)u * T * K, *k = J->k + (size_t)u * T * K, *ga = J->ga + (size_t)u * T * K;
    const double *v = J->v + (size_t)u * T * V, *gb = J->gb + (size_t)u * T * V;
    const double *dO = J->d_out + (size_t)u * T * V;
    double *dq = J->dq + (size_t)u * T * K, *dk = J->dk + (size_t)u * T * K, *dga = J->dga + (size_t)u * T * K;
    double *dv = J->dv + (size_t)u * T * V, *dgb = J->dgb + (size_t)u * T * V;
    const int nseg = (T + BETA_CKPT - 1) / BETA_CKPT;
    double *ckpt = (double *)malloc((size_t)(nseg + 1) * KV * sizeof(double));
    double *seg = (double *)malloc((size_t)(BETA_CKPT + 1) * KV * sizeof(double));
    double *dS = (double *)malloc(KV * sizeof(double));
    if (!ckpt || !seg || !dS) { J->error = 1; free(ckpt); free(seg); free(dS); return; }
    if (J->h0) memcpy(ckpt, J->h0 + u * KV, KV * sizeof(double));
    else memset(ckpt, 0, KV * sizeof(double));
    for (int j = 0; j < nseg; ++j) {            /* forward sweep keeping S_{64 j} */
        double *nxt = ckpt + (size_t)(j + 1) * KV;
        memcpy(nxt, ckpt + (size_t)j * KV, KV * sizeof(double));
        const int t1 = (j + 1) * BETA_CKPT < T ? (j + 1) * BETA_CKPT : T;
        for (int t = j * BETA_CKPT; t < t1; ++t)
            bstep(nxt, k + (size_t)t * K, v + (size_t)t * V, ga + (size_t)t * K, gb + (size_t)t * V, K, V);
    }
    if (J->d_final) memcpy(dS, J->d_final + u * KV, KV * sizeof(double));
    else memset(dS, 0, KV * sizeof(double));
    for (int j = nseg - 1; j >= 0; --j) {
        const int t0 = j * BETA_CKPT, t1 = (j + 1) * BETA_CKPT < T ? (j + 1) * BETA_CKPT : T;
        memcpy(seg, ckpt + (size_t)j * KV, KV * sizeof(double));
        for (int t = t0; t < t1; ++t) {
            memcpy(seg + (size_t)(t - t0 + 1) * KV, seg + (size_t)(t - t0) * KV, KV * sizeof(double));
            bstep(seg + (size_t)(t - t0 + 1) * KV, k + (size_t)t * K, v + (size_t)t * V, ga + (size_t)t * K,
                  gb + (size_t)t * V, K, V);
        }
        for (int t = t1 - 1; t >= t0; --t) {
            const double *St = seg + (size_t)(t - t0 + 1) * KV, *Sp = seg + (size_t)(t - t0) * KV;
            const double *qt = q + (size_t)t * K, *kt = k + (size_t)t * K, *gat = ga + (size_t)t * K;
            const double *vt = v + (size_t)t * V, *gbt = gb + (size_t)t * V, *dot = dO + (size_t)t * V;
            for (int m = 0; m < K; ++m) {       /* dq_t = S_t do_t^T */
                double acc = 0.0;
                for (int c = 0; c < V; ++c) acc += St[(size_t)m * V + c] * dot[c];
                dq[(size_t)t * K + m] = acc;
            }
            for (int m = 0; m < K; ++m)         /* dS += q_t^T do_t */
                for (int c = 0; c < V; ++c) dS[(size_t)m * V + c] += qt[m] * dot[c];
            for (int c = 0; c < V; ++c) dgb[(size_t)t * V + c] = 0.0;
            for (int m = 0; m < K; ++m) {
                double acc_k = 0.0, acc_a = 0.0;
                const double a = exp(gat[m]);
                for (int c = 0; c < V; ++c) {
                    const double w = a * exp(gbt[c]) * Sp[(size_t)m * V + c] * dS[(size_t)m * V + c];
                    acc_k += dS[(size_t)m * V + c] * vt[c];
                    acc_a += w;
                    dgb[(size_t)t * V + c] += w;
                }
                dk[(size_t)t * K + m] = acc_k;
                dga[(size_t)t * K + m] = acc_a;
            }
            for (int c = 0; c < V; ++c) {       /* dv_t = k_t dS */
                double acc = 0.0;
                for (int m = 0; m < K; ++m) acc += dS[(size_t)m * V + c] * kt[m];
                dv[(size_t)t * V + c] = acc;
            }
            for (int m = 0; m < K; ++m) {       /* dS <- G_t (.) dS */
                const double a = exp(gat[m]);
                for (int c = 0; c < V; ++c) dS[(size_t)m * V + c] *= a * exp(gbt[c]);
            }
        }
    }
    if (J->dh0) memcpy(J->dh0 + u * KV, dS, KV * sizeof(double));
    free(ckpt); free(seg); free(dS);
}

typedef void (*bunit_fn)(bjob_t *, int);
typedef struct { bjob_t *J; bunit_fn fn; } bworker_arg;

static void *bworker(void *p)
{
    bworker_arg *a = (bworker_arg *)p;
    for (;;) {
        pthread_mutex_lock(&a->J->mu);
        const int u = a->J->next_unit++;
        pthread_mutex_unlock(&a->J->mu);
        if (u >= a->J->B * a->J->H) break;
        a->fn(a->J, u);
    }
    return NULL;
}

static int brun(bjob_t *J, bunit_fn fn, int nthreads)
{
    const int units = J->B * J->H;
    if (nthreads < 1) nthreads = 1;
    if (nthreads > units) nthreads = units;
    J->next_unit = 0;
    J->error = 0;
    pthread_mutex_init(&J->mu, NULL);
    bworker_arg a = {J, fn};
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)(nthreads > 0 ? nthreads : 1));
    for (int i = 1; i < nthreads; ++i) pthread_create(&th[i], NULL, bworker, &a);
    bworker(&a);
    for (int i = 1; i < nthreads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&J->mu);
    return J->error;
}

int oracle_fwd_beta(int B, int H, int T, int K, int V, const double *q, const double *k, const double *v,
                    const double *log_alpha, const double *log_beta, const double *h0, double *o,
                    double *final_state, int nthreads)
{
    if (B < 0 || H < 0 || T < 0 || K <= 0 || V <= 0) return 1;
    bjob_t J;
    memset(&J, 0, sizeof(J));
    J.B = B; J.H = H; J.T = T; J.K = K; J.V = V;
    J.q = q; J.k = k; J.v = v; J.ga = log_alpha; J.gb = log_beta; J.h0 = h0; J.o = o; J.final_state = final_state;
    return brun(&J, bfwd_unit, nthreads);
}

int oracle_bwd_beta(int B, int H, int T, int K, int V, const double *q, const double *k, const double *v,
                    const double *log_alpha, const double *log_beta, const double *h0, const double *d_out,
                    const double *d_final, double *dq, double *dk, double *dv, double *dlog_alpha,
                    double *dlog_beta, double *dh0, int nthreads)
{
    if (B < 0 || H < 0 || T < 0 || K <= 0 || V <= 0) return 1;
    bjob_t J;
    memset(&J, 0, sizeof(J));
    J.B = B; J.H = H; J.T = T; J.K = K; J.V = V;
    J.q = q; J.k = k; J.v = v; J.ga = log_alpha; J.gb = log_beta; J.h0 = h0; J.d_out = d_out; J.d_final = d_final;
    J.dq = dq; J.dk = dk; J.dv = dv; J.dga = dlog_alpha; J.dgb = dlog_beta; J.dh0 = dh0;
    return brun(&J, bbwd_unit, nthreads);
}

/* One decode step with both gates for every (b,h): S <- (alpha^T beta) (.) S + k^T v; o = q S. */
int oracle_step_beta(int B, int H, int K, int V, const double *q, const double *k, const double *v,
                     const double *log_alpha, const double *log_beta, double *state, double *o)
{
    if (B < 0 || H < 0 || K <= 0 || V <= 0) return 1;
    const size_t KV = (size_t)K * V;
    for (int u = 0; u < B * H; ++u) {
        bstep(state + u * KV, k + (size_t)u * K, v + (size_t)u * V, log_alpha + (size_t)u * K,
              log_beta + (size_t)u * V, K, V);
        bread(state + u * KV, q + (size_t)u * K, o + (size_t)u * V, K, V);
    }
    return 0;
}
