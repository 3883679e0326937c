/*
 * cosched_oracle.c -- CPU restatement of the reference's pair x knob sweep.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library; it is
 * the checker, never the product.  The product path (paper_2405_03831_b200/)
 * never links or imports it and has no CPU fallback.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below
 * against fixtures produced by the UNMODIFIED reference (tests/golden/
 * make_golden.py): the full 256-app graph, the 20-app graphs at 400/350 W,
 * seeded samples at N=1024 (five budgets) and N=4096 (default and fine grid).
 *
 * Everything is IEEE fp64, as in the reference (numpy float64).  Dot products
 * use explicit fma() in a fixed order (compile with -ffp-contract=off), the
 * same order the GPU's exact fp64 path uses, so those GPU outputs compare
 * bit-for-bit against this file.  Two forms:
 *
 *  - orc_predict / orc_decide_pair: the direct form.  normalize_input
 *    (core.py:334-377) builds the 40-vector, forward_batch (fnn.py:161-165)
 *    evaluates 40-18-18-1 with ReLU on every layer, slowdown() floors at 0.5
 *    (estimator.py:98-109), corun_time = max over members with member 2 seeing
 *    reversed partitions (estimator.py:112-129), optimize_corun takes the
 *    first strict minimum in enumeration order (hwopt.py:44-65), solorun_time
 *    takes each job's first-minimum split and sums (0.0 + t1) + t2
 *    (estimator.py:139-180), decide_pair flags co-run on <= (hwopt.py:77-87).
 *
 *  - orc_sweep: the factored form of SURVEY.md §8c.  Layer 1 splits exactly
 *    into a per-app partial of the primary block (A), a per-app partial of the
 *    co-runner block (B) and a per-knob partial (K), so each (pair, config)
 *    evaluation is b1 + A_i + B_j + K_c followed by layer 2 and the head.  It is
 *    the same arithmetic up to fp64 summation order (checked <= 1e-12 relative
 *    against the reference fixtures) and is ~3x cheaper; it is also the CPU
 *    baseline that bench.py times ("kind": "port"), threaded over pair ranges.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define NF 18      /* counters per job            core.py:18 */
#define IN 40      /* model input width           core.py:21 */
#define HD 18      /* hidden width                fnn.py:19  */
#define FLOOR 0.5  /* SLOWDOWN_FLOOR              estimator.py:33 */

typedef struct {
    double w1[HD * IN];
    double b1[HD];
    double w2[HD * HD];
    double b2[HD];
    double wo[HD];
    double bo;
    double bounds[2 * NF];
} orc_net;

static double clip01(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

/* normalize_input (core.py:367-377): knob[4] = [cores1/32, gpcs1/8, ccap/250,
 * gcap/250] already divided by the caller; co == NULL zeroes the co block. */
static void orc_input(const orc_net *net, const double *f1, const double *co,
                      const double *knob, double *x) {
    for (int k = 0; k < 4; ++k) x[k] = knob[k];
    for (int k = 0; k < NF; ++k) x[4 + k] = clip01(f1[k] / net->bounds[k]);
    for (int k = 0; k < NF; ++k)
        x[4 + NF + k] = co ? clip01(co[k] / net->bounds[NF + k]) : 0.0;
}

/* Layers 2 + head from a layer-1 pre-activation z1 (fnn.py:163-165). */
static double orc_head(const orc_net *net, const double *z1) {
    double h1[HD], y = 0.0;
    for (int k = 0; k < HD; ++k) h1[k] = z1[k] > 0.0 ? z1[k] : 0.0;
    for (int o = 0; o < HD; ++o) {
        double acc = 0.0;
        for (int k = 0; k < HD; ++k) acc = fma(h1[k], net->w2[o * HD + k], acc);
        acc = acc + net->b2[o];
        y = fma(acc > 0.0 ? acc : 0.0, net->wo[o], y);
    }
    y = y + net->bo;
    return y > 0.0 ? y : 0.0;
}

/* FnnSlowdownModel.predict_slowdown (estimator.py:65-67), unfloored. */
double orc_predict(const orc_net *net, const double *f1, const double *co, const double *knob) {
    double x[IN], z1[HD];
    orc_input(net, f1, co, knob, x);
    for (int h = 0; h < HD; ++h) {
        double acc = 0.0;
        for (int k = 0; k < IN; ++k) acc = fma(x[k], net->w1[h * IN + k], acc);
        z1[h] = acc + net->b1[h];
    }
    return orc_head(net, z1);
}

static double floored(double pred, int64_t *clamps) {
    if (pred < FLOOR) {           /* estimator.py:106-109 */
        if (clamps) ++*clamps;
        return FLOOR;
    }
    return pred;
}

/* Decision record shared by both forms. */
typedef struct {
    int32_t corun_index;    /* index into the caller's config list */
    double corun_time;
    int32_t solo_split[2];  /* index into the caller's solo-split list */
    double solo_time;
    int32_t corun_chosen;
    double weight;
    double margin;          /* (second best - best) / best over configs; +inf if C == 1 */
} orc_decision;

/* hwopt.decide_pair (hwopt.py:77-87), direct form, one budget.
 * knob1/knob2: C x 4 normalized inputs for the member-1 view and the
 * reversed-partition member-2 view; solo_knob: S x 4. */
int orc_decide_pair(const orc_net *net, const double *fi, double ti, const double *fj,
                    double tj, const double *knob1, const double *knob2, int n_cfg,
                    const double *solo_knob, int n_solo, orc_decision *out, int64_t *clamps) {
    if (n_cfg <= 0) return -1;   /* hwopt.py:62-64: no co-run configs */
    if (n_solo <= 0) return -2;  /* estimator.py:165-167: unreachable */
    double best = 0.0, second = INFINITY;
    int arg = -1;
    for (int c = 0; c < n_cfg; ++c) {
        double t1 = floored(orc_predict(net, fi, fj, knob1 + 4 * c), clamps) * ti;
        double t2 = floored(orc_predict(net, fj, fi, knob2 + 4 * c), clamps) * tj;
        double t = t1 > t2 ? t1 : t2;                       /* estimator.py:129 */
        if (arg < 0 || t < best) {                          /* hwopt.py:59 */
            if (arg >= 0) second = best < second ? best : second;
            best = t; arg = c;
        } else if (t < second) {
            second = t;
        }
    }
    double total = 0.0;
    const double *fs[2] = {fi, fj};
    const double ts[2] = {ti, tj};
    for (int m = 0; m < 2; ++m) {
        double bt = 0.0; int bs = -1;
        for (int s = 0; s < n_solo; ++s) {
            double t = floored(orc_predict(net, fs[m], NULL, solo_knob + 4 * s), clamps) * ts[m];
            if (bs < 0 || t < bt) { bt = t; bs = s; }       /* estimator.py:175 */
        }
        total += bt;
        out->solo_split[m] = bs;
    }
    out->corun_index = arg;
    out->corun_time = best;
    out->solo_time = total;
    out->corun_chosen = best <= total;                      /* hwopt.py:86 */
    out->weight = out->corun_chosen ? best : total;         /* hwopt.py:39-41 */
    out->margin = isinf(second) ? INFINITY : (second - best) / best;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* Factored sweep over a pair range, L budgets at once.                     */
/* ------------------------------------------------------------------------ */

typedef struct {
    const orc_net *net;
    int n;                    /* apps */
    const double *base_time;  /* n */
    const double *A, *B;      /* n x HD: primary / co-runner layer-1 partials */
    const double *K1, *K2;    /* G x HD: knob partials, member-1 / member-2 view, b1 folded */
    const uint32_t *mask;     /* G: bit l = config valid in budget l */
    int G, L;
    const double *solo_time;  /* L x n */
    int64_t p0, p1;           /* pair range [p0, p1) of this worker */
    int64_t p_begin, P;       /* output base and stride per budget */
    int32_t *corun_index;     /* L x P */
    double *corun_time, *weight, *margin;
    uint8_t *chosen;
    int64_t clamps[32];
} orc_job;

static void pair_of(int64_t p, int n, int *i, int *j) {
    /* row-major i < j enumeration (scheduler.py:61) */
    int64_t row = 0, start = 0;
    while (start + (n - 1 - row) <= p) { start += n - 1 - row; ++row; }
    *i = (int)row;
    *j = (int)(row + 1 + (p - start));
}

static void *sweep_worker(void *arg) {
    orc_job *jb = (orc_job *)arg;
    const orc_net *net = jb->net;
    int i, j;
    if (jb->p0 >= jb->p1) return NULL;
    pair_of(jb->p0, jb->n, &i, &j);
    double z[HD];
    double best[32], second[32];
    int arg_[32];
    for (int64_t p = jb->p0; p < jb->p1; ++p) {
        const double *Ai = jb->A + (size_t)i * HD, *Aj = jb->A + (size_t)j * HD;
        const double *Bi = jb->B + (size_t)i * HD, *Bj = jb->B + (size_t)j * HD;
        double ti = jb->base_time[i], tj = jb->base_time[j];
        for (int l = 0; l < jb->L; ++l) { arg_[l] = -1; best[l] = 0.0; second[l] = INFINITY; }
        for (int c = 0; c < jb->G; ++c) {
            uint32_t m = jb->mask[c];
            if (!m) continue;
            const double *k1 = jb->K1 + (size_t)c * HD, *k2 = jb->K2 + (size_t)c * HD;
            for (int h = 0; h < HD; ++h) z[h] = (Ai[h] + Bj[h]) + k1[h];
            double y1 = orc_head(net, z);
            for (int h = 0; h < HD; ++h) z[h] = (Aj[h] + Bi[h]) + k2[h];
            double y2 = orc_head(net, z);
            int c1 = y1 < FLOOR, c2 = y2 < FLOOR;
            double t1 = (c1 ? FLOOR : y1) * ti, t2 = (c2 ? FLOOR : y2) * tj;
            double t = t1 > t2 ? t1 : t2;
            for (int l = 0; l < jb->L; ++l) {
                if (!((m >> l) & 1u)) continue;
                jb->clamps[l] += c1 + c2;
                if (arg_[l] < 0 || t < best[l]) {
                    if (arg_[l] >= 0 && best[l] < second[l]) second[l] = best[l];
                    best[l] = t; arg_[l] = c;
                } else if (t < second[l]) {
                    second[l] = t;
                }
            }
        }
        for (int l = 0; l < jb->L; ++l) {
            int64_t o = (int64_t)l * jb->P + (p - jb->p_begin);
            double solo = (0.0 + jb->solo_time[(size_t)l * jb->n + i]) +
                          jb->solo_time[(size_t)l * jb->n + j];
            int ch = arg_[l] >= 0 && best[l] <= solo;
            jb->corun_index[o] = arg_[l];
            jb->corun_time[o] = arg_[l] >= 0 ? best[l] : NAN;
            jb->chosen[o] = (uint8_t)ch;
            jb->weight[o] = ch ? best[l] : solo;
            jb->margin[o] = isinf(second[l]) ? INFINITY : (second[l] - best[l]) / best[l];
        }
        if (++j == jb->n) { ++i; j = i + 1; }
    }
    return NULL;
}

/* Per-app factored tables (fp64): A = W1[:,4:22] n1(f), B = W1[:,22:40] n2(f). */
void orc_app_tables(const orc_net *net, const double *feats, int n, double *A, double *B) {
    for (int a = 0; a < n; ++a) {
        const double *f = feats + (size_t)a * NF;
        for (int h = 0; h < HD; ++h) {
            double sa = 0.0, sb = 0.0;
            for (int k = 0; k < NF; ++k) {
                sa = fma(clip01(f[k] / net->bounds[k]), net->w1[h * IN + 4 + k], sa);
                sb = fma(clip01(f[k] / net->bounds[NF + k]), net->w1[h * IN + 4 + NF + k], sb);
            }
            A[(size_t)a * HD + h] = sa;
            B[(size_t)a * HD + h] = sb;
        }
    }
}

/* Knob partials with b1 folded in: K = W1[:,0:4] knob + b1. */
void orc_knob_table(const orc_net *net, const double *knob, int g, double *K) {
    for (int c = 0; c < g; ++c)
        for (int h = 0; h < HD; ++h) {
            double s = 0.0;
            for (int k = 0; k < 4; ++k) s = fma(knob[4 * c + k], net->w1[h * IN + k], s);
            K[(size_t)c * HD + h] = s + net->b1[h];
        }
}

/* Per-app best solo split per budget (estimator.py:139-180, hoisted: it does
 * not depend on the partner).  solo_knob: S_tot x 4, budget l owns rows
 * [solo_off[l], solo_off[l+1]).  Returns the clamp count of ONE evaluation
 * of every (app, split); build_graph re-evaluates it (n - 1) times per app. */
int64_t orc_solo(const orc_net *net, const double *A, const double *base_time, int n,
                 const double *solo_knob, const int32_t *solo_off, int L,
                 double *solo_time, int32_t *solo_split) {
    int S = solo_off[L];
    double *KS = (double *)malloc(sizeof(double) * (size_t)(S > 0 ? S : 1) * HD);
    orc_knob_table(net, solo_knob, S, KS);
    int64_t clamps = 0;
    double z[HD];
    for (int l = 0; l < L; ++l)
        for (int a = 0; a < n; ++a) {
            double bt = INFINITY; int bs = -1;
            for (int s = solo_off[l]; s < solo_off[l + 1]; ++s) {
                for (int h = 0; h < HD; ++h) z[h] = A[(size_t)a * HD + h] + KS[(size_t)s * HD + h];
                double y = orc_head(net, z);
                if (y < FLOOR) { ++clamps; y = FLOOR; }
                double t = y * base_time[a];
                if (bs < 0 || t < bt) { bt = t; bs = s - solo_off[l]; }
            }
            solo_time[(size_t)l * n + a] = bs < 0 ? NAN : bt;
            solo_split[(size_t)l * n + a] = bs;
        }
    free(KS);
    return clamps;
}

/* The factored sweep over pairs [p_begin, p_end) for L budgets, threaded.
 * Outputs are L x (p_end - p_begin), budget-major.  clamps_out[l] receives
 * the co-run clamp count of budget l (solo clamps: see orc_solo). */
int orc_sweep(const orc_net *net, const double *feats, const double *base_time, int n,
              const double *knob1, const double *knob2, const uint32_t *mask, int G, int L,
              const double *solo_time, int64_t p_begin, int64_t p_end, int nthreads,
              int32_t *corun_index, double *corun_time, uint8_t *chosen, double *weight,
              double *margin, int64_t *clamps_out) {
    if (L < 1 || L > 32 || n < 2) return -1;
    int64_t P = p_end - p_begin;
    if (P < 0) return -1;
    double *A = (double *)malloc(sizeof(double) * (size_t)n * HD);
    double *B = (double *)malloc(sizeof(double) * (size_t)n * HD);
    double *K1 = (double *)malloc(sizeof(double) * (size_t)(G > 0 ? G : 1) * HD);
    double *K2 = (double *)malloc(sizeof(double) * (size_t)(G > 0 ? G : 1) * HD);
    orc_app_tables(net, feats, n, A, B);
    orc_knob_table(net, knob1, G, K1);
    orc_knob_table(net, knob2, G, K2);
    if (nthreads < 1) nthreads = 1;
    if (nthreads > 256) nthreads = 256;
    orc_job *jobs = (orc_job *)calloc((size_t)nthreads, sizeof(orc_job));
    pthread_t *tid = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        orc_job *jb = &jobs[t];
        jb->net = net; jb->n = n; jb->base_time = base_time;
        jb->A = A; jb->B = B; jb->K1 = K1; jb->K2 = K2; jb->mask = mask;
        jb->G = G; jb->L = L; jb->solo_time = solo_time;
        jb->p0 = p_begin + P * t / nthreads;
        jb->p1 = p_begin + P * (t + 1) / nthreads;
        jb->p_begin = p_begin; jb->P = P;
        jb->corun_index = corun_index; jb->corun_time = corun_time; jb->chosen = chosen;
        jb->weight = weight; jb->margin = margin;
        if (nthreads > 1) pthread_create(&tid[t], NULL, sweep_worker, jb);
        else sweep_worker(jb);
    }
    if (clamps_out) memset(clamps_out, 0, sizeof(int64_t) * (size_t)L);
    for (int t = 0; t < nthreads; ++t) {
        if (nthreads > 1) pthread_join(tid[t], NULL);
        if (clamps_out)
            for (int l = 0; l < L; ++l) clamps_out[l] += jobs[t].clamps[l];
    }
    free(jobs); free(tid); free(A); free(B); free(K1); free(K2);
    return 0;
}

/* Reference matching weight helper for tests: sum of w[i][j] over sorted pairs
 * (matcher.py:66-69). */
double orc_matching_weight(const double *w, int n, const int32_t *pairs, int m) {
    double s = 0.0;
    for (int k = 0; k < m; ++k) {
        int a = pairs[2 * k], b = pairs[2 * k + 1];
        int i = a < b ? a : b, j = a < b ? b : a;
        s += w[(size_t)i * n + j];
    }
    return s;
}
