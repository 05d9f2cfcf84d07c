/*
 * ekya_oracle.c -- TEST INFRASTRUCTURE ONLY (see ekya_oracle.h).
 *
 * A plain, slow, single-threaded CPU implementation of what the Ekya thief
 * scheduler's hot path computes (arXiv 2012.10557, final paper P:441-1738):
 *
 *   EstimateAccuracy   (Alg. 2 line 7; closed form of draft P:73)
 *   PickConfigs        (Algorithm 2)
 *   fair_allocation    (Alg. 1 line 2; reading C9)
 *   Thief scheduler    (Algorithm 1) in two readings (C12):
 *                        LITERAL  = the pseudocode verbatim,
 *                        STEEPEST = best single-Delta steal per step
 *   Eq. 1 brute force for tiny instances
 *   History profiler   (draft appendix; P:30 five clusters)
 *
 * Arithmetic: IEEE-754 binary32, round-to-nearest-even, ONE rounding per
 * operation (compile with -ffp-contract=off, no fast-math).  The precision is
 * fp32 because BASELINE.json's north star fixes the objective in fp32 and
 * demands identical decisions; every decision (argmax, feasibility,
 * acceptance) is therefore taken in fp32 exactly as written here.  Sums of
 * per-stream accuracies are exact integers (Q32, reading C15).
 *
 * Nothing here is blocked, fused or reordered: every PickConfigs call
 * enumerates all (lambda, gamma) pairs of every stream; every thief candidate
 * re-runs a full PickConfigs.
 *
 * Parity status per function: see DESIGN.md section 4 ("pins").
 */
#include "ekya_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_LAMBDA_NONE 7
#define ORC_LMU_PAD 0xFFFFu

/* ------------------------------------------------------------------------ */
/* Rule 1 ("avoids configurations whose retraining durations exceed  */
/* ||T||"; P:1155 GPU-time per epoch at 100% GPU scaled by the allocation;  */
/* S:237 duration = cost / share).  t_r/||T|| = cost / (rt * delta * ||T||). */
/* ------------------------------------------------------------------------ */
float orc_retrain_fraction(float cost, int32_t rt, float uT)
{
    float denom = (float)rt * uT;          /* fl(float(rt) * uT) */
    float f = cost / denom;                /* fl(cost / denom)   */
    return f;
}

int32_t orc_gamma_feasible(float cost, int32_t rt, float uT)
{
    if (rt < 1) return 0;                  /* no GPU -> never finishes */
    float f = orc_retrain_fraction(cost, rt, uT);
    return f <= 1.0f;                      /* t_r == ||T|| is feasible (C5) */
}

/* Rule 2: window-averaged accuracy of retraining with gamma, as a fraction of
 * the inference factor: draft P:73 base_acc = ((tau - t) a + (T - tau) A)/T at
 * t = 0, i.e. f*stale + (1-f)*post, written as post - f*(post - stale). */
float orc_window_accuracy(float stale, float post, float cost, int32_t rt, float uT)
{
    float f = orc_retrain_fraction(cost, rt, uT);
    float diff = post - stale;
    float prod = f * diff;
    float g = post - prod;
    return g;
}

/* Rule 4: exact fixed-point value x * 2^32, rounded to nearest even. */
uint64_t orc_q32(float x)
{
    float y = x * 4294967296.0f;           /* exact: power-of-two scaling */
    return (uint64_t)llrintf(y);           /* default rounding mode = RNE */
}

static float orc_mean_from_q32(uint64_t s, int32_t n)
{
    double m = (double)s / ((double)n * 4294967296.0);
    return (float)m;
}

/* Alg. 2 lines 3-4: lambda pool = {resource_cost < alloc  &&
 * accuracy >= a_MIN}; pick max accuracy (lowest index on ties, C7).
 * Keep-up test in integer units (C2): ri >= lam_min_units.
 * Accuracy of lambda = stale * factor (C1).  Returns -1 if the pool is empty. */
static int orc_lambda_star(float stale, const uint16_t* lmu, const float* lf, int nl,
                           int32_t ri, float a_min)
{
    int best = -1;
    float best_acc = 0.0f;
    for (int l = 0; l < nl; ++l) {
        if (lmu[l] == ORC_LMU_PAD) continue;
        if (ri < (int32_t)lmu[l]) continue;
        float acc = stale * lf[l];
        if (!(acc >= a_min)) continue;
        if (best < 0 || acc > best_acc) {
            best = l;
            best_acc = acc;
        }
    }
    return best;
}

/* Rule 3: the per-stream part of PickConfigs (Alg. 2 lines 3-14). */
float orc_stream_value(const orc_dims* d, float stale, const float* cost, const float* post,
                       const uint16_t* lmu, const float* lf, int32_t rt, int32_t ri, uint8_t* cfg)
{
    int l = orc_lambda_star(stale, lmu, lf, d->n_lambda, ri, d->a_min);
    if (l < 0) {                           /* C8: no admissible lambda */
        if (cfg) *cfg = (uint8_t)(ORC_LAMBDA_NONE << 5);
        return 0.0f;
    }
    float fac = lf[l];
    /* gamma = empty set first (index 0, C6): the stale model all window */
    float best = fac * stale;
    int bg = 0;
    for (int g = 0; g < d->n_gamma; ++g) {
        if (!orc_gamma_feasible(cost[g], rt, d->unit_gpu_seconds)) continue;
        float w = orc_window_accuracy(stale, post[g], cost[g], rt, d->unit_gpu_seconds);
        float a = fac * w;                 /* EstimateAccuracy(gamma, lambda, rt, T) */
        if (a > best) {                    /* strict '>': lowest index wins */
            best = a;
            bg = g + 1;
        }
    }
    if (cfg) *cfg = (uint8_t)(bg | (l << 5));
    return best;
}

/* ------------------------------------------------------------------------ */
/* instance access + validation                                             */
/* ------------------------------------------------------------------------ */
typedef struct {
    const float* stale;    /* [V]     */
    const float* cost;     /* [V][nG] */
    const float* post;     /* [V][nG] */
    const uint16_t* lmu;   /* [V][nL] */
    const float* lf;       /* [V][nL] */
} orc_inst;

static orc_inst orc_instance(const orc_dims* d, int64_t b, const float* stale, const float* cost,
                             const float* post, const uint16_t* lmu, const float* lf)
{
    orc_inst in;
    int64_t V = d->n_streams;
    in.stale = stale + b * V;
    in.cost = cost ? cost + b * V * d->n_gamma : NULL;
    in.post = post ? post + b * V * d->n_gamma : NULL;
    in.lmu = lmu + b * V * d->n_lambda;
    in.lf = lf + b * V * d->n_lambda;
    return in;
}

static int orc_in01(float x) { return x >= 0.0f && x <= 1.0f; }

/* Data validity (error behaviour): stale in [0,1]; cost >= 0 or
 * +INF (padding); post in [0,1] where cost is finite; factor in [0,1] where
 * lam_min_units is not the padding value. */
static int orc_instance_valid(const orc_dims* d, const orc_inst* in)
{
    for (int v = 0; v < d->n_streams; ++v) {
        if (!orc_in01(in->stale[v])) return 0;
        for (int g = 0; g < d->n_gamma; ++g) {
            float c = in->cost[v * d->n_gamma + g];
            if (!(c >= 0.0f)) return 0;    /* NaN or negative */
            if (isinf(c)) continue;
            if (!orc_in01(in->post[v * d->n_gamma + g])) return 0;
        }
        for (int l = 0; l < d->n_lambda; ++l) {
            if (in->lmu[v * d->n_lambda + l] == ORC_LMU_PAD) continue;
            if (!orc_in01(in->lf[v * d->n_lambda + l])) return 0;
        }
    }
    return 1;
}

static int orc_dims_valid(const orc_dims* d)
{
    if (d->n_inst < 0 || d->n_streams < 1 || d->n_gamma < 0 || d->n_gamma > 31) return 0;
    if (d->n_lambda < 1 || d->n_lambda > 7) return 0;
    if (d->units < 1 || d->units > 65534 || d->steal_units < 1) return 0;
    if (!(d->unit_gpu_seconds > 0.0f) || isinf(d->unit_gpu_seconds)) return 0;
    if (isnan(d->a_min) || isinf(d->a_min)) return 0;
    return 1;
}

/* Objective of one full allocation (Alg. 2 return value, exact form C15). */
static uint64_t orc_pick(const orc_dims* d, const orc_inst* in, const int32_t* alloc,
                         uint8_t* cfg_out, float* val_out)
{
    uint64_t s = 0;
    for (int v = 0; v < d->n_streams; ++v) {
        uint8_t c = 0;
        float val = orc_stream_value(d, in->stale[v], in->cost + (int64_t)v * d->n_gamma,
                                     in->post + (int64_t)v * d->n_gamma,
                                     in->lmu + (int64_t)v * d->n_lambda,
                                     in->lf + (int64_t)v * d->n_lambda,
                                     alloc[2 * v + 1], alloc[2 * v], &c);
        if (cfg_out) cfg_out[v] = c;
        if (val_out) val_out[v] = val;
        s += orc_q32(val);
    }
    return s;
}

uint64_t orc_pickconfigs(const orc_dims* d, int64_t b, const float* stale, const float* cost,
                         const float* post, const uint16_t* lmu, const float* lf,
                         const int32_t* alloc, uint8_t* cfg_out, float* val_out)
{
    orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
    return orc_pick(d, &in, alloc, cfg_out, val_out);
}

/* C9: equal split over streams (remainder to the lowest-numbered streams),
 * then half to retraining (floor), the rest to inference. Job 2v = inference,
 * job 2v+1 = retraining (C10). */
void orc_fair(const orc_dims* d, int32_t* alloc)
{
    int32_t V = d->n_streams, U = d->units;
    for (int32_t v = 0; v < V; ++v) {
        int32_t share = U / V + (v < U % V ? 1 : 0);
        int32_t rt = share / 2;
        alloc[2 * v + 1] = rt;
        alloc[2 * v] = share - rt;
    }
}

/* ------------------------------------------------------------------------ */
/* GRID / LIST evaluators                                                   */
/* ------------------------------------------------------------------------ */
int64_t orc_eval_grid(const orc_dims* d, const float* stale, const float* cost, const float* post,
                      const uint16_t* lmu, const float* lf, float* out_grid, uint8_t* out_grid_cfg)
{
    if (!orc_dims_valid(d)) return -1;
    int64_t U = d->units, V = d->n_streams;
    int64_t ncell = (U + 1) * (U + 2) / 2;
    int64_t bad = 0;
    for (int64_t b = 0; b < d->n_inst; ++b) {
        orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
        int ok = orc_instance_valid(d, &in);
        if (!ok) ++bad;
        for (int64_t v = 0; v < V; ++v) {
            int64_t base = (b * V + v) * ncell;
            int64_t c = 0;
            for (int32_t rt = 0; rt <= U; ++rt) {
                for (int32_t ri = 0; ri + rt <= U; ++ri, ++c) {
                    uint8_t cfg = 0;
                    float val = 0.0f;
                    if (ok)
                        val = orc_stream_value(d, in.stale[v], in.cost + v * d->n_gamma,
                                               in.post + v * d->n_gamma, in.lmu + v * d->n_lambda,
                                               in.lf + v * d->n_lambda, rt, ri, &cfg);
                    out_grid[base + c] = val;
                    if (out_grid_cfg) out_grid_cfg[base + c] = cfg;
                }
            }
        }
    }
    return bad;
}

int64_t orc_eval_list(const orc_dims* d, const float* stale, const float* cost, const float* post,
                      const uint16_t* lmu, const float* lf, int32_t n_alloc, const uint16_t* alloc,
                      uint64_t* out_sum, float* out_mean, uint8_t* out_cfg)
{
    if (!orc_dims_valid(d) || n_alloc < 0) return -1;
    int64_t V = d->n_streams, J = 2 * V;
    int32_t* a = (int32_t*)malloc(sizeof(int32_t) * J);
    uint8_t* cfg = (uint8_t*)malloc(V);
    int64_t bad = 0;
    for (int64_t b = 0; b < d->n_inst; ++b) {
        orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
        int ok = orc_instance_valid(d, &in);
        for (int64_t n = 0; n < n_alloc; ++n) {
            const uint16_t* row = alloc + (b * n_alloc + n) * J;
            int64_t tot = 0;
            int row_ok = ok;
            for (int64_t j = 0; j < J; ++j) {
                a[j] = row[j];
                tot += row[j];
                if (row[j] > d->units) row_ok = 0;
            }
            if (tot > d->units) row_ok = 0;   /* Eq. 1 constraint 2 */
            uint64_t s = 0;
            memset(cfg, 0, V);
            if (row_ok) s = orc_pick(d, &in, a, cfg, NULL);
            else ++bad;
            int64_t o = b * n_alloc + n;
            out_sum[o] = s;
            if (out_mean) out_mean[o] = row_ok ? orc_mean_from_q32(s, d->n_streams) : 0.0f;
            if (out_cfg) memcpy(out_cfg + o * V, cfg, V);
        }
    }
    free(a);
    free(cfg);
    return bad;
}

/* ------------------------------------------------------------------------ */
/* Thief scheduler, Algorithm 1                               */
/* ------------------------------------------------------------------------ */

/* LITERAL: the pseudocode verbatim (C10 job order, C13 strict acceptance,
 * C14 victim floor). */
static uint64_t orc_thief_literal(const orc_dims* d, const orc_inst* in, int32_t* best,
                                  uint32_t* steps)
{
    int32_t J = 2 * d->n_streams, D = d->steal_units;
    int32_t* temp = (int32_t*)malloc(sizeof(int32_t) * J);
    orc_fair(d, best);                                     /* line 2 */
    uint64_t best_acc = orc_pick(d, in, best, NULL, NULL); /* line 3 */
    uint32_t n = 0;
    for (int32_t thief = 0; thief < J; ++thief) {          /* line 5 */
        for (int32_t victim = 0; victim < J; ++victim) {   /* line 6 */
            if (thief == victim) continue;                 /* line 7 */
            memcpy(temp, best, sizeof(int32_t) * J);       /* line 8 */
            for (;;) {                                     /* line 9 */
                temp[victim] -= D;                         /* line 10 */
                temp[thief] += D;                          /* line 11 */
                if (temp[victim] < 0) break;               /* lines 12-13 */
                uint64_t acc = orc_pick(d, in, temp, NULL, NULL); /* line 14 */
                if (acc > best_acc) {                      /* line 15 */
                    memcpy(best, temp, sizeof(int32_t) * J);
                    best_acc = acc;
                    ++n;
                } else {
                    break;
                }
            }
        }
    }
    free(temp);
    *steps = n;
    return best_acc;
}

/* STEEPEST: from the fair start, repeatedly apply the single Delta-steal
 * (thief t, victim w) that maximises the objective over ALL ordered pairs,
 * ties to the lexicographically smallest (t, w); stop when no steal strictly
 * improves (C12, north star "every candidate steal evaluated ... best one"). */
static uint64_t orc_thief_steepest(const orc_dims* d, const orc_inst* in, int32_t* alloc,
                                   uint32_t* steps)
{
    int32_t J = 2 * d->n_streams, D = d->steal_units;
    orc_fair(d, alloc);
    uint64_t cur = orc_pick(d, in, alloc, NULL, NULL);
    uint32_t n = 0;
    for (;;) {
        uint64_t best = cur;
        int32_t bt = -1, bw = -1;
        for (int32_t t = 0; t < J; ++t) {
            for (int32_t w = 0; w < J; ++w) {
                if (t == w || alloc[w] < D) continue;
                alloc[w] -= D;
                alloc[t] += D;
                uint64_t s = orc_pick(d, in, alloc, NULL, NULL);
                alloc[w] += D;
                alloc[t] -= D;
                if (s > best) {
                    best = s;
                    bt = t;
                    bw = w;
                }
            }
        }
        if (bt < 0) break;
        alloc[bw] -= D;
        alloc[bt] += D;
        cur = best;
        ++n;
    }
    *steps = n;
    return cur;
}

int64_t orc_thief(const orc_dims* d, const float* stale, const float* cost, const float* post,
                  const uint16_t* lmu, const float* lf, int32_t mode,
                  uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean,
                  uint32_t* out_steps)
{
    if (!orc_dims_valid(d) || (mode != 0 && mode != 1)) return -1;
    int64_t V = d->n_streams, J = 2 * V;
    int32_t* a = (int32_t*)malloc(sizeof(int32_t) * J);
    int64_t bad = 0;
    for (int64_t b = 0; b < d->n_inst; ++b) {
        orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
        uint64_t s = 0;
        uint32_t steps = 0;
        if (orc_instance_valid(d, &in)) {
            if (mode == 0) s = orc_thief_steepest(d, &in, a, &steps);
            else s = orc_thief_literal(d, &in, a, &steps);
            for (int64_t j = 0; j < J; ++j) out_alloc[b * J + j] = (uint16_t)a[j];
            orc_pick(d, &in, a, out_cfg + b * V, NULL);
            if (out_mean) out_mean[b] = orc_mean_from_q32(s, d->n_streams);
        } else {
            ++bad;
            memset(out_alloc + b * J, 0, sizeof(uint16_t) * J);
            memset(out_cfg + b * V, 0, V);
            if (out_mean) out_mean[b] = 0.0f;
        }
        out_sum[b] = s;
        if (out_steps) out_steps[b] = steps;
    }
    free(a);
    return bad;
}

/* ------------------------------------------------------------------------ */
/* Eq. 1 brute force: maximise the objective over every         */
/* allocation with sum <= U (constraint 2); per-job feasibility is inside   */
/* PickConfigs, which implies constraint 1 (C16); constraint 3 holds because */
/* PickConfigs picks exactly one (gamma, lambda) per stream.  Ties: the     */
/* lexicographically smallest allocation vector.                            */
/* ------------------------------------------------------------------------ */
typedef struct {
    const orc_dims* d;
    const orc_inst* in;
    int32_t* cur;
    int32_t* best;
    uint64_t best_s;
    int have;
} orc_bf;

static void orc_bf_rec(orc_bf* st, int32_t j, int32_t left)
{
    int32_t J = 2 * st->d->n_streams;
    if (j == J) {
        uint64_t s = orc_pick(st->d, st->in, st->cur, NULL, NULL);
        if (!st->have || s > st->best_s) {
            st->have = 1;
            st->best_s = s;
            memcpy(st->best, st->cur, sizeof(int32_t) * J);
        }
        return;
    }
    for (int32_t x = 0; x <= left; ++x) {
        st->cur[j] = x;
        orc_bf_rec(st, j + 1, left - x);
    }
}

int64_t orc_bruteforce(const orc_dims* d, const float* stale, const float* cost, const float* post,
                       const uint16_t* lmu, const float* lf,
                       uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum)
{
    if (!orc_dims_valid(d)) return -1;
    int64_t V = d->n_streams, J = 2 * V;
    /* guard: number of allocations C(U+J, J) must stay small */
    double count = 1.0;
    for (int64_t i = 1; i <= J; ++i) count = count * (double)(d->units + i) / (double)i;
    if (count > 2.0e7) return -2;
    int32_t* cur = (int32_t*)malloc(sizeof(int32_t) * J);
    int32_t* best = (int32_t*)malloc(sizeof(int32_t) * J);
    int64_t bad = 0;
    for (int64_t b = 0; b < d->n_inst; ++b) {
        orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
        if (!orc_instance_valid(d, &in)) {
            ++bad;
            memset(out_alloc + b * J, 0, sizeof(uint16_t) * J);
            memset(out_cfg + b * V, 0, V);
            out_sum[b] = 0;
            continue;
        }
        orc_bf st = {d, &in, cur, best, 0, 0};
        orc_bf_rec(&st, 0, d->units);
        for (int64_t j = 0; j < J; ++j) out_alloc[b * J + j] = (uint16_t)best[j];
        orc_pick(d, &in, best, out_cfg + b * V, NULL);
        out_sum[b] = st.best_s;
    }
    free(cur);
    free(best);
    return bad;
}

/* ------------------------------------------------------------------------ */
/* History / class-distribution-similarity profiler                          */
/* (draft appendix)                                         */
/* ------------------------------------------------------------------------ */

/* Rule 5: squared Euclidean distance, summed sequentially over classes. */
static float orc_dist2(const float* a, const float* b, int32_t C)
{
    float s = 0.0f;
    for (int32_t c = 0; c < C; ++c) {
        float diff = a[c] - b[c];
        float sq = diff * diff;
        s = s + sq;
    }
    return s;
}

static int orc_nearest(const float* x, const float* mu, int32_t k, int32_t C)
{
    int best = 0;
    float bd = orc_dist2(x, mu, C);
    for (int i = 1; i < k; ++i) {
        float di = orc_dist2(x, mu + (int64_t)i * C, C);
        if (di < bd) {                     /* lowest index on ties (C19) */
            bd = di;
            best = i;
        }
    }
    return best;
}

/* out_passes (optional, telemetry): Lloyd assignment passes per CLUSTER query (the
 * initial assignment + one per iteration; 0 for RADIUS, empty histories and invalid
 * queries). */
int64_t orc_profile_ex(const orc_profile_dims* p, const float* cur, const float* hist,
                       const float* hist_acc, const float* fallback,
                       float* out_est, int32_t* out_n, int32_t* out_cluster, int32_t* out_passes)
{
    int64_t Q = p->n_query, H = p->n_hist, C = p->n_class, G = p->n_gamma;
    if (Q < 0 || H < 0 || C < 1 || G < 1 || (p->mode != 0 && p->mode != 1)) return -1;
    if (p->mode == 0 && !(p->tau >= 0.0f)) return -1;
    if (p->mode == 1 && (p->k < 1 || p->max_iter < 0)) return -1;
    int64_t K = p->mode == 1 ? p->k : 1;
    unsigned char* sim = (unsigned char*)malloc(H > 0 ? H : 1);
    int32_t* assign = (int32_t*)malloc(sizeof(int32_t) * (H > 0 ? H : 1));
    int32_t* nassign = (int32_t*)malloc(sizeof(int32_t) * (H > 0 ? H : 1));
    float* mu = (float*)malloc(sizeof(float) * K * C);
    uint64_t* acc_sum = (uint64_t*)malloc(sizeof(uint64_t) * K * C);
    int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * K);
    int64_t bad = 0;

    for (int64_t q = 0; q < Q; ++q) {
        const float* cq = cur + q * C;
        const float* hq = hist + q * H * C;
        const float* aq = hist_acc + q * H * G;
        if (out_passes) out_passes[q] = 0;
        int ok = 1;
        for (int64_t c = 0; c < C; ++c) ok &= orc_in01(cq[c]);
        for (int64_t i = 0; i < H * C; ++i) ok &= orc_in01(hq[i]);
        for (int64_t i = 0; i < H * G; ++i) ok &= (isnan(aq[i]) || orc_in01(aq[i]));
        if (!ok) {
            ++bad;
            for (int64_t g = 0; g < G; ++g) {
                out_est[q * G + g] = 0.0f;
                out_n[q * G + g] = 0;
            }
            if (out_cluster && p->mode == 1)
                for (int64_t h = 0; h <= H; ++h) out_cluster[q * (H + 1) + h] = 0;
            continue;
        }
        if (p->mode == 0) {
            /* RADIUS: similar iff Euclidean distance <= tau (C17) */
            for (int64_t h = 0; h < H; ++h) {
                float d2 = orc_dist2(cq, hq + h * C, (int32_t)C);
                float dist = sqrtf(d2);
                sim[h] = dist <= p->tau;
            }
        } else {
            /* CLUSTER: Lloyd k-means over the H history windows (C19) */
            int32_t qc = -1;
            if (H > 0) {
                for (int64_t i = 0; i < K; ++i)
                    memcpy(mu + i * C, hq + ((i * H) / K) * C, sizeof(float) * C);
                for (int64_t h = 0; h < H; ++h)
                    assign[h] = orc_nearest(hq + h * C, mu, (int32_t)K, (int32_t)C);
                if (out_passes) out_passes[q] = 1;   /* assignment passes: the initial one ... */
                for (int32_t it = 0; it < p->max_iter; ++it) {
                    if (out_passes) out_passes[q] += 1;   /* ... plus one per iteration */
                    memset(acc_sum, 0, sizeof(uint64_t) * K * C);
                    memset(cnt, 0, sizeof(int64_t) * K);
                    for (int64_t h = 0; h < H; ++h) {
                        cnt[assign[h]] += 1;
                        for (int64_t c = 0; c < C; ++c)
                            acc_sum[assign[h] * C + c] += orc_q32(hq[h * C + c]);
                    }
                    for (int64_t i = 0; i < K; ++i) {
                        if (cnt[i] == 0) continue;   /* empty cluster keeps its centroid */
                        for (int64_t c = 0; c < C; ++c)
                            mu[i * C + c] = orc_mean_from_q32(acc_sum[i * C + c], (int32_t)cnt[i]);
                    }
                    int changed = 0;
                    for (int64_t h = 0; h < H; ++h) {
                        nassign[h] = orc_nearest(hq + h * C, mu, (int32_t)K, (int32_t)C);
                        changed |= nassign[h] != assign[h];
                    }
                    if (!changed) break;
                    memcpy(assign, nassign, sizeof(int32_t) * H);
                }
                qc = orc_nearest(cq, mu, (int32_t)K, (int32_t)C);
            }
            for (int64_t h = 0; h < H; ++h) sim[h] = assign[h] == qc;
            if (out_cluster) {
                for (int64_t h = 0; h < H; ++h) out_cluster[q * (H + 1) + h] = assign[h];
                out_cluster[q * (H + 1) + H] = qc;
            }
        }
        /* mean past accuracy of gamma over similar windows that measured it
         * (P:29 footnote, C18); none -> caller's fallback (C20) */
        for (int64_t g = 0; g < G; ++g) {
            uint64_t s = 0;
            int32_t n = 0;
            for (int64_t h = 0; h < H; ++h) {
                float a = aq[h * G + g];
                if (!sim[h] || isnan(a)) continue;
                s += orc_q32(a);
                ++n;
            }
            out_n[q * G + g] = n;
            out_est[q * G + g] = n > 0 ? orc_mean_from_q32(s, n) : fallback[q * G + g];
        }
    }
    free(sim);
    free(assign);
    free(nassign);
    free(mu);
    free(acc_sum);
    free(cnt);
    return bad;
}

int64_t orc_profile(const orc_profile_dims* p, const float* cur, const float* hist,
                    const float* hist_acc, const float* fallback,
                    float* out_est, int32_t* out_n, int32_t* out_cluster)
{
    return orc_profile_ex(p, cur, hist, hist_acc, fallback, out_est, out_n, out_cluster, NULL);
}

/* ========================================================================
 * NEXT-4: placement onto GPUs and the checkpoint decision.
 * ======================================================================== */

/* PL1: the fractional part r/U of a GPU (0 < r < U) quantized DOWN to the largest
 * inverse power of two 2^-k, k >= 1 ("quantizes the allocations to inverse powers of
 * two (e.g. 1/2, 1/4, 1/8)"; "largest value 2^(-k) <= share, round down; never
 * over-subscribes").  Exact integer test: 2^-k <= r/U  <=>  U <= r 2^k.
 * Returned in quanta of 2^-16 GPU; U <= 65534 < 2^16 guarantees k <= 16. */
int32_t orc_quantize_frac(int64_t r, int32_t U)
{
    if (r <= 0 || r >= U) return 0;
    int k = 1;
    while ((r << k) < (int64_t)U) ++k;
    return (int32_t)(ORC_Q_ONE >> k);
}

typedef struct { int32_t job, piece; uint32_t q; } orc_piece;

/* descending demand, then ascending job id, then piece index */
static int orc_piece_cmp(const void* x, const void* y)
{
    const orc_piece* a = (const orc_piece*)x;
    const orc_piece* b = (const orc_piece*)y;
    if (a->q != b->q) return a->q > b->q ? -1 : 1;
    if (a->job != b->job) return a->job < b->job ? -1 : 1;
    return a->piece < b->piece ? -1 : (a->piece > b->piece);
}

/* PL2 first-fit decreasing of `np` pieces already sorted by orc_piece_cmp onto `gpus`
 * GPUs of capacity one GPU (ORC_Q_ONE quanta): each piece goes to the lowest-index GPU it
 * still fits in, else it is unplaced (-1). */
static void orc_ffd(const orc_piece* pc, int32_t np, int32_t gpus, int16_t* gpu_out, uint32_t* load)
{
    for (int32_t g = 0; g < gpus; ++g) load[g] = 0;
    for (int32_t i = 0; i < np; ++i) {
        gpu_out[i] = -1;
        for (int32_t g = 0; g < gpus; ++g) {
            if (load[g] + pc[i].q <= ORC_Q_ONE) { gpu_out[i] = (int16_t)g; load[g] += pc[i].q; break; }
        }
    }
}

/* S:333-339 pack() on its own (pinned with the spec's examples): demands in quanta,
 * job ids = input order; outputs per input job its GPU (-1 unplaced) and the loads. */
int64_t orc_pack(int32_t n, const uint32_t* q, int32_t gpus, int16_t* gpu_of_job, uint32_t* load)
{
    if (n < 0 || gpus < 1) return -1;
    orc_piece* pc = (orc_piece*)malloc(sizeof(orc_piece) * (size_t)(n > 0 ? n : 1));
    int16_t* go = (int16_t*)malloc(sizeof(int16_t) * (size_t)(n > 0 ? n : 1));
    for (int32_t i = 0; i < n; ++i) { pc[i].job = i; pc[i].piece = 0; pc[i].q = q[i]; }
    qsort(pc, (size_t)n, sizeof(orc_piece), orc_piece_cmp);
    orc_ffd(pc, n, gpus, go, load);
    for (int32_t i = 0; i < n; ++i) gpu_of_job[pc[i].job] = go[i];
    free(pc);
    free(go);
    return 0;
}

/* Placement of every instance's job allocations (units) onto `gpus` GPUs.
 * PL1: job j with a_j units holds a_j G / U GPUs (delta = G/U GPU per unit):
 *      floor(a_j G / U) whole GPUs, each a piece of one GPU, plus the remainder
 *      quantized down to 2^-k (orc_quantize_frac) as one more piece if non-zero.
 * PL2: pieces sorted by descending demand, ties by job id then piece index;
 *      first fit over GPUs 0..G-1 (capacity one GPU, in quanta); a piece that fits
 *      nowhere is unplaced (gpu -1).
 * PL3: outputs per instance: the sorted pieces (job, quanta, gpu) -- at most J + G
 *      of them when sum a_j <= U -- their count, and the per-GPU load in quanta.
 * Rows with sum a_j > U are data errors (R-ERR): zero pieces, counted. */
int64_t orc_place(int32_t n_inst, int32_t n_jobs, int32_t units, int32_t gpus, const uint16_t* alloc,
                  uint16_t* piece_job, uint32_t* piece_q, int16_t* piece_gpu, uint16_t* n_pieces,
                  uint32_t* gpu_load)
{
    if (n_inst < 0 || n_jobs < 1 || units < 1 || units > 65534 || gpus < 1) return -1;
    const int32_t P = n_jobs + gpus;
    orc_piece* pc = (orc_piece*)malloc(sizeof(orc_piece) * (size_t)P);
    uint32_t* load = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)gpus);
    int64_t bad = 0;
    for (int64_t b = 0; b < n_inst; ++b) {
        const uint16_t* a = alloc + b * n_jobs;
        int64_t tot = 0;
        for (int32_t j = 0; j < n_jobs; ++j) tot += a[j];
        int32_t np = 0;
        if (tot > units) {
            ++bad;
        } else {
            for (int32_t j = 0; j < n_jobs; ++j) {
                const int64_t share = (int64_t)a[j] * gpus;           /* in 1/U GPU */
                const int64_t whole = share / units, r = share % units;
                for (int64_t w = 0; w < whole; ++w) {
                    pc[np].job = j; pc[np].piece = (int32_t)w; pc[np].q = ORC_Q_ONE; ++np;
                }
                const int32_t fq = orc_quantize_frac(r, units);
                if (fq > 0) {
                    pc[np].job = j; pc[np].piece = (int32_t)whole; pc[np].q = (uint32_t)fq; ++np;
                }
            }
            qsort(pc, (size_t)np, sizeof(orc_piece), orc_piece_cmp);
        }
        orc_ffd(pc, np, gpus, piece_gpu + b * P, load);
        for (int32_t i = 0; i < P; ++i) {
            piece_job[b * P + i] = i < np ? (uint16_t)pc[i].job : 0;
            piece_q[b * P + i] = i < np ? pc[i].q : 0;
            if (i >= np) piece_gpu[b * P + i] = -1;
        }
        n_pieces[b] = (uint16_t)np;
        if (gpu_load)
            for (int32_t g = 0; g < gpus; ++g) gpu_load[b * gpus + g] = load[g];
    }
    free(pc);
    free(load);
    return bad;
}

/* CK1: checkpoint now iff acc > base_acc (draft P:74-81) with
 *   base_acc = ((tau-t) a + (T-tau) A) / T,  acc = ((tau-t) a* + (T-tau-delta) A) / T,
 * i.e. (tau-t)(a*-a) > delta A ("equivalently"): evaluated in that form, one
 * binary32 rounding per operation.  Elements violating 0 <= t <= tau <= T, T > 0,
 * accuracies in [0,1], delta >= 0 are data errors (decision 0, counted). */
int64_t orc_checkpoint(int64_t n, const float* tau, const float* t, const float* T, const float* a,
                       const float* a_star, const float* A, const float* delta_ckpt, uint8_t* out)
{
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        const int ok = T[i] > 0.0f && t[i] >= 0.0f && t[i] <= tau[i] && tau[i] <= T[i] &&
                       orc_in01(a[i]) && orc_in01(a_star[i]) && orc_in01(A[i]) && delta_ckpt[i] >= 0.0f;
        if (!ok) { ++bad; out[i] = 0; continue; }
        const float rem = tau[i] - t[i];
        const float gain = a_star[i] - a[i];
        const float lhs = rem * gain;
        const float rhs = delta_ckpt[i] * A[i];
        out[i] = lhs > rhs;
    }
    return bad;
}

/* ========================================================================
 * NEXT-3: the uniform baseline and the Pareto frontier of the
 * retraining configurations.
 * ======================================================================== */

/* U1 + U2: the uniform scheduler ("evenly splits the GPUs between video streams,
 * and each stream evenly partitions its allocated GPUs"; "a fixed retraining
 * configuration, and a static retraining/inference resource allocation").
 * U1: share_v as C9; r_train = floor(fl(share fl(1 - w))), r_infer = share - r_train
 *     (w = inference_weight in (0,1); w = 1/2 is exactly C9's fair start).
 * U2: the retraining config is fixed: fixed_gamma >= 1 is config fixed_gamma - 1 of every
 *     stream, 0 = no retraining, -1 = each stream's highest post-retraining accuracy
 *     ("the configuration ... that results in the highest accuracy"; lowest index on
 *     ties; none if the stream has no real config).  lambda* as rule 3.  Value =
 *     fl(factor g(gamma, r_train)) when gamma is feasible at r_train (rule 1), else the
 *     retraining does not finish within the window and the value is fl(factor stale);
 *     no admissible lambda -> 0 (C8).  cfg reports the fixed gamma and lambda*.
 * Returns the number of invalid instances (R-ERR: outputs zeroed). */
int64_t orc_uniform(const orc_dims* d, const float* stale, const float* cost, const float* post,
                    const uint16_t* lmu, const float* lf, int32_t fixed_gamma, float inference_weight,
                    uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean)
{
    if (!orc_dims_valid(d) || fixed_gamma < -1 || fixed_gamma > d->n_gamma ||
        !(inference_weight > 0.0f && inference_weight < 1.0f))
        return -1;
    const int32_t V = d->n_streams, J = 2 * V, nG = d->n_gamma, nL = d->n_lambda;
    int64_t bad = 0;
    for (int64_t b = 0; b < d->n_inst; ++b) {
        orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
        if (!orc_instance_valid(d, &in)) {
            ++bad;
            for (int32_t j = 0; j < J; ++j) out_alloc[b * J + j] = 0;
            for (int32_t v = 0; v < V; ++v) out_cfg[b * V + v] = 0;
            out_sum[b] = 0;
            if (out_mean) out_mean[b] = 0.0f;
            continue;
        }
        uint64_t S = 0;
        for (int32_t v = 0; v < V; ++v) {
            const int32_t share = d->units / V + (v < d->units % V ? 1 : 0);
            const float keep = 1.0f - inference_weight;
            const float x = (float)share * keep;
            const int32_t rt = (int32_t)floorf(x);
            const int32_t ri = share - rt;
            out_alloc[b * J + 2 * v] = (uint16_t)ri;
            out_alloc[b * J + 2 * v + 1] = (uint16_t)rt;
            const float st = in.stale[v];
            const float* cv = in.cost + (int64_t)v * nG;
            const float* pv = in.post + (int64_t)v * nG;
            int g = fixed_gamma;                       /* 1-based config, 0 = none */
            if (g < 0) {
                g = 0;
                float bp = 0.0f;
                for (int k = 0; k < nG; ++k) {
                    if (isinf(cv[k])) continue;        /* padding */
                    if (g == 0 || pv[k] > bp) { g = k + 1; bp = pv[k]; }
                }
            }
            const int l = orc_lambda_star(st, in.lmu + (int64_t)v * nL, in.lf + (int64_t)v * nL, nL, ri,
                                          d->a_min);
            float val = 0.0f;
            uint8_t cfg = (uint8_t)(ORC_LAMBDA_NONE << 5);
            if (l >= 0) {
                const float fac = in.lf[(int64_t)v * nL + l];
                float acc = st;
                if (g > 0 && orc_gamma_feasible(cv[g - 1], rt, d->unit_gpu_seconds))
                    acc = orc_window_accuracy(st, pv[g - 1], cv[g - 1], rt, d->unit_gpu_seconds);
                val = fac * acc;
                cfg = (uint8_t)(g | (l << 5));
            }
            out_cfg[b * V + v] = cfg;
            S += orc_q32(val);
        }
        out_sum[b] = S;
        if (out_mean) out_mean[b] = orc_mean_from_q32(S, V);
    }
    return bad;
}

/* PR1: the Pareto frontier of a stream's configurations in (cost, accuracy) (Figure 3,
 * P:147 "Pareto boundary"): config k is on it iff no other real config k'
 * has cost' <= cost and post' >= post with at least one strict.  Padding (cost +INF) is
 * never on it.  Bit k of out_mask[set] (k = 0..n-1) marks config k.  Invalid data (R-ERR:
 * a cost that is NaN, negative or -INF, a real config's accuracy outside [0,1] or NaN):
 * that set's mask is 0 and it is counted in the return value.  n = 0 (no configurations
 * at all, S:115's empty input) is an argument error. */
int64_t orc_pareto(int64_t n_sets, int32_t n, const float* cost, const float* post, uint32_t* out_mask)
{
    if (n_sets < 0 || n < 1 || n > 32) return -1;
    int64_t bad = 0;
    for (int64_t s = 0; s < n_sets; ++s) {
        const float* c = cost + s * n;
        const float* p = post + s * n;
        uint32_t m = 0;
        int valid = 1;
        for (int32_t k = 0; k < n; ++k) {
            if (!(c[k] >= 0.0f)) valid = 0;                       /* NaN, negative, -INF */
            else if (!isinf(c[k]) && !(p[k] >= 0.0f && p[k] <= 1.0f)) valid = 0;
        }
        if (!valid) {
            ++bad;
            out_mask[s] = 0;
            continue;
        }
        for (int32_t k = 0; k < n; ++k) {
            if (isinf(c[k])) continue;
            int dominated = 0;
            for (int32_t j = 0; j < n && !dominated; ++j) {
                if (j == k || isinf(c[j])) continue;
                if (c[j] <= c[k] && p[j] >= p[k] && (c[j] < c[k] || p[j] > p[k])) dominated = 1;
            }
            if (!dominated) m |= 1u << k;
        }
        out_mask[s] = m;
    }
    return bad;
}

/* PN1-PN3: pruning of configurations that have historically not been useful (P:1179-1180
 * "configurations that are usually significantly distant from the configurations on the
 * Pareto curve of the resource-accuracy profile").  Per stream (query q) and history window
 * j, the Pareto boundary at config k's cost is the best accuracy of any real config measured
 * in j whose cost is not above cost[k] (PN1; k itself counts, so the gap is >= 0 and 0 on
 * the boundary); config k is "far" in j iff fl(boundary - acc_j(k)) > margin.  Config k is
 * pruned iff it is far in strictly more than half of the windows that measured it (PN2);
 * never-measured configs are kept, padding (cost +INF) is never kept.  Costs are the
 * stream's current profile (PN3).  Invalid data (cost NaN or < 0, a real config's
 * measured accuracy outside [0,1]): keep mask 0, counted in the return value.  Literal
 * O(H n^2) loops. */
int64_t orc_prune(int64_t n_query, int32_t H, int32_t n, const float* cost, const float* hist_acc, float margin,
                  uint32_t* out_keep)
{
    if (n_query < 0 || H < 0 || n < 0 || n > 31 || isnan(margin)) return -1;
    int64_t bad = 0;
    for (int64_t q = 0; q < n_query; ++q) {
        const float* c = cost + q * n;
        const float* A = hist_acc + q * (int64_t)H * n;
        int ok = 1;
        for (int32_t k = 0; k < n; ++k) {
            if (!(c[k] >= 0.0f)) ok = 0;
            else if (!isinf(c[k]))
                for (int32_t j = 0; j < H; ++j)
                    if (!isnan(A[(int64_t)j * n + k]) && !orc_in01(A[(int64_t)j * n + k])) ok = 0;
        }
        if (!ok) {
            out_keep[q] = 0;
            ++bad;
            continue;
        }
        uint32_t keep = 0;
        for (int32_t k = 0; k < n; ++k) {
            if (isinf(c[k])) continue;
            int64_t measured = 0, far = 0;
            for (int32_t j = 0; j < H; ++j) {
                const float* a = A + (int64_t)j * n;
                if (isnan(a[k])) continue;
                ++measured;
                float boundary = a[k];
                for (int32_t k2 = 0; k2 < n; ++k2) {
                    if (isinf(c[k2]) || isnan(a[k2])) continue;
                    if (c[k2] <= c[k] && a[k2] > boundary) boundary = a[k2];
                }
                const float gap = boundary - a[k];
                if (gap > margin) ++far;
            }
            if (!(2 * far > measured)) keep |= 1u << k;
        }
        out_keep[q] = keep;
    }
    return bad;
}

/* ========================================================================
 * NEXT-2: the micro-profiler's curve fit and extrapolation
 * ("fit the accuracy-epoch points to the a non-linear curve model ...
 * using a non-negative least squares solver ... extrapolate"; S:106-108,
 * S:147-163).  Readings CF1-CF3 in DESIGN.md.
 * ======================================================================== */

/* CF1 model: accuracy(k) = 1 - (1/(beta0 k + beta1) + beta2), beta >= 0.  With
 * alpha = 1/beta0 and c = beta1/beta0 the loss term is alpha/(k + c): for a fixed c >= 0
 * the fit is a two-variable non-negative least squares problem in (alpha, beta2).
 * orc_nnls2: min sum_k (alpha x_k + b - y_k)^2, alpha, b >= 0, closed form by the active
 * set: the unconstrained solution if both >= 0, else the better of the two boundary
 * solutions (alpha = 0, b = max(0, mean y)) and (b = 0, alpha = max(0, Sxy/Sxx)).
 * Sums sequential in k; one binary32 rounding per operation.  Returns the SSE. */
static float orc_sse(const float* x, const float* y, int n, float al, float b)
{
    float e = 0.0f;
    for (int k = 0; k < n; ++k) {
        const float r = al * x[k];
        const float t = r + b;
        const float d = t - y[k];
        const float dd = d * d;
        e = e + dd;
    }
    return e;
}

static float orc_nnls2(const float* x, const float* y, int n, float* al_out, float* b_out)
{
    float sx = 0.0f, sy = 0.0f, sxx = 0.0f, sxy = 0.0f;
    for (int k = 0; k < n; ++k) {
        sx = sx + x[k];
        sy = sy + y[k];
        const float xx = x[k] * x[k];
        sxx = sxx + xx;
        const float xy = x[k] * y[k];
        sxy = sxy + xy;
    }
    const float fn = (float)n;
    const float a1 = fn * sxx, a2 = sx * sx;
    const float det = a1 - a2;
    if (det > 0.0f) {
        const float u1 = fn * sxy, u2 = sx * sy;
        const float al = (u1 - u2) / det;
        const float v1 = sxx * sy, v2 = sx * sxy;
        const float b = (v1 - v2) / det;
        if (al >= 0.0f && b >= 0.0f) {
            *al_out = al;
            *b_out = b;
            return orc_sse(x, y, n, al, b);
        }
    }
    /* boundary candidates (both feasible): alpha = 0, or b = 0 */
    const float m = sy / fn;
    const float b0 = m > 0.0f ? m : 0.0f;
    const float e0 = orc_sse(x, y, n, 0.0f, b0);
    const float q = sxx > 0.0f ? sxy / sxx : 0.0f;
    const float a0 = q > 0.0f ? q : 0.0f;
    const float e1 = orc_sse(x, y, n, a0, 0.0f);
    if (e1 < e0) {
        *al_out = a0;
        *b_out = 0.0f;
        return e1;
    }
    *al_out = 0.0f;
    *b_out = b0;
    return e0;
}

/* CF2: the non-linear parameter c over the fixed grid c_i = i/8, i = 0..256 (c in [0, 32]
 * epochs; exact binary32 values); the lowest SSE wins, lowest i on ties.  CF3: the
 * extrapolated accuracy at epoch K, 1 - (alpha/(K + c) + beta2), clamped to [0, 1].
 * acc [n_sets][n_points] at epochs 1..n_points (2 <= n_points <= 32), full_epochs [n_sets]
 * >= 1; out_pred [n_sets]; out_params [n_sets][3] = (alpha, c, beta2) or NULL.  A set
 * with an accuracy outside [0,1] or full_epochs < 1 is a data error (pred 0). */
#define ORC_CF_GRID 257
int64_t orc_curve_fit(int64_t n_sets, int32_t n_points, const float* acc, const int32_t* full_epochs,
                      float* out_pred, float* out_params)
{
    if (n_sets < 0 || n_points < 2 || n_points > 32) return -1;
    int64_t bad = 0;
    float x[32], y[32];
    for (int64_t s = 0; s < n_sets; ++s) {
        const float* a = acc + s * n_points;
        int ok = full_epochs[s] >= 1;
        for (int k = 0; k < n_points; ++k) ok &= orc_in01(a[k]);
        if (!ok) {
            ++bad;
            out_pred[s] = 0.0f;
            if (out_params) out_params[s * 3] = out_params[s * 3 + 1] = out_params[s * 3 + 2] = 0.0f;
            continue;
        }
        for (int k = 0; k < n_points; ++k) y[k] = 1.0f - a[k];
        float best = 0.0f, bal = 0.0f, bb = 0.0f, bc = 0.0f;
        for (int i = 0; i < ORC_CF_GRID; ++i) {
            const float c = (float)i * 0.125f;
            for (int k = 0; k < n_points; ++k) {
                const float den = (float)(k + 1) + c;
                x[k] = 1.0f / den;
            }
            float al, b;
            const float e = orc_nnls2(x, y, n_points, &al, &b);
            if (i == 0 || e < best) {
                best = e;
                bal = al;
                bb = b;
                bc = c;
            }
        }
        const float den = (float)full_epochs[s] + bc;
        const float l1 = bal / den;
        const float l = l1 + bb;
        float p = 1.0f - l;
        p = p < 0.0f ? 0.0f : (p > 1.0f ? 1.0f : p);
        out_pred[s] = p;
        if (out_params) {
            out_params[s * 3] = bal;
            out_params[s * 3 + 1] = bc;
            out_params[s * 3 + 2] = bb;
        }
    }
    return bad;
}

/* ========================================================================
 * NEXT-1: the retraining window as a timeline, with the thief
 * re-invoked at every retraining completion ("Algorithm 1 is invoked at
 * the beginning of each retraining window, as well as on the completion of
 * every training job during the window to reallocate resources to the other
 * training and inference jobs").  Readings W1-W6 in DESIGN.md.
 * Time is the window fraction tau in [0, 1]; every step one binary32 rounding.
 * ======================================================================== */
/* Per instance: st_v 0 idle / 1 retraining (config g_v, remaining work R_v in cost
 * units) / 2 done; m_v the stream's model accuracy (stale, then post of its config).
 * Invocation at tau (W2): the residual problem is the instance's own tables with
 *   stale' = m_v; idle: cost' = fl(cost fl(1/fl(1 - tau))) (the remaining window is
 *   shorter, W3); retraining: only config g_v, cost' = fl(R_v fl(1/fl(1 - tau)));
 *   done: no config.  The thief (same mode, from its fair start, Alg. 1 line 2) decides
 *   allocations and configs for [tau, 1].
 * W4: a stream retraining with config g at rt units finishes at
 *   tau_v = fl(tau + fl(f fl(1 - tau))), f = rule 1's fraction of the residual
 *   window; the next event is the earliest tau_v (1 if none).
 * W5: inference accuracy over [tau, tau*] is fl(factor_lambda m_v) (lambda from the
 *   thief's config, none -> 0); A_v += fl(fl(tau* - tau) fl(factor m_v)).
 * W6: at tau*: streams with tau_v <= tau* are done (m_v = post_g); the others
 *   retraining keep R_v = fl(R_v' fl(1 - fl(fl(tau* - tau) / fl(tau_v - tau)))) with
 *   R_v' their residual work in cost units (idle streams starting: cost_g); a config-0
 *   choice for a retraining stream pauses it.  At most V + 1 invocations.
 * Outputs: out_avg[b] = fl(sum_v A_v (sequential) / V); out_events[b] = invocations;
 * out_done[b][v] = completion time (1 if none). */
int64_t orc_window(const orc_dims* d, const float* stale, const float* cost, const float* post,
                   const uint16_t* lmu, const float* lf, int32_t mode, float* out_avg, uint32_t* out_events,
                   float* out_done)
{
    if (!orc_dims_valid(d) || (mode != 0 && mode != 1)) return -1;
    const int32_t V = d->n_streams, nG = d->n_gamma, nL = d->n_lambda, J = 2 * V;
    orc_dims d1 = *d;
    d1.n_inst = 1;
    float* st1 = (float*)malloc(sizeof(float) * V);
    float* c1 = (float*)malloc(sizeof(float) * (size_t)(V * nG + 1));
    uint16_t* a1 = (uint16_t*)malloc(sizeof(uint16_t) * J);
    uint8_t* cf1 = (uint8_t*)malloc((size_t)V);
    float* m = (float*)malloc(sizeof(float) * V);
    float* R = (float*)malloc(sizeof(float) * V);
    float* A = (float*)malloc(sizeof(float) * V);
    float* tv = (float*)malloc(sizeof(float) * V);
    int32_t* stt = (int32_t*)malloc(sizeof(int32_t) * V);
    int32_t* g = (int32_t*)malloc(sizeof(int32_t) * V);
    int64_t bad = 0;
    for (int64_t b = 0; b < d->n_inst; ++b) {
        orc_inst in = orc_instance(d, b, stale, cost, post, lmu, lf);
        if (!orc_instance_valid(d, &in)) {
            ++bad;
            out_avg[b] = 0.0f;
            out_events[b] = 0;
            for (int32_t v = 0; v < V; ++v) out_done[b * V + v] = 0.0f;
            continue;
        }
        for (int32_t v = 0; v < V; ++v) {
            m[v] = in.stale[v]; R[v] = 0.0f; A[v] = 0.0f; stt[v] = 0; g[v] = 0;
            out_done[b * V + v] = 1.0f;
        }
        float tau = 0.0f;
        uint32_t ev = 0;
        while (tau < 1.0f && ev <= (uint32_t)V) {
            const float rem = 1.0f - tau;
            const float sc = 1.0f / rem;
            for (int32_t v = 0; v < V; ++v) {
                st1[v] = m[v];
                for (int32_t k = 0; k < nG; ++k) {
                    const float c = in.cost[(int64_t)v * nG + k];
                    float cs = INFINITY;
                    if (stt[v] == 0) cs = isinf(c) ? c : c * sc;
                    else if (stt[v] == 1 && k + 1 == g[v]) cs = R[v] * sc;
                    c1[v * nG + k] = cs;
                }
            }
            uint64_t s1;
            orc_thief(&d1, st1, c1, in.post, in.lmu, in.lf, mode, a1, cf1, &s1, NULL, NULL);
            ++ev;
            /* W4: completion times of the streams retraining in [tau, 1] */
            float tnext = 1.0f;
            for (int32_t v = 0; v < V; ++v) {
                const int32_t gv = cf1[v] & 31, rt = a1[2 * v + 1];
                tv[v] = 2.0f;
                if (gv > 0) {
                    const float f = orc_retrain_fraction(c1[v * nG + gv - 1], rt, d->unit_gpu_seconds);
                    const float dt = f * rem;
                    tv[v] = tau + dt;
                    if (tv[v] < tnext) tnext = tv[v];
                }
            }
            /* W5: accuracy over [tau, tnext] */
            const float span = tnext - tau;
            for (int32_t v = 0; v < V; ++v) {
                const int32_t l = cf1[v] >> 5;
                const float fac = l == ORC_LAMBDA_NONE ? 0.0f : in.lf[(int64_t)v * nL + l];
                const float acc = fac * m[v];
                const float seg = span * acc;
                A[v] = A[v] + seg;
            }
            /* W6: completions and remaining work */
            for (int32_t v = 0; v < V; ++v) {
                const int32_t gv = cf1[v] & 31;
                if (gv == 0) continue;
                if (tv[v] <= tnext) {
                    stt[v] = 2;
                    m[v] = in.post[(int64_t)v * nG + gv - 1];
                    out_done[b * V + v] = tv[v];
                } else {
                    const float base = stt[v] == 1 ? R[v] : in.cost[(int64_t)v * nG + gv - 1];
                    const float q = span / (tv[v] - tau);
                    const float keep = 1.0f - q;
                    R[v] = base * keep;
                    stt[v] = 1;
                    g[v] = gv;
                }
            }
            tau = tnext;
        }
        float sum = 0.0f;
        for (int32_t v = 0; v < V; ++v) sum = sum + A[v];
        out_avg[b] = sum / (float)V;
        out_events[b] = ev;
    }
    free(st1); free(c1); free(a1); free(cf1); free(m); free(R); free(A); free(tv); free(stt); free(g);
    return bad;
}
