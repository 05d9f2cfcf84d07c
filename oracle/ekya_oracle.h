/*
 * ekya_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Declarations of the plain, slow CPU oracle for Ekya's scheduling objective
 * (arXiv 2012.10557).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product
 * (paper_2012_10557_b200/, include/ekya.h) shares no code, header, type or
 * constant with it.
 *
 * Citations: P:<line> = PAPER.md line, S:<line> = SPEC.md line, C<n> = the
 * reading numbered <n> in DESIGN.md section 3.
 */
#ifndef EKYA_ORACLE_H
#define EKYA_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scheduling-instance dimensions (Table 2 notation). */
typedef struct {
    int32_t n_inst;      /* B independent instances                       */
    int32_t n_streams;   /* V = |V| video streams                         */
    int32_t n_gamma;     /* |Gamma_v| real retraining configs (0..31)      */
    int32_t n_lambda;    /* |Lambda_v| inference configs (1..7)            */
    int32_t units;       /* U = G/delta allocation units                  */
    int32_t steal_units; /* Delta/delta >= 1                               */
    float   unit_gpu_seconds; /* uT = delta * ||T|| GPU-seconds per unit   */
    float   a_min;       /* a_MIN                                 */
} orc_dims;

typedef struct {
    int32_t n_query, n_hist, n_class, n_gamma;
    int32_t mode;        /* 0 RADIUS, 1 CLUSTER */
    float   tau;         /* RADIUS threshold on Euclidean distance (C17) */
    int32_t k, max_iter; /* CLUSTER (C19) */
} orc_profile_dims;

/* ---- single-quantity primitives (exposed for pins) ---- */
float    orc_retrain_fraction(float cost, int32_t rt, float uT);
int32_t  orc_gamma_feasible(float cost, int32_t rt, float uT);
float    orc_window_accuracy(float stale, float post, float cost, int32_t rt, float uT);
uint64_t orc_q32(float x);
float    orc_stream_value(const orc_dims* d, float stale, const float* cost, const float* post,
                          const uint16_t* lam_min_units, const float* lam_factor,
                          int32_t rt, int32_t ri, uint8_t* cfg);

/* ---- per-instance procedures (instance b of a batched table set) ---- */
uint64_t orc_pickconfigs(const orc_dims* d, int64_t b, const float* stale, const float* cost,
                         const float* post, const uint16_t* lmu, const float* lf,
                         const int32_t* alloc, uint8_t* cfg_out, float* val_out);
void     orc_fair(const orc_dims* d, int32_t* alloc);

/* ---- batched procedures (return number of instances/rows with a data error, <0 on bad dims) ---- */
int64_t orc_eval_grid(const orc_dims* d, const float* stale, const float* cost, const float* post,
                      const uint16_t* lmu, const float* lf, float* out_grid, uint8_t* out_grid_cfg);
int64_t orc_eval_list(const orc_dims* d, const float* stale, const float* cost, const float* post,
                      const uint16_t* lmu, const float* lf, int32_t n_alloc, const uint16_t* alloc,
                      uint64_t* out_sum, float* out_mean, uint8_t* out_cfg);
int64_t orc_thief(const orc_dims* d, const float* stale, const float* cost, const float* post,
                  const uint16_t* lmu, const float* lf, int32_t mode,
                  uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean,
                  uint32_t* out_steps);
int64_t orc_bruteforce(const orc_dims* d, const float* stale, const float* cost, const float* post,
                       const uint16_t* lmu, const float* lf,
                       uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum);
int64_t orc_profile(const orc_profile_dims* p, const float* cur, const float* hist,
                    const float* hist_acc, const float* fallback,
                    float* out_est, int32_t* out_n, int32_t* out_cluster);
int64_t orc_profile_ex(const orc_profile_dims* p, const float* cur, const float* hist,
                       const float* hist_acc, const float* fallback,
                       float* out_est, int32_t* out_n, int32_t* out_cluster, int32_t* out_passes);

/* ---- NEXT-4: placement of decisions onto GPUs and the
 *      checkpoint decision (draft P:62-81); readings PL1-PL3, CK1 ---- */
#define ORC_Q_ONE 65536   /* one GPU in quanta of 2^-16 GPU */
int32_t orc_quantize_frac(int64_t r, int32_t U);   /* largest 2^-k (k >= 1) <= r/U, in quanta */
int64_t orc_pack(int32_t n, const uint32_t* q, int32_t gpus, int16_t* gpu_of_job, uint32_t* load);
int64_t orc_place(int32_t n_inst, int32_t n_jobs, int32_t units, int32_t gpus, const uint16_t* alloc,
                  uint16_t* piece_job, uint32_t* piece_q, int16_t* piece_gpu, uint16_t* n_pieces,
                  uint32_t* gpu_load);
int64_t orc_checkpoint(int64_t n, const float* tau, const float* t, const float* T, const float* a,
                       const float* a_star, const float* A, const float* delta_ckpt, uint8_t* out);

/* ---- NEXT-3: uniform baseline (readings U1, U2) and the
 *      Pareto frontier of a stream's configurations (reading PR1) ---- */
int64_t orc_uniform(const orc_dims* d, const float* stale, const float* cost, const float* post,
                    const uint16_t* lmu, const float* lf, int32_t fixed_gamma, float inference_weight,
                    uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean);
int64_t orc_pareto(int64_t n_sets, int32_t n, const float* cost, const float* post, uint32_t* out_mask);
/* history-based pruning of configurations far from the Pareto boundary (
 * readings PN1-PN3) */
int64_t orc_prune(int64_t n_query, int32_t H, int32_t n, const float* cost, const float* hist_acc, float margin,
                  uint32_t* out_keep);

/* ---- NEXT-2: micro-profiler curve fit + extrapolation (
 *      readings CF1-CF3) ---- */
int64_t orc_curve_fit(int64_t n_sets, int32_t n_points, const float* acc, const int32_t* full_epochs,
                      float* out_pred, float* out_params);

/* ---- NEXT-1: the window as a timeline with re-invocation at completions (P:1022,
 *      P:1123-1125; readings W1-W6) ---- */
int64_t orc_window(const orc_dims* d, const float* stale, const float* cost, const float* post,
                   const uint16_t* lmu, const float* lf, int32_t mode, float* out_avg, uint32_t* out_events,
                   float* out_done);

#ifdef __cplusplus
}
#endif
#endif
