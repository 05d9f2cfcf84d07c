/*
 * ekya.h -- C ABI of the B200 (sm_100a) hot path of Ekya's thief scheduler.
 *
 * Paper: "Ekya: Continuous Learning of Video Analytics Models on Edge Compute
 * Servers" (arXiv 2012.10557).  P:<n> = line of PAPER.md (final paper
 * P:441-1738), S:<n> = line of SPEC.md.  The arithmetic contract (one IEEE
 * binary32 rounding per operation, exact Q32 objective sums) and the readings
 * C1..C23 are in DESIGN.md sections 2-3.
 *
 * Conventions for every call
 *  - All array pointers are DEVICE pointers owned by the caller (e.g. torch
 *    tensors).  Layout: instance-major, row-major, no padding.  The library
 *    never allocates on these paths and never keeps a pointer after returning.
 *  - Every compute call is asynchronous on `stream` (0 = legacy default).
 *  - Input arrays are read by the TMA bulk-copy engine in whole 16-byte
 *    granules: the library may read (never write) bytes of the 16-byte-aligned
 *    granules that contain an input array's first and last element, i.e. at
 *    most 15 bytes before/after it.  Such reads never cross a page, so any
 *    cudaMalloc / torch allocation is safe.
 *  - Return value: EKYA_OK (0) or a negative EKYA_ERR_* code.  Host-side
 *    argument checks fail synchronously before anything is launched.
 *  - Data errors found on the device (R-ERR in DESIGN.md: NaN/negative cost,
 *    accuracies or factors outside [0,1], LIST rows with an entry > U or a sum
 *    > U) do not abort: the affected instance / row gets all-zero outputs and
 *    a device error word is set; ekya_last_error() synchronises and returns
 *    EKYA_ERR_DATA once (then clears it).
 *  - Infeasibility is data, not an error: a stream with no admissible lambda
 *    contributes 0 and reports lambda = 7 (C8); an infeasible gamma is never
 *    chosen.
 *
 * Job numbering (C10): job 2v is stream v's inference job (r_infer units),
 * job 2v+1 its retraining job (r_train units).
 *
 * Config byte (cfg): bits 0..4 = gamma (0 = no retraining, 1..|Gamma| = the
 * retraining config gamma-1), bits 5..7 = lambda (0..6, 7 = none).
 */
#ifndef EKYA_H
#define EKYA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EKYA_OK               0
#define EKYA_ERR_ARG         -1   /* null pointer / bad enum / bad handle          */
#define EKYA_ERR_LIMIT       -2   /* |Gamma| > 31, |Lambda| > 7, U > 65534, ...     */
#define EKYA_ERR_SHAPE       -3   /* sizes inconsistent or too large for a mode      */
#define EKYA_ERR_CUDA        -4   /* a CUDA runtime call failed                      */
#define EKYA_ERR_NCCL        -5   /* an NCCL call failed / comm not initialised      */
#define EKYA_ERR_DATA        -6   /* (ekya_last_error only) device found bad data   */

#define EKYA_LAMBDA_NONE      7
#define EKYA_LMU_PAD     0xFFFFu  /* lam_min_units padding sentinel (unused lambda) */
/* gamma padding sentinel: cost = +INF (never feasible)                             */

/* cudaStream_t without including the CUDA headers */
typedef struct CUstream_st* ekya_stream_t;

typedef struct ekya_handle ekya_handle;

/* Create a handle bound to CUDA device `device`.  `workspace_bytes` is ignored
 * (reserved; the handle owns only its 64-byte device error word and counters). */
int  ekya_create(ekya_handle** h, int device, size_t workspace_bytes);
void ekya_destroy(ekya_handle* h);
/* Synchronises the device, returns EKYA_ERR_DATA if any kernel since the last
 * call found bad data (then clears the flag), EKYA_ERR_CUDA on a sticky CUDA
 * error, else EKYA_OK. */
int  ekya_last_error(ekya_handle* h);
/* Number of kernels this handle has launched so far (for launch accounting). */
uint64_t ekya_launch_count(const ekya_handle* h);
/* Telemetry (synchronises): out[0] = kernels launched, out[1] = cumulative
 * CLUSTER-mode Lloyd assignment passes (initial assignment + iterations, summed
 * over queries) -- the unit of the CLUSTER kernel's algorithmic work.  Writes
 * min(n, 2) values. */
int ekya_counters(ekya_handle* h, uint64_t* out, int n);
const char* ekya_version(void);

/* Problem statement of a batch of scheduling instances (Eq. 1, P:876-973;
 * notation Table 2).  [ClusterSpec S:43-46, RetrainWindow S:27-30] */
typedef struct {
    int32_t n_inst;            /* B >= 0 independent instances                     */
    int32_t n_streams;         /* V = |V| >= 1 video streams per instance          */
    int32_t n_gamma;           /* max |Gamma_v|, 0..31 (excluding gamma = none)    */
    int32_t n_lambda;          /* max |Lambda_v|, 1..7                             */
    int32_t units;             /* U = G/delta total allocation units, 1..65534     */
    int32_t steal_units;       /* Delta/delta >= 1 (C11)                           */
    float   unit_gpu_seconds;  /* uT = delta * ||T|| GPU-seconds per unit, > 0     */
    float   a_min;             /* a_MIN, finite                           */
} ekya_dims;

/* Resource-accuracy profiles (D3/D4).  [ConfigProfile S:58-61,
 * InferenceConfig S:38-41, WindowTrace.stale_accuracy S:64] */
typedef struct {
    const float*    stale;          /* [B][V]     current-model accuracy in [0,1]                */
    const float*    cost;           /* [B][V][nG] GPU-seconds to retrain at 100% GPU;
                                       +INF = padding; may be NULL iff nG == 0                  */
    const float*    post;           /* [B][V][nG] estimated post-retraining accuracy in [0,1]
                                       (e.g. ekya_profile_estimate's out_est)                   */
    const uint16_t* lam_min_units;  /* [B][V][nL] smallest r_infer that keeps up under the
                                       strict "<" of P:1088 (C2); 0xFFFF = padding              */
    const float*    lam_factor;     /* [B][V][nL] accuracy multiplier in [0,1] (C1)             */
} ekya_tables;

/* ---------------------------------------------------------------------------
 * ekya_eval_allocations -- PickConfigs (Algorithm 2) over many
 * allocations.  [pick_configs S:244-252]
 *
 * mode EKYA_EVAL_LIST: for each instance b and each of its n_alloc full
 *   allocation vectors alloc[b][n][0..2V) (u16 units, job order C10), the
 *   exact objective out_sum_q32[b][n] = sum_v Q32(value_v) (u64), optionally
 *   out_mean[b][n] = (float)(S / (V 2^32)) and out_cfg[b][n][v].  Requires the
 *   per-instance tables, V * (73 (U+1) + 32) bytes, plus ~20 KB of staging to fit
 *   in the device's opt-in shared memory per block (227 KB on B200: V (U+1) <~
 *   3300), else EKYA_ERR_SHAPE.
 * mode EKYA_EVAL_GRID: for each (b, v) and every split with r_train + r_infer
 *   <= U, out_grid[b][v][c] = value of stream v alone (f32) and
 *   out_grid_cfg[b][v][c] = its argmax config byte, cell c = rowstart(rt) + ri,
 *   rowstart(rt) = rt*(U+1) - rt*(rt-1)/2, i.e. (U+1)(U+2)/2 cells per stream
 *   (north star "for every v, gamma, lambda and (r_train, r_infer) ... per-stream
 *   argmax").  GRID needs one stream's tables, 68 (U+1) + ~600 bytes, in shared
 *   memory (U <~ 3400 on B200), else EKYA_ERR_SHAPE.  GRID writes whole 16-byte
 *   value quads: out_grid must be 16-byte aligned and out_grid_cfg 4-byte
 *   aligned; LIST reads rows as 4/8-byte words: alloc must be 4-byte aligned
 *   (EKYA_ERR_ARG otherwise; every cudaMalloc / torch allocation qualifies).
 * Outputs not used by the mode may be NULL; out_mean/out_cfg/out_grid_cfg are
 * optional.
 * ------------------------------------------------------------------------- */
enum { EKYA_EVAL_LIST = 0, EKYA_EVAL_GRID = 1 };
int ekya_eval_allocations(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int mode,
                          int32_t n_alloc, const uint16_t* alloc,
                          uint64_t* out_sum_q32, float* out_mean, uint8_t* out_cfg,
                          float* out_grid, uint8_t* out_grid_cfg, ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * ekya_thief_schedule -- Algorithm 1 for each instance, from
 * the fair start (C9).  [thief_schedule S:254-262]
 *   EKYA_THIEF_STEEPEST: per step apply the single Delta-steal (thief t,
 *     victim w) with the largest objective gain over all ordered pairs,
 *     lexicographically smallest (t, w) on ties; stop when no steal strictly
 *     improves (C12, north star).
 *   EKYA_THIEF_LITERAL: the pseudocode verbatim (thief, then victim loops,
 *     steal repeatedly while strictly improving).
 * Outputs: out_alloc[b][2V] (u16 units, sum = U), out_cfg[b][V],
 * out_sum_q32[b] (exact objective), optional out_mean[b], out_steps[b]
 * (accepted steals).  Any V, U within the limits; n_inst < 2^32 - 2^24
 * (EKYA_ERR_LIMIT).  LITERAL and wide instances (V > 16) run persistent warps
 * that claim instances from a counter in the handle's device state, so one
 * handle's thief launches must be stream-ordered (as for its error word).
 * ------------------------------------------------------------------------- */
enum { EKYA_THIEF_STEEPEST = 0, EKYA_THIEF_LITERAL = 1 };
int ekya_thief_schedule(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int mode,
                        uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum_q32,
                        float* out_mean, uint32_t* out_steps, ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * ekya_profile_estimate -- history / class-distribution-similarity estimator
 * (draft appendix).  [history_estimate S:165-173,
 * distribution_distance S:175-183]
 * For each query q (one stream's current window) with current class
 * histogram cur[q][C], history histograms hist[q][H][C] and the accuracy
 * hist_acc[q][H][G] each history window reached with retraining config g (NaN
 * = not measured), out_est[q][g] = mean accuracy over the SIMILAR windows that
 * measured g (exact Q32 mean), out_n[q][g] = their count; no such window ->
 * out_est = fallback[q][g] (the online micro-profiler's estimate), n = 0.
 *   mode 0 RADIUS : similar iff Euclidean distance <= tau (C17).
 *   mode 1 CLUSTER: Lloyd k-means (k clusters, "5 clusters", C19) over the
 *                   H windows; similar iff same cluster as the query's nearest
 *                   centroid.  out_cluster[q][0..H) = window clusters,
 *                   out_cluster[q][H] = the query's cluster (may be NULL).
 * Limits: 1 <= C <= 1024, 1 <= G <= 256, H >= 0, 1 <= k <= 32, max_iter >= 0.
 * With q = b*V + v, out_est is exactly ekya_tables.post for a batch.
 * ------------------------------------------------------------------------- */
enum { EKYA_PROFILE_RADIUS = 0, EKYA_PROFILE_CLUSTER = 1 };
typedef struct {
    int32_t n_query, n_hist, n_class, n_gamma;
    int32_t mode;
    float   tau;
    int32_t k, max_iter;
} ekya_profile_dims;
int ekya_profile_estimate(ekya_handle* h, const ekya_profile_dims* p,
                          const float* cur, const float* hist, const float* hist_acc,
                          const float* fallback, float* out_est, int32_t* out_n,
                          int32_t* out_cluster, ekya_stream_t stream);
/* Both estimates of the same queries (p->mode is ignored; tau, k and max_iter are all
 * used): out_est_radius / out_n_radius exactly as mode 0, out_est_cluster /
 * out_n_cluster / out_cluster exactly as mode 1.  For k = 5, C = 27, H <= 512 (the
 * paper's Waymo shape) one kernel computes both from a single read of each query's
 * history tile; other shapes run the two modes back to back.  Same limits and errors as
 * ekya_profile_estimate; every output array is [Q][G] (out_cluster as in mode 1). */
int ekya_profile_estimate_both(ekya_handle* h, const ekya_profile_dims* p,
                               const float* cur, const float* hist, const float* hist_acc,
                               const float* fallback, float* out_est_radius, int32_t* out_n_radius,
                               float* out_est_cluster, int32_t* out_n_cluster, int32_t* out_cluster,
                               ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * ekya_window_schedule -- the retraining window as a timeline (SURVEY 8(f)
 * NEXT-1; "Algorithm 1 is invoked at the beginning of each retraining
 * window, as well as on the completion of every training job during the window
 * to reallocate resources to the other training and inference jobs";
 * P:1123-1125).  Readings W1-W6: time is the window fraction tau;
 * at tau = 0 and at every retraining completion the thief (`mode`) re-plans the
 * residual window on residual tables (finished streams: their new model accuracy
 * as `stale` and no config; streams retraining: only their config, remaining
 * work; idle streams: all configs; costs scaled by 1/(1 - tau)); a stream's
 * inference accuracy over each interval is factor(lambda) x model accuracy.
 * out_avg [B]: realized window-average accuracy over the streams; out_events [B]:
 * thief invocations (<= V + 1); out_done [B][V]: completion time (1 = none).
 * `workspace` (device, >= ekya_window_workspace_bytes(d) bytes, caller-owned)
 * holds the residual tables and the timeline state.  V <= 127.  Invalid
 * instances: outputs 0, EKYA_ERR_DATA.
 * ------------------------------------------------------------------------- */
size_t ekya_window_workspace_bytes(const ekya_dims* d);
int ekya_window_schedule(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int mode, void* workspace,
                         size_t workspace_bytes, float* out_avg, uint32_t* out_events, float* out_done,
                         ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * ekya_curve_fit -- the micro-profiler's accuracy extrapolation (SURVEY 8(f)
 * NEXT-2; "fit the accuracy-epoch points to the a non-linear curve model
 * ... using a non-negative least squares solver ... extrapolate the accuracy that
 * would be obtained by retraining with all the data for larger number of epochs";
 * S:106-108).  acc [n_sets][n_points]: validation accuracy after epochs
 * 1..n_points (2 <= n_points <= 32) of each (stream, config) micro-profile;
 * full_epochs [n_sets] (>= 1).  Readings:
 *   CF1 model acc(k) = 1 - (1/(b0 k + b1) + b2), b >= 0, written alpha/(k + c) + b2
 *       (alpha = 1/b0, c = b1/b0); for fixed c a two-variable NNLS in (alpha, b2),
 *       solved in closed form (active set).
 *   CF2 c over the grid i/8, i = 0..256; lowest residual, lowest i on ties.
 *   CF3 out_pred = 1 - (alpha/(K + c) + b2) clamped to [0,1] (the `post` input of the
 *       tables); out_params [n_sets][3] = (alpha, c, b2) or NULL.
 * One binary32 rounding per operation.  Invalid sets (accuracy outside [0,1] or
 * full_epochs < 1): outputs 0, EKYA_ERR_DATA.
 * ------------------------------------------------------------------------- */
int ekya_curve_fit(ekya_handle* h, int64_t n_sets, int32_t n_points, const float* acc, const int32_t* full_epochs,
                   float* out_pred, float* out_params, ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * ekya_uniform_schedule -- the uniform scheduler the paper compares against
 * ("evenly splits the GPUs between video streams, and
 * each stream evenly partitions its allocated GPUs for retraining and inference
 * ... always picks the configuration for retraining that results in the highest
 * accuracy"; "a fixed retraining configuration, and a static
 * retraining/inference resource allocation").  Readings:
 *   U1 share_v as the fair start (C9); r_train = floor(fl(share fl(1 - w))),
 *      r_infer = share - r_train, w = inference_weight in (0,1) (w = 1/2: C9).
 *   U2 retraining config fixed_gamma: >= 1 = config fixed_gamma-1 of every stream,
 *      0 = no retraining, -1 = each stream's highest post accuracy (lowest index on
 *      ties).  lambda* as rule 3; value = fl(factor g(gamma, r_train)) if gamma
 *      finishes in the window (rule 1), else fl(factor stale); no lambda -> 0.
 * Outputs as ekya_thief_schedule (alloc [B][2V], cfg [B][V] with the fixed gamma,
 * exact sum [B], mean [B] or NULL).  Invalid instances: zeroed + EKYA_ERR_DATA.
 *
 * ekya_pareto -- Pareto frontier of each of n_sets sets of n <= 31 configurations
 * (cost [n_sets][n], post [n_sets][n]; e.g. a table's cost/post with n_sets =
 * B*V): bit k of out_mask[s] set iff config k is real (cost finite) and no other
 * real config has cost' <= cost and post' >= post with one strict (P:147 Figure
 * 3's "Pareto boundary"; reading PR1).  n = 0 with n_sets > 0 (sets
 * without configurations, S:115's empty input): EKYA_ERR_SHAPE.  Invalid data
 * (R-ERR: a cost NaN, negative or -INF -- only +INF is padding --, a real config's
 * post outside [0,1] or NaN): that set's mask 0 + EKYA_ERR_DATA.
 *
 * ekya_prune_configs -- pruning of configurations "that have historically not been
 * useful ... usually significantly distant from the configurations on the Pareto
 * curve of the resource-accuracy profile".  Per stream q of n_query:
 * cost [n_query][n] (the current profile; +INF = padding), hist_acc
 * [n_query][n_hist][n] (the stream's history windows, NaN = not measured; the
 * layout of ekya_profile_estimate's hist_acc).
 *   PN1 in window j the Pareto boundary at config k's cost is the best accuracy of
 *       any real config measured in j with cost <= cost[k] (k included); k is far
 *       in j iff fl(boundary - acc_j(k)) > margin.
 *   PN2 bit k of out_keep[q] is set iff k is real and far in at most half of the
 *       windows that measured it (never-measured configs are kept).
 *   PN3 costs do not depend on the window (epochs x per-epoch cost x data
 *       fraction).
 * Limits: n <= 31, n_hist <= 2^20 (EKYA_ERR_LIMIT); margin NaN: EKYA_ERR_ARG.
 * Invalid stream (cost NaN or < 0, a real config's measured accuracy outside
 * [0,1]): out_keep 0 + EKYA_ERR_DATA.
 * ------------------------------------------------------------------------- */
int ekya_uniform_schedule(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int32_t fixed_gamma,
                          float inference_weight, uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum_q32,
                          float* out_mean, ekya_stream_t stream);
int ekya_pareto(ekya_handle* h, int64_t n_sets, int32_t n, const float* cost, const float* post,
                uint32_t* out_mask, ekya_stream_t stream);
int ekya_prune_configs(ekya_handle* h, int64_t n_query, int32_t n_hist, int32_t n, const float* cost,
                       const float* hist_acc, float margin, uint32_t* out_keep, ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * ekya_place -- placement of scheduling decisions onto discrete GPUs (SURVEY 8(f)
 * NEXT-4; "quantizes the allocations to inverse powers of two ...
 * allocates jobs to GPUs in descending order of demands").
 * alloc [B][n_jobs] u16: units per job (e.g. ekya_thief_schedule's out_alloc),
 *   U = units, G = gpus (one unit = G/U GPU).  Readings:
 *   PL1 job j holds a_j G / U GPUs exactly: floor(a_j G / U) whole-GPU pieces plus
 *       the remainder r/U quantized DOWN to the largest 2^-k (k >= 1), as one more
 *       piece; demands in quanta of 2^-16 GPU (a whole GPU = 65536).
 *   PL2 first-fit decreasing: pieces by descending demand, ties by job then piece,
 *       each to the lowest-index GPU with room (capacity 65536), else unplaced.
 *   PL3 per instance, in that order: out_piece_job [B][n_jobs+G] u16,
 *       out_piece_q [B][n_jobs+G] u32, out_piece_gpu [B][n_jobs+G] i16 (-1 =
 *       unplaced or unused), out_n_pieces [B] u16, out_gpu_load [B][G] u32 (quanta;
 *       may be NULL).  Slots past n_pieces: job 0, 0 quanta, gpu -1.
 *   A row with sum a_j > U is a data error (R-ERR): zero pieces, error word set.
 * Limits: 1 <= U <= 65534, 1 <= G <= 128, n_jobs + G <= 4096 (EKYA_ERR_LIMIT).
 *
 * ekya_checkpoint_decide -- the checkpoint decision of draft P:62-81 for n
 * independent (stream, time) points: out[i] = 1 iff acc > base_acc,
 * evaluated as fl(fl(tau-t) fl(a*-a)) > fl(delta A) (reading CK1; the averaged
 * accuracies differ by that amount over T).  Points violating 0 <= t <= tau <= T,
 * T > 0, accuracies in [0,1] or delta >= 0 are data errors (out = 0).
 * ------------------------------------------------------------------------- */
int ekya_place(ekya_handle* h, int32_t n_inst, int32_t n_jobs, int32_t units, int32_t gpus,
               const uint16_t* alloc, uint16_t* out_piece_job, uint32_t* out_piece_q, int16_t* out_piece_gpu,
               uint16_t* out_n_pieces, uint32_t* out_gpu_load, ekya_stream_t stream);
int ekya_checkpoint_decide(ekya_handle* h, int64_t n, const float* tau, const float* t, const float* T,
                           const float* a, const float* a_star, const float* A, const float* delta_ckpt,
                           uint8_t* out, ekya_stream_t stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU (one process per GPU).  Instances are independent, so
 * ranks own contiguous instance blocks and the only collective is a gather of
 * the fixed-size decision records to a root rank (north star "only a final NCCL
 * gather of decisions").
 * ekya_comm_unique_id: fills 128 bytes (ncclUniqueId) on the root; broadcast
 *   them out of band (e.g. torch.distributed), then every rank calls
 *   ekya_comm_init with the same bytes (nranks = 1 is allowed: a one-rank NCCL
 *   communicator).  EKYA_ERR_NCCL on failure; a handle takes one communicator.
 * ekya_comm_info: the communicator's rank count and this rank (ncclCommCount /
 *   ncclCommUserRank); without a communicator 1 and 0.
 * ekya_gather_decisions: root_buf[r*bytes_per_rank ...] <- rank r's `local`
 *   (device pointers, caller-owned; root_buf used on the root only), enqueued on
 *   `stream` as ncclGather when a communicator exists, else (single process) a
 *   device-to-device copy.  Every rank passes the same bytes_per_rank.  Callers
 *   that overlap the gather with compute split their records into chunks and
 *   gather each chunk on a second stream (bench.py config 5).
 * ------------------------------------------------------------------------- */
int ekya_comm_unique_id(void* out_id_128_bytes);
int ekya_comm_init(ekya_handle* h, const void* id_128_bytes, int nranks, int rank);
int ekya_comm_info(ekya_handle* h, int* out_nranks, int* out_rank);
int ekya_gather_decisions(ekya_handle* h, const void* local, size_t bytes_per_rank,
                          void* root_buf, int root, ekya_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* EKYA_H */
