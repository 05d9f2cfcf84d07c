// api.cu -- the extern "C" boundary of libekya (include/ekya.h): handle
// management, synchronous argument checks, and dispatch to the launchers.
#include <cmath>
#include <cstdlib>
#include <new>

#include "launch.h"

using namespace ekya;

namespace {

bool dims_ok(const ekya_dims* d, int* why) {
    if (!d) { *why = EKYA_ERR_ARG; return false; }
    if (d->n_inst < 0 || d->n_streams < 1) { *why = EKYA_ERR_SHAPE; return false; }
    if (d->n_gamma < 0 || d->n_gamma > kMaxGamma || d->n_lambda < 1 || d->n_lambda > kMaxLambda ||
        d->units < 1 || d->units > 65534 || d->steal_units < 1) {
        *why = EKYA_ERR_LIMIT;
        return false;
    }
    if (!(d->unit_gpu_seconds > 0.0f) || std::isinf(d->unit_gpu_seconds) || std::isnan(d->a_min) ||
        std::isinf(d->a_min)) {
        *why = EKYA_ERR_ARG;
        return false;
    }
    return true;
}

bool tables_ok(const ekya_dims* d, const ekya_tables* t) {
    if (!t) return false;
    if (d->n_inst == 0) return true;
    if (!t->stale || !t->lam_min_units || !t->lam_factor) return false;
    if (d->n_gamma > 0 && (!t->cost || !t->post)) return false;
    return true;
}

}  // namespace

namespace ekya {
void* handle_scratch(ekya_handle* h, size_t bytes) {
    if (bytes <= h->scratch_bytes) return h->scratch;
    // a larger launch than any before: the previous buffer may still be in use by queued
    // kernels, so wait for the device before replacing it (one-time cost per size step)
    if (h->scratch) {
        if (cudaDeviceSynchronize() != cudaSuccess) return nullptr;
        cudaFree(h->scratch);
        h->scratch = nullptr;
        h->scratch_bytes = 0;
    }
    if (cudaMalloc(&h->scratch, bytes) != cudaSuccess) {
        h->scratch = nullptr;
        return nullptr;
    }
    h->scratch_bytes = bytes;
    return h->scratch;
}
}  // namespace ekya

extern "C" {

const char* ekya_version(void) { return "ekya-b200 0.1 (sm_100a)"; }

int ekya_create(ekya_handle** out, int device, size_t /*workspace_bytes*/) {
    if (!out) return EKYA_ERR_ARG;
    *out = nullptr;
    if (cudaSetDevice(device) != cudaSuccess) return EKYA_ERR_CUDA;
    ekya_handle* h = new (std::nothrow) ekya_handle();
    if (!h) return EKYA_ERR_ARG;
    h->device = device;
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    h->sm_count = v;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    h->smem_optin = (size_t)v;
    if (cudaMalloc(&h->dstate, sizeof(DevState)) != cudaSuccess ||
        cudaMemset(h->dstate, 0, sizeof(DevState)) != cudaSuccess) {
        delete h;
        return EKYA_ERR_CUDA;
    }
    h->launches = 0;
    h->nccl_comm = nullptr;
    h->nranks = 1;
    h->rank = 0;
    h->scratch = nullptr;
    h->scratch_bytes = 0;
    *out = h;
    return EKYA_OK;
}

void ekya_comm_destroy_internal(ekya_handle* h);

void ekya_destroy(ekya_handle* h) {
    if (!h) return;
    ekya_comm_destroy_internal(h);
    if (h->scratch) cudaFree(h->scratch);
    cudaFree(h->dstate);
    delete h;
}

int ekya_last_error(ekya_handle* h) {
    if (!h) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    if (cudaDeviceSynchronize() != cudaSuccess) return EKYA_ERR_CUDA;
    DevState st;
    if (cudaMemcpy(&st, h->dstate, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return EKYA_ERR_CUDA;
    if (st.err) {
        cudaMemset(&h->dstate->err, 0, sizeof(unsigned));
        return EKYA_ERR_DATA;
    }
    return EKYA_OK;
}

uint64_t ekya_launch_count(const ekya_handle* h) { return h ? h->launches : 0; }

int ekya_counters(ekya_handle* h, uint64_t* out, int n) {
    if (!h || !out || n < 0) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return EKYA_ERR_CUDA;
    DevState st;
    if (cudaMemcpy(&st, h->dstate, sizeof(st), cudaMemcpyDeviceToHost) != cudaSuccess) return EKYA_ERR_CUDA;
    const uint64_t v[2] = {h->launches, st.lloyd_passes};
    for (int i = 0; i < n && i < 2; ++i) out[i] = v[i];
    return EKYA_OK;
}

int ekya_eval_allocations(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int mode,
                          int32_t n_alloc, const uint16_t* alloc, uint64_t* out_sum_q32,
                          float* out_mean, uint8_t* out_cfg, float* out_grid, uint8_t* out_grid_cfg,
                          ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_eval_allocations");
    if (!h) return EKYA_ERR_ARG;
    int why = EKYA_OK;
    if (!dims_ok(d, &why)) return why;
    if (!tables_ok(d, t)) return EKYA_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    if (mode == EKYA_EVAL_LIST) {
        if (n_alloc < 0) return EKYA_ERR_SHAPE;
        if (d->n_inst > 0 && n_alloc > 0 && (!alloc || !out_sum_q32)) return EKYA_ERR_ARG;
        return launch_eval_list(h, *d, *t, n_alloc, alloc, out_sum_q32, out_mean, out_cfg, s);
    }
    if (mode == EKYA_EVAL_GRID) {
        if (d->n_inst > 0 && !out_grid) return EKYA_ERR_ARG;
        return launch_eval_grid(h, *d, *t, out_grid, out_grid_cfg, s);
    }
    return EKYA_ERR_ARG;
}

int ekya_thief_schedule(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int mode,
                        uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum_q32,
                        float* out_mean, uint32_t* out_steps, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_thief_schedule");
    if (!h) return EKYA_ERR_ARG;
    int why = EKYA_OK;
    if (!dims_ok(d, &why)) return why;
    if (!tables_ok(d, t)) return EKYA_ERR_ARG;
    if (mode != EKYA_THIEF_STEEPEST && mode != EKYA_THIEF_LITERAL) return EKYA_ERR_ARG;
    if (d->n_inst > 0 && (!out_alloc || !out_cfg || !out_sum_q32)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_thief(h, *d, *t, mode, out_alloc, out_cfg, out_sum_q32, out_mean, out_steps,
                        reinterpret_cast<cudaStream_t>(stream));
}

int ekya_profile_estimate(ekya_handle* h, const ekya_profile_dims* p, const float* cur,
                          const float* hist, const float* hist_acc, const float* fallback,
                          float* out_est, int32_t* out_n, int32_t* out_cluster, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_profile_estimate");
    if (!h || !p) return EKYA_ERR_ARG;
    if (p->n_query < 0 || p->n_hist < 0) return EKYA_ERR_SHAPE;
    if (p->n_class < 1 || p->n_class > 1024 || p->n_gamma < 1 || p->n_gamma > 256) return EKYA_ERR_LIMIT;
    if (p->mode == EKYA_PROFILE_RADIUS) {
        if (!(p->tau >= 0.0f)) return EKYA_ERR_ARG;
    } else if (p->mode == EKYA_PROFILE_CLUSTER) {
        if (p->k < 1 || p->k > 32 || p->max_iter < 0) return EKYA_ERR_LIMIT;
    } else {
        return EKYA_ERR_ARG;
    }
    if (p->n_query > 0 && (!cur || !fallback || !out_est || !out_n)) return EKYA_ERR_ARG;
    if (p->n_query > 0 && p->n_hist > 0 && (!hist || !hist_acc)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_profile(h, *p, cur, hist, hist_acc, fallback, out_est, out_n, out_cluster,
                          reinterpret_cast<cudaStream_t>(stream));
}

int ekya_profile_estimate_both(ekya_handle* h, const ekya_profile_dims* p, const float* cur,
                               const float* hist, const float* hist_acc, const float* fallback,
                               float* out_est_radius, int32_t* out_n_radius, float* out_est_cluster,
                               int32_t* out_n_cluster, int32_t* out_cluster, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_profile_estimate_both");
    if (!h || !p) return EKYA_ERR_ARG;
    if (p->n_query < 0 || p->n_hist < 0) return EKYA_ERR_SHAPE;
    if (p->n_class < 1 || p->n_class > 1024 || p->n_gamma < 1 || p->n_gamma > 256) return EKYA_ERR_LIMIT;
    if (!(p->tau >= 0.0f)) return EKYA_ERR_ARG;
    if (p->k < 1 || p->k > 32 || p->max_iter < 0) return EKYA_ERR_LIMIT;
    if (p->n_query > 0 && (!cur || !fallback || !out_est_radius || !out_n_radius || !out_est_cluster ||
                           !out_n_cluster))
        return EKYA_ERR_ARG;
    if (p->n_query > 0 && p->n_hist > 0 && (!hist || !hist_acc)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_profile_both(h, *p, cur, hist, hist_acc, fallback, out_est_radius, out_n_radius, out_est_cluster,
                               out_n_cluster, out_cluster, reinterpret_cast<cudaStream_t>(stream));
}

int ekya_uniform_schedule(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int32_t fixed_gamma,
                          float inference_weight, uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum_q32,
                          float* out_mean, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_uniform_schedule");
    if (!h) return EKYA_ERR_ARG;
    int why = EKYA_OK;
    if (!dims_ok(d, &why)) return why;
    if (!tables_ok(d, t)) return EKYA_ERR_ARG;
    if (fixed_gamma < -1 || fixed_gamma > d->n_gamma || !(inference_weight > 0.0f && inference_weight < 1.0f))
        return EKYA_ERR_ARG;
    if (d->n_inst > 0 && (!out_alloc || !out_cfg || !out_sum_q32)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_uniform(h, *d, *t, fixed_gamma, inference_weight, out_alloc, out_cfg, out_sum_q32, out_mean,
                          reinterpret_cast<cudaStream_t>(stream));
}

int ekya_pareto(ekya_handle* h, int64_t n_sets, int32_t n, const float* cost, const float* post,
                uint32_t* out_mask, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_pareto");
    if (!h) return EKYA_ERR_ARG;
    if (n_sets < 0 || n < 0) return EKYA_ERR_SHAPE;
    if (n > 31) return EKYA_ERR_LIMIT;
    if (n_sets > 0 && n == 0) return EKYA_ERR_SHAPE;   // no configurations: S:115's empty input
    if (n_sets > 0 && (!cost || !post || !out_mask)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_pareto(h, (long long)n_sets, n, cost, post, out_mask, reinterpret_cast<cudaStream_t>(stream));
}

int ekya_prune_configs(ekya_handle* h, int64_t n_query, int32_t n_hist, int32_t n, const float* cost,
                       const float* hist_acc, float margin, uint32_t* out_keep, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_prune_configs");
    if (!h) return EKYA_ERR_ARG;
    if (n_query < 0 || n_hist < 0 || n < 0) return EKYA_ERR_SHAPE;
    if (n > 31 || n_hist > (1 << 20)) return EKYA_ERR_LIMIT;
    if (margin != margin) return EKYA_ERR_ARG;
    if (n_query > 0 && (!out_keep || (n > 0 && !cost) || (n > 0 && n_hist > 0 && !hist_acc))) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_prune(h, (long long)n_query, n_hist, n, cost, hist_acc, margin, out_keep,
                        reinterpret_cast<cudaStream_t>(stream));
}

size_t ekya_window_workspace_bytes(const ekya_dims* d) {
    if (!d || d->n_inst < 0 || d->n_streams < 1) return 0;
    return window_workspace_bytes(*d);
}

int ekya_window_schedule(ekya_handle* h, const ekya_dims* d, const ekya_tables* t, int mode, void* workspace,
                         size_t workspace_bytes, float* out_avg, uint32_t* out_events, float* out_done,
                         ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_window_schedule");
    if (!h) return EKYA_ERR_ARG;
    int why = EKYA_OK;
    if (!dims_ok(d, &why)) return why;
    if (!tables_ok(d, t)) return EKYA_ERR_ARG;
    if (mode != EKYA_THIEF_STEEPEST && mode != EKYA_THIEF_LITERAL) return EKYA_ERR_ARG;
    if (d->n_streams > 127) return EKYA_ERR_LIMIT;
    if (d->n_inst > 0 && (!out_avg || !out_events || !out_done)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_window(h, *d, *t, mode, workspace, workspace_bytes, out_avg, out_events, out_done,
                         reinterpret_cast<cudaStream_t>(stream));
}

int ekya_curve_fit(ekya_handle* h, int64_t n_sets, int32_t n_points, const float* acc, const int32_t* full_epochs,
                   float* out_pred, float* out_params, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_curve_fit");
    if (!h) return EKYA_ERR_ARG;
    if (n_sets < 0) return EKYA_ERR_SHAPE;
    if (n_points < 2 || n_points > 32) return EKYA_ERR_LIMIT;
    if (n_sets > 0 && (!acc || !full_epochs || !out_pred)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_curve_fit(h, (long long)n_sets, n_points, acc, full_epochs, out_pred, out_params,
                            reinterpret_cast<cudaStream_t>(stream));
}

int ekya_place(ekya_handle* h, int32_t n_inst, int32_t n_jobs, int32_t units, int32_t gpus,
               const uint16_t* alloc, uint16_t* out_piece_job, uint32_t* out_piece_q, int16_t* out_piece_gpu,
               uint16_t* out_n_pieces, uint32_t* out_gpu_load, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_place");
    if (!h) return EKYA_ERR_ARG;
    if (n_inst < 0 || n_jobs < 1) return EKYA_ERR_SHAPE;
    if (units < 1 || units > 65534 || gpus < 1 || gpus > 128 || n_jobs + gpus > 4096) return EKYA_ERR_LIMIT;
    if (n_inst > 0 && (!alloc || !out_piece_job || !out_piece_q || !out_piece_gpu || !out_n_pieces))
        return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_place(h, n_inst, n_jobs, units, gpus, alloc, out_piece_job, out_piece_q, out_piece_gpu,
                        out_n_pieces, out_gpu_load, reinterpret_cast<cudaStream_t>(stream));
}

int ekya_checkpoint_decide(ekya_handle* h, int64_t n, const float* tau, const float* t, const float* T,
                           const float* a, const float* a_star, const float* A, const float* delta_ckpt,
                           uint8_t* out, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_checkpoint_decide");
    if (!h) return EKYA_ERR_ARG;
    if (n < 0) return EKYA_ERR_SHAPE;
    if (n > 0 && (!tau || !t || !T || !a || !a_star || !A || !delta_ckpt || !out)) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    return launch_checkpoint(h, (long long)n, tau, t, T, a, a_star, A, delta_ckpt, out,
                             reinterpret_cast<cudaStream_t>(stream));
}

}  // extern "C"
