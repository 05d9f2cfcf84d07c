// launch.h -- host-side launchers behind the C ABI (internal to libekya).
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cstddef>
#include <cstdint>

#include "../../include/ekya.h"
#include "ekya_common.cuh"

struct ekya_handle {
    int device;
    int sm_count;
    size_t smem_optin;                 // max dynamic shared memory per block
    ekya::DevState* dstate;            // device error word
    unsigned long long launches;       // kernels launched through this handle
    void* nccl_comm;                   // ncclComm_t when initialised
    int nranks, rank;
    void* scratch;                     // kernel scratch (CLUSTER work lists), grown on demand
    size_t scratch_bytes;
};

namespace ekya {
// Device scratch of at least `bytes` owned by the handle (allocated once, reused by every
// later launch; grows only when a larger launch needs more).  nullptr on failure.
void* handle_scratch(ekya_handle* h, size_t bytes);
}

namespace ekya {

int launch_eval_grid(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, float* out_grid,
                     uint8_t* out_grid_cfg, cudaStream_t s);
int launch_eval_list(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int n_alloc,
                     const uint16_t* alloc, uint64_t* out_sum, float* out_mean, uint8_t* out_cfg,
                     cudaStream_t s);
int launch_thief(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int mode,
                 uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean,
                 uint32_t* out_steps, cudaStream_t s);
int launch_profile(ekya_handle* h, const ekya_profile_dims& p, const float* cur, const float* hist,
                   const float* hist_acc, const float* fallback, float* out_est, int32_t* out_n,
                   int32_t* out_cluster, cudaStream_t s, float* rad_est = nullptr, int32_t* rad_n = nullptr,
                   float rad_tau = 0.0f);
int launch_profile_both(ekya_handle* h, const ekya_profile_dims& p, const float* cur, const float* hist,
                        const float* hist_acc, const float* fallback, float* rad_est, int32_t* rad_n,
                        float* cl_est, int32_t* cl_n, int32_t* out_cluster, cudaStream_t s);

int launch_place(ekya_handle* h, int32_t n_inst, int32_t n_jobs, int32_t units, int32_t gpus,
                 const uint16_t* alloc, uint16_t* piece_job, uint32_t* piece_q, int16_t* piece_gpu,
                 uint16_t* n_pieces, uint32_t* gpu_load, cudaStream_t s);
int launch_checkpoint(ekya_handle* h, long long n, const float* tau, const float* t, const float* T,
                      const float* a, const float* a_star, const float* A, const float* delta, uint8_t* out,
                      cudaStream_t s);

int launch_uniform(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int fixed_gamma, float weight,
                   uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean, cudaStream_t s);
int launch_pareto(ekya_handle* h, long long n_sets, int n, const float* cost, const float* post,
                  uint32_t* out_mask, cudaStream_t s);
int launch_prune(ekya_handle* h, long long n_query, int H, int n, const float* cost, const float* acc, float margin,
                 uint32_t* out_keep, cudaStream_t s);

int launch_curve_fit(ekya_handle* h, long long n_sets, int np, const float* acc, const int* full_epochs,
                     float* out_pred, float* out_params, cudaStream_t s);

size_t window_workspace_bytes(const ekya_dims& d);
int launch_window(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int mode, void* ws, size_t ws_bytes,
                  float* out_avg, uint32_t* out_events, float* out_done, cudaStream_t s);

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? EKYA_OK : EKYA_ERR_CUDA; }

// NVTX range around every C-ABI call (one named range per API call, visible in
// nsys / ncu --nvtx timelines; a no-op unless a tool is attached)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

}  // namespace ekya
