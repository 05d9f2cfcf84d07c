// comm.cu -- multi-GPU decision gather.
//
// Scheduling instances are independent, so each rank evaluates its own
// contiguous block of instances with no data-path collective.  The only
// exchange is the final gather of fixed-size decision records to a root rank
// (north star "only a final NCCL gather of decisions"), enqueued on the caller's
// stream with NCCL's native ncclGather over NVLink 5 / NVSwitch.
#include <nccl.h>

#include <cstring>

#include "launch.h"

extern "C" {

int ekya_comm_unique_id(void* out) {
    if (!out) return EKYA_ERR_ARG;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return EKYA_ERR_NCCL;
    std::memcpy(out, &id, sizeof(id));
    return EKYA_OK;
}

int ekya_comm_init(ekya_handle* h, const void* id_bytes, int nranks, int rank) {
    ekya::NvtxRange nvtx_range("ekya_comm_init");
    if (!h || !id_bytes || nranks < 1 || rank < 0 || rank >= nranks) return EKYA_ERR_ARG;
    if (h->nccl_comm) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    ncclComm_t comm = nullptr;
    if (ncclCommInitRank(&comm, nranks, id, rank) != ncclSuccess) return EKYA_ERR_NCCL;
    h->nccl_comm = comm;
    h->nranks = nranks;
    h->rank = rank;
    return EKYA_OK;
}

int ekya_gather_decisions(ekya_handle* h, const void* local, size_t bytes_per_rank, void* root_buf,
                          int root, ekya_stream_t stream) {
    ekya::NvtxRange nvtx_range("ekya_gather_decisions");
    if (!h || !local) return EKYA_ERR_ARG;
    if (root < 0 || root >= h->nranks) return EKYA_ERR_ARG;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!h->nccl_comm) {   // single process without a communicator: the gather is a copy
        if (h->nranks != 1) return EKYA_ERR_NCCL;
        if (!root_buf) return EKYA_ERR_ARG;
        if (root_buf == local || bytes_per_rank == 0) return EKYA_OK;
        if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
        return ekya::cuda_status(cudaMemcpyAsync(root_buf, local, bytes_per_rank, cudaMemcpyDeviceToDevice, s));
    }
    if (h->rank == root && !root_buf) return EKYA_ERR_ARG;
    if (cudaSetDevice(h->device) != cudaSuccess) return EKYA_ERR_CUDA;
    ncclResult_t r = ncclGather(local, root_buf, bytes_per_rank, ncclUint8, root,
                                static_cast<ncclComm_t>(h->nccl_comm), s);
    return r == ncclSuccess ? EKYA_OK : EKYA_ERR_NCCL;
}

int ekya_comm_info(ekya_handle* h, int* out_nranks, int* out_rank) {
    if (!h || !out_nranks || !out_rank) return EKYA_ERR_ARG;
    if (!h->nccl_comm) {
        *out_nranks = h->nranks;
        *out_rank = h->rank;
        return EKYA_OK;
    }
    int n = 0, r = 0;
    if (ncclCommCount(static_cast<ncclComm_t>(h->nccl_comm), &n) != ncclSuccess ||
        ncclCommUserRank(static_cast<ncclComm_t>(h->nccl_comm), &r) != ncclSuccess)
        return EKYA_ERR_NCCL;
    *out_nranks = n;
    *out_rank = r;
    return EKYA_OK;
}

void ekya_comm_destroy_internal(ekya_handle* h) {
    if (h && h->nccl_comm) {
        ncclCommDestroy(static_cast<ncclComm_t>(h->nccl_comm));
        h->nccl_comm = nullptr;
    }
}

}  // extern "C"
