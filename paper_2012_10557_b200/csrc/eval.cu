// eval.cu -- ekya_eval_allocations: the allocation evaluator.
//
// GRID: one CTA per (instance, stream) work item (grid-stride loop sized to
// the resident-CTA count).  It builds the stream's PickConfigs tables in
// shared memory (stream_tables.cuh) and writes every (rt, ri) cell of the
// stream's triangle, row by row, one warp per row: lanes write consecutive
// cells, so every warp store is a contiguous 128-byte (f32) / 32-byte (u8)
// run.  The kernel is bound by the 5 B/cell output stream to HBM.
//
// LIST: one CTA per instance builds the tables of all V streams in shared
// memory, then streams the instance's allocation rows through shared memory
// (16-byte vector loads) with one thread per row: V table lookups, exact Q32
// sum, and the optional mean/config outputs.
#include <algorithm>

#include "launch.h"
#include "stream_tables.cuh"

namespace ekya {

namespace {

constexpr int kEvalThreads = 256;
constexpr int kListRowsPerChunk = kEvalThreads;

struct EvalParams {
    ekya_dims d;
    ekya_tables t;
    DevState* st;
    // GRID
    float* out_grid;
    uint8_t* out_grid_cfg;
    // LIST
    int n_alloc;
    const uint16_t* alloc;
    unsigned long long* out_sum;
    float* out_mean;
    uint8_t* out_cfg;
    int R;            // table-build chunk rows
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct GridLayout {
    size_t in, gbuf, gstar, mask, tval, tcfg, lad, total;
};

__host__ __device__ inline GridLayout grid_layout(int U, int nG, int nL, int R, int nstreams) {
    GridLayout L;
    size_t o = 0;
    L.in = o;    o += align16(sizeof(StreamIn));
    L.gbuf = o;  o += align16(sizeof(float) * (size_t)R * (nG + 1));
    L.gstar = o; o += align16(sizeof(float) * (size_t)(U + 1));
    L.mask = o;  o += align16(sizeof(uint32_t) * (size_t)(U + 1));
    L.tval = o;  o += align16(sizeof(float) * (size_t)nstreams * (U + 1) * nL);
    L.tcfg = o;  o += align16((size_t)nstreams * (U + 1) * nL);
    L.lad = o;   o += align16((size_t)nstreams * (U + 1));
    L.total = o;
    return L;
}

__global__ void __launch_bounds__(kEvalThreads) grid_kernel(EvalParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int U = d.units, nG = d.n_gamma, nL = d.n_lambda, V = d.n_streams;
    GridLayout L = grid_layout(U, nG, nL, p.R, 1);
    StreamIn* sin = reinterpret_cast<StreamIn*>(smem + L.in);
    TabScratch sc{reinterpret_cast<float*>(smem + L.gbuf), reinterpret_cast<float*>(smem + L.gstar),
                  reinterpret_cast<uint32_t*>(smem + L.mask), p.R};
    float* tval = reinterpret_cast<float*>(smem + L.tval);
    uint8_t* tcfg = smem + L.tcfg;
    uint8_t* lad = smem + L.lad;

    const long long NC = (long long)(U + 1) * (U + 2) / 2;
    const long long items = (long long)d.n_inst * V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;

    for (long long item = blockIdx.x; item < items; item += gridDim.x) {
        const long long b = item / V;
        const bool ok = instance_valid(p.t, b, V, nG, nL);
        load_stream(sin, p.t, item, nG, nL);
        __syncthreads();
        if (ok) {
            build_stream_tables(sin, U, nG, nL, d.unit_gpu_seconds, d.a_min, sc, lad, tval, tcfg);
        } else if (threadIdx.x == 0) {
            flag_data_error(p.st);
        }
        float* og = p.out_grid + item * NC;
        uint8_t* oc = p.out_grid_cfg ? p.out_grid_cfg + item * NC : nullptr;
        for (int rt = warp; rt <= U; rt += nw) {
            const long long rs = (long long)rt * (U + 1) - (long long)rt * (rt - 1) / 2;
            const float* tv = tval + rt * nL;
            const uint8_t* tc = tcfg + rt * nL;
            for (int ri = lane; ri <= U - rt; ri += 32) {
                float val = 0.0f;
                uint8_t c = 0;
                if (ok) {
                    int l = lad[ri];
                    c = (uint8_t)(kLambdaNone << 5);
                    if (l != kLambdaNone) {
                        val = tv[l];
                        c = tc[l];
                    }
                }
                og[rs + ri] = val;
                if (oc) oc[rs + ri] = c;
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kEvalThreads) list_kernel(EvalParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int U = d.units, nG = d.n_gamma, nL = d.n_lambda, V = d.n_streams, J = 2 * V;
    GridLayout L = grid_layout(U, nG, nL, p.R, V);
    StreamIn* sin = reinterpret_cast<StreamIn*>(smem + L.in);
    TabScratch sc{reinterpret_cast<float*>(smem + L.gbuf), reinterpret_cast<float*>(smem + L.gstar),
                  reinterpret_cast<uint32_t*>(smem + L.mask), p.R};
    float* tval = reinterpret_cast<float*>(smem + L.tval);
    uint8_t* tcfg = smem + L.tcfg;
    uint8_t* lad = smem + L.lad;
    unsigned char* rowbuf = smem + L.total;                                   // CH*J*2 + 16
    unsigned char* cfgbuf = rowbuf + align16((size_t)kListRowsPerChunk * J * 2 + 16);  // CH*V + 16
    const size_t tabs = (size_t)(U + 1) * nL;

    for (long long b = blockIdx.x; b < d.n_inst; b += gridDim.x) {
        const bool ok = instance_valid(p.t, b, V, nG, nL);
        if (ok) {
            for (int v = 0; v < V; ++v) {
                load_stream(sin, p.t, b * V + v, nG, nL);
                __syncthreads();
                build_stream_tables(sin, U, nG, nL, d.unit_gpu_seconds, d.a_min, sc,
                                    lad + (size_t)v * (U + 1), tval + v * tabs, tcfg + v * tabs);
            }
        } else if (threadIdx.x == 0) {
            flag_data_error(p.st);
        }
        for (long long n0 = 0; n0 < p.n_alloc; n0 += kListRowsPerChunk) {
            const int rows = (int)min((long long)kListRowsPerChunk, (long long)p.n_alloc - n0);
            const long long row0 = b * p.n_alloc + n0;
            const uint16_t* rsrc = p.alloc + row0 * J;
            const uint16_t* rs = reinterpret_cast<const uint16_t*>(
                stage_to_smem(rowbuf, rsrc, (size_t)rows * J * sizeof(uint16_t)));
            uint8_t* cstage = nullptr;
            if (p.out_cfg) cstage = cfgbuf + (reinterpret_cast<uintptr_t>(p.out_cfg + row0 * V) & 15u);
            __syncthreads();
            const int r = threadIdx.x;
            if (r < rows) {
                const uint16_t* row = rs + (size_t)r * J;
                bool rok = ok;
                int tot = 0;
                for (int v = 0; v < V; ++v) {
                    int ri = row[2 * v], rt = row[2 * v + 1];
                    tot += ri + rt;
                    rok &= (ri <= U) & (rt <= U);
                }
                rok &= tot <= U;                     // Eq. 1 constraint 2
                unsigned long long S = 0;
                for (int v = 0; v < V; ++v) {
                    uint8_t c = 0;
                    if (rok) {
                        int ri = row[2 * v], rt = row[2 * v + 1];
                        int l = lad[(size_t)v * (U + 1) + ri];
                        c = (uint8_t)(kLambdaNone << 5);
                        if (l != kLambdaNone) {
                            size_t e = v * tabs + (size_t)rt * nL + l;
                            S += q32(tval[e]);
                            c = tcfg[e];
                        }
                    }
                    if (cstage) cstage[(size_t)r * V + v] = c;
                }
                if (!rok && ok) flag_data_error(p.st);
                const long long o = row0 + r;
                p.out_sum[o] = S;
                if (p.out_mean) p.out_mean[o] = rok ? mean_q32(S, V) : 0.0f;
            }
            __syncthreads();
            if (cstage) {
                store_from_smem(p.out_cfg + row0 * V, cstage, (size_t)rows * V);
                __syncthreads();
            }
        }
    }
}

int pick_rows(int U, int nG) {
    int G1 = nG + 1;
    int R = 4096 / G1;                    // <= 16 KB of g values per chunk
    return std::max(1, std::min(R, U + 1));
}

int resident_grid(ekya_handle* h, const void* fn, size_t smem, long long work) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kEvalThreads, smem);
    per_sm = std::max(per_sm, 1);
    long long g = (long long)h->sm_count * per_sm;
    return (int)std::max(1LL, std::min(g, work));
}

}  // namespace

int launch_eval_grid(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, float* out_grid,
                     uint8_t* out_grid_cfg, cudaStream_t s) {
    if (d.units > 4094) return EKYA_ERR_SHAPE;
    EvalParams p{};
    p.d = d;
    p.t = t;
    p.st = h->dstate;
    p.out_grid = out_grid;
    p.out_grid_cfg = out_grid_cfg;
    p.R = pick_rows(d.units, d.n_gamma);
    size_t smem = grid_layout(d.units, d.n_gamma, d.n_lambda, p.R, 1).total;
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    long long items = (long long)d.n_inst * d.n_streams;
    if (items == 0) return EKYA_OK;
    cudaError_t e = cudaFuncSetAttribute(grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    int grid = resident_grid(h, (const void*)grid_kernel, smem, items);
    grid_kernel<<<grid, kEvalThreads, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

int launch_eval_list(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int n_alloc,
                     const uint16_t* alloc, uint64_t* out_sum, float* out_mean, uint8_t* out_cfg,
                     cudaStream_t s) {
    EvalParams p{};
    p.d = d;
    p.t = t;
    p.st = h->dstate;
    p.n_alloc = n_alloc;
    p.alloc = alloc;
    p.out_sum = reinterpret_cast<unsigned long long*>(out_sum);
    p.out_mean = out_mean;
    p.out_cfg = out_cfg;
    p.R = pick_rows(d.units, d.n_gamma);
    const int V = d.n_streams, J = 2 * V;
    size_t smem = grid_layout(d.units, d.n_gamma, d.n_lambda, p.R, V).total +
                  align16((size_t)kListRowsPerChunk * J * 2 + 16) +
                  align16((size_t)kListRowsPerChunk * V + 16);
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    if (d.n_inst == 0 || n_alloc == 0) return EKYA_OK;
    cudaError_t e = cudaFuncSetAttribute(list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    int grid = resident_grid(h, (const void*)list_kernel, smem, d.n_inst);
    list_kernel<<<grid, kEvalThreads, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
