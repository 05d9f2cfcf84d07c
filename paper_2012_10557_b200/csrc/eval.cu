// eval.cu -- ekya_eval_allocations: the allocation evaluator.
//
// GRID: one warp per (instance, stream) work item, persistent grid.  The warp
// builds the stream's PickConfigs tables in its slice of shared memory
// (stream_tables.cuh: lanes over r_train, gamma loop in registers), then writes
// the stream's triangle row by row: lanes cover consecutive r_infer cells, the
// per-cell lookup is lad[ri] (lambda*) -> a warp shuffle from the 8 lanes that
// hold the row's (value, config) slots, so every row costs 2 shared loads and
// each warp store is a contiguous 128-byte (f32) / 32-byte (u8) run.  Bound by
// the 5 B/cell output stream to HBM.
//
// LIST: one persistent CTA per SM walks its instances; for each instance the 8
// warps build the V stream tables in parallel, and the instance's allocation
// rows stream through a two-stage shared-memory pipeline fed by TMA bulk copies
// (cp.async.bulk + mbarrier), one thread per row: V table lookups, exact Q32
// sum, mean and config bytes (staged in shared memory and written with 16-byte
// vector stores).
#include <algorithm>

#include "launch.h"
#include "stream_tables.cuh"

namespace ekya {

namespace {

constexpr int kGridWarps = 16;
constexpr int kListThreads = 256;
constexpr int kListRows = 512;      // rows per pipeline stage
constexpr int kListStages = 2;

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

// per-stream table footprint
__host__ __device__ inline size_t tab_bytes(int U) {
    return a16((size_t)(U + 1)) + a16((size_t)(U + 1) * kSlots * 4) + a16((size_t)(U + 1) * kSlots);
}

struct Tabs {
    uint8_t* lad;
    float* tv;
    uint8_t* tc;
};
__device__ __forceinline__ Tabs carve_tabs(unsigned char* p, int U) {
    Tabs t;
    t.lad = p;
    t.tv = reinterpret_cast<float*>(p + a16((size_t)(U + 1)));
    t.tc = p + a16((size_t)(U + 1)) + a16((size_t)(U + 1) * kSlots * 4);
    return t;
}

struct EvalParams {
    ekya_dims d;
    ekya_tables t;
    DevState* st;
    float* out_grid;
    uint8_t* out_grid_cfg;
    int n_alloc;
    const uint16_t* alloc;
    unsigned long long* out_sum;
    float* out_mean;
    uint8_t* out_cfg;
    size_t warp_bytes;   // GRID: shared bytes per warp
};

// ------------------------------------------------------------------------
// GRID
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(kGridWarps * 32, 1) grid_kernel(EvalParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int U = d.units, nG = d.n_gamma, nL = d.n_lambda, V = d.n_streams;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned char* mine = smem + (size_t)warp * p.warp_bytes;
    StreamIn* sin = reinterpret_cast<StreamIn*>(mine);
    Tabs T = carve_tabs(mine + a16(sizeof(StreamIn)), U);

    const long long NC = (long long)(U + 1) * (U + 2) / 2;
    const long long nwarps = (long long)gridDim.x * kGridWarps;
    // one warp per instance (validated once), its V streams in turn
    for (long long b = (long long)blockIdx.x * kGridWarps + warp; b < d.n_inst; b += nwarps) {
        const bool ok = warp_instance_valid(p.t, b, V, nG, nL);
        if (!ok && lane == 0) flag_data_error(p.st);
        for (int v = 0; v < V; ++v) {
            const long long item = b * V + v;
            if (ok) {
                warp_load_stream(sin, p.t, item, nG, nL);
                warp_build_tables(sin, U, nG, nL, d.unit_gpu_seconds, d.a_min, T.lad, T.tv, T.tc);
            }
            float* og = p.out_grid + item * NC;
            uint8_t* oc = p.out_grid_cfg ? p.out_grid_cfg + item * NC : nullptr;
            long long rs = 0;
            for (int rt = 0; rt <= U; ++rt) {
                const int len = U + 1 - rt;
                float tvl = 0.0f;
                unsigned tcl = 0;
                if (ok) {
                    tvl = T.tv[rt * kSlots + (lane & 7)];
                    tcl = T.tc[rt * kSlots + (lane & 7)];
                }
                for (int k = 0; k < len; k += 32) {
                    const int ri = k + lane;
                    const bool act = ri < len;
                    const int l = (act && ok) ? T.lad[ri] : kLambdaNone;
                    const float val = __shfl_sync(0xffffffffu, tvl, l);
                    const unsigned c = __shfl_sync(0xffffffffu, tcl, l);
                    if (act) {
                        og[rs + ri] = val;
                        if (oc) oc[rs + ri] = (uint8_t)c;
                    }
                }
                rs += len;
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------------
// LIST
// ------------------------------------------------------------------------
struct ListLayout {
    size_t sin, tabs, stage, cfgbuf, bars, misc, total, stage_bytes;
};
__host__ __device__ inline ListLayout list_layout(int U, int V) {
    ListLayout L;
    const int J = 2 * V;
    size_t o = 0;
    L.sin = o;    o += a16(sizeof(StreamIn)) * (kListThreads / 32);
    L.tabs = o;   o += tab_bytes(U) * V;
    L.stage_bytes = a16((size_t)kListRows * J * 2) + 16;
    L.stage = o;  o += L.stage_bytes * kListStages;
    L.cfgbuf = o; o += a16((size_t)kListRows * V) + 16;
    L.bars = o;   o += 64;
    L.misc = o;   o += 16;
    L.total = o;
    return L;
}

__global__ void __launch_bounds__(kListThreads) list_kernel(EvalParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int U = d.units, nG = d.n_gamma, nL = d.n_lambda, V = d.n_streams, J = 2 * V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = kListThreads / 32;
    const ListLayout L = list_layout(U, V);
    StreamIn* sin = reinterpret_cast<StreamIn*>(smem + L.sin + warp * a16(sizeof(StreamIn)));
    unsigned char* tabs = smem + L.tabs;
    const size_t tb = tab_bytes(U);
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + L.bars);
    int* misc = reinterpret_cast<int*>(smem + L.misc);

    const long long N = p.n_alloc;
    const long long nch = (N + kListRows - 1) / kListRows;
    const long long nb_local = d.n_inst > blockIdx.x ? (d.n_inst - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long items = nb_local * nch;
    auto item_b = [&](long long i) { return (long long)blockIdx.x + (i / nch) * gridDim.x; };
    auto item_n0 = [&](long long i) { return (i % nch) * kListRows; };
    auto issue = [&](long long i) {   // leader thread only
        const long long b = item_b(i), n0 = item_n0(i);
        const long long rows = min((long long)kListRows, N - n0);
        Granules g = granules(p.alloc + (b * N + n0) * J, (size_t)rows * J * 2);
        unsigned char* dst = smem + L.stage + (i % kListStages) * L.stage_bytes;
        mbar_arrive_expect_tx(&bar[i % kListStages], g.bytes);
        bulk_g2s(dst, g.g0, g.bytes, &bar[i % kListStages]);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kListStages; ++s) mbar_init(&bar[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (long long i = 0; i < kListStages && i < items; ++i) issue(i);

    bool ok = true;
    for (long long i = 0; i < items; ++i) {
        const long long b = item_b(i), n0 = item_n0(i);
        const int rows = (int)min((long long)kListRows, N - n0);
        const int s = (int)(i % kListStages);
        if (n0 == 0) {
            // new instance: validate and build all V stream tables (warps in parallel)
            const bool wok = warp_instance_valid(p.t, b, V, nG, nL);
            if (wok) {
                for (int v = warp; v < V; v += nw) {
                    warp_load_stream(sin, p.t, b * V + v, nG, nL);
                    Tabs T = carve_tabs(tabs + v * tb, U);
                    warp_build_tables(sin, U, nG, nL, d.unit_gpu_seconds, d.a_min, T.lad, T.tv, T.tc);
                }
            }
            ok = wok;
            if (!ok && threadIdx.x == 0) flag_data_error(p.st);
            __syncthreads();
        }
        mbar_wait(&bar[s], (unsigned)((i / kListStages) & 1));
        const uint16_t* src = p.alloc + (b * N + n0) * J;
        const uint16_t* rs = reinterpret_cast<const uint16_t*>(smem + L.stage + s * L.stage_bytes +
                                                                granules(src, 2).off);
        uint8_t* cdst = p.out_cfg ? p.out_cfg + (b * N + n0) * V : nullptr;
        uint8_t* cst = smem + L.cfgbuf + (cdst ? granules(cdst, 1).off : 0);
        for (int r = threadIdx.x; r < rows; r += kListThreads) {
            const uint16_t* row = rs + (size_t)r * J;
            bool rok = ok;
            int tot = 0;
            for (int j = 0; j < J; ++j) {
                const int x = row[j];
                tot += x;
                rok &= x <= U;
            }
            rok &= tot <= U;                     // Eq. 1 constraint 2
            unsigned long long S = 0;
            for (int v = 0; v < V; ++v) {
                uint8_t c = 0;
                if (rok) {
                    const int ri = row[2 * v], rt = row[2 * v + 1];
                    const unsigned char* tp = tabs + v * tb;
                    const int l = tp[ri];
                    const int e = rt * kSlots + l;
                    const float val = reinterpret_cast<const float*>(tp + a16((size_t)(U + 1)))[e];
                    c = (tp + a16((size_t)(U + 1)) + a16((size_t)(U + 1) * kSlots * 4))[e];
                    S += q32(val);
                }
                if (cdst) cst[(size_t)r * V + v] = c;
            }
            if (!rok && ok) flag_data_error(p.st);
            const long long o = b * N + n0 + r;
            p.out_sum[o] = S;
            if (p.out_mean) p.out_mean[o] = rok ? mean_q32(S, V) : 0.0f;
        }
        __syncthreads();   // stage s consumed, config bytes staged
        if (threadIdx.x == 0 && i + kListStages < items) issue(i + kListStages);
        if (cdst) {
            store_from_smem(cdst, cst, (size_t)rows * V);
            __syncthreads();
        }
    }
    (void)misc;
    (void)lane;
}

int resident_grid(ekya_handle* h, const void* fn, int threads, size_t smem, long long work) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
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
    p.warp_bytes = a16(sizeof(StreamIn)) + tab_bytes(d.units);
    int warps = kGridWarps;
    size_t smem = p.warp_bytes * warps;
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    if (d.n_inst == 0) return EKYA_OK;
    cudaError_t e = cudaFuncSetAttribute(grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    int grid = resident_grid(h, (const void*)grid_kernel, kGridWarps * 32, smem, (d.n_inst + warps - 1) / warps);
    grid_kernel<<<grid, kGridWarps * 32, smem, s>>>(p);
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
    size_t smem = list_layout(d.units, d.n_streams).total;
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    if (d.n_inst == 0 || n_alloc == 0) return EKYA_OK;
    cudaError_t e = cudaFuncSetAttribute(list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    int grid = resident_grid(h, (const void*)list_kernel, kListThreads, smem, d.n_inst);
    list_kernel<<<grid, kListThreads, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
