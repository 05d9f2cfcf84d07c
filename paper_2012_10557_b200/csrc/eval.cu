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
// LIST: one persistent 32-warp CTA per SM walks its instances.  Instance
// inputs arrive by TMA bulk copy (cp.async.bulk + mbarrier) two instances
// ahead and each instance's allocation rows are bulk-prefetched into L2 one
// instance ahead.  With two table sets in shared memory, step j builds instance
// j+1's V stream tables -- (stream, 32-row block) warp tasks, entries = exact
// Q32 value | config byte -- while instance j's rows are evaluated in 32-row
// chunks, both pulled from one shared task counter (interleaved 1:1).  A row
// is one thread: 8-byte pair loads, one SIMD min clamps both halves (any clamp
// marks the row bad), V table lookups, an add-with-carry exact sum, the mean
// by a correctly rounded reciprocal, 2-byte config stores.
#include <algorithm>
#include <cstdlib>

#include <type_traits>

#include "launch.h"
#include "stream_tables.cuh"

namespace ekya {

namespace {

constexpr int kGridWarps = 32;
constexpr int kListThreads = 1024;

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }

// per-stream table footprint: lad[U+1] + tvc[U+1][rs] (8-byte entries)
// GRID: lad[U+1] (u8 lambda*, 7 = none) + tvc[8][U+1] (lambda-major).  The quads' lanes read
// lad[4 lane + const]: byte entries keep those reads on distinct banks (4-byte entries at a
// 16-byte stride conflicted 4-way)
__host__ __device__ inline size_t grid_tab_bytes(int U) {
    return a16((size_t)(U + 1)) + a16((size_t)(U + 1) * kSlots * 8);
}
__host__ __device__ inline size_t tab_bytes(int U, int rs = kSlots) {
    return a16((size_t)(U + 1)) + a16((size_t)(U + 1) * rs * 8);
}

// first cell of row rt of a stream's triangle
__device__ __forceinline__ int rowstart(int rt, int U) { return rt * (U + 1) - rt * (rt - 1) / 2; }

// row of local cell c: the largest rt in [0, U] with rowstart(rt) <= c
// (float estimate from the quadratic, then exact integer correction)
__device__ __forceinline__ int row_of(int c, int U) {
    const float A = 2.0f * (float)U + 3.0f;
    const float disc = fmaxf(A * A - 8.0f * (float)c, 0.0f);
    int r = (int)((A - sqrtf(disc)) * 0.5f);
    r = max(0, min(r, U));
    while (r < U && rowstart(r + 1, U) <= c) ++r;
    while (r > 0 && rowstart(r, U) > c) --r;
    return r;
}

__device__ __forceinline__ unsigned ld_shared_u8(unsigned a) {
    unsigned v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint2 ld_shared_v2(unsigned a) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
    return v;
}

struct GridTabs {
    uint8_t* lad;
    uint2* tvc;
};
__device__ __forceinline__ GridTabs carve_grid_tabs(unsigned char* p, int U) {
    GridTabs t;
    t.lad = p;
    t.tvc = reinterpret_cast<uint2*>(p + a16((size_t)(U + 1)));
    return t;
}

struct Tabs {
    uint8_t* lad;
    uint2* tvc;
};

// Instance inputs (stale, cost, post, lam_min_units, lam_factor of one
// instance), staged by the TMA one instance ahead (double buffer).
struct InstLayout {
    size_t stale, cost, post, lmu, lf, total;
};
__host__ __device__ inline InstLayout inst_layout(int V, int nG, int nL) {
    InstLayout L;
    size_t o = 0;
    L.stale = o; o += a16((size_t)V * 4) + 16;
    L.cost = o;  o += a16((size_t)V * nG * 4) + 16;
    L.post = o;  o += a16((size_t)V * nG * 4) + 16;
    L.lmu = o;   o += a16((size_t)V * nL * 2) + 16;
    L.lf = o;    o += a16((size_t)V * nL * 4) + 16;
    L.total = a16(o);
    return L;
}

struct ListLayout {
    size_t sin, tabs, tabset, inst, bars, total, inst_bytes;
    int ntabs;   // 2 = double-buffered table sets (build of instance j+1 overlaps rows of j)
};
__host__ __device__ inline ListLayout list_layout(int U, int V, int nG, int nL, int ntabs) {
    ListLayout L;
    size_t o = 0;
    L.ntabs = ntabs;
    L.sin = o;    o += a16(sizeof(StreamIn)) * (size_t)(kListThreads / 32);
    L.tabset = tab_bytes(U, kListRow) * V;
    L.tabs = o;   o += L.tabset * ntabs;
    L.inst_bytes = inst_layout(V, nG, nL).total;
    L.inst = o;   o += 2 * L.inst_bytes;
    L.bars = o;   o += 416;  // list_kernel: 2 mbarriers + 2 task counters; list2_kernel: 18 mbarriers, counter,
                             // bad[2], 32 per-warp row-copy mbarriers
    L.total = o;
    return L;
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
    int grid_qs;         // GRID: 1 = cell-position table staged in shared memory
    ListLayout L;        // LIST: shared-memory layout (host-computed, read from the param space)
    InstLayout IL;
    size_t tb;           // LIST: bytes per stream table
    double rcp_v;        // LIST: RN(1 / V), for the exact mean
    int build_rows;      // LIST: r_train rows per table-build task (multiple of 32)
};

// ------------------------------------------------------------------------
// GRID
// ------------------------------------------------------------------------
// Cell-position table, shared by every stream (the triangle depends only on U):
// for each of the 4 alignments phi of a stream's first cell within a 16-byte
// quad, quad k of the stream covers local cells c = 4k - phi + j (j < 4) and
// qs[phi][k] holds their (rt, ri) as bytes (U <= 255): .x = cells 0, 1 and
// .y = cells 2, 3, each cell ri | rt << 8 (cells outside the stream clamped to
// its first / last cell, never stored).  Larger U: (rt, ri) of the quad's first
// cell is located arithmetically and the others follow along the row.
__host__ __device__ inline size_t cellinfo_quads(int U) {
    const long long NC = (long long)(U + 1) * (U + 2) / 2;
    return (size_t)((NC + 3) / 4 + 1);
}

// NGT / NLT > 0: |Gamma| / |Lambda| fixed at compile time (table build without guards)
template <int GM, int NGT, int NLT>
__global__ void __launch_bounds__(kGridWarps * 32, 1) grid_kernel(EvalParams p) {   // <= 64 regs
    extern __shared__ __align__(128) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int U = d.units, nG = d.n_gamma, nL = d.n_lambda, V = d.n_streams;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t nq_tab = cellinfo_quads(U);
    const bool use_qs = p.grid_qs != 0;   // byte position table in shared memory (U <= 255)
    uint2* qs = reinterpret_cast<uint2*>(smem);
    unsigned char* mine = smem + (use_qs ? a16(4 * nq_tab * sizeof(uint2)) : 0) + (size_t)warp * p.warp_bytes;
    StreamIn* sin = reinterpret_cast<StreamIn*>(mine);
    GridTabs T = carve_grid_tabs(mine + a16(sizeof(StreamIn)), U);
    const int lblk = (U + 1) * 8;   // bytes per lambda block of tvc
    const int NC = (U + 1) * (U + 2) / 2;

    for (int t = threadIdx.x; use_qs && t < (int)(4 * nq_tab); t += blockDim.x) {
        const int phi = t / (int)nq_tab, k = t - phi * (int)nq_tab;
        unsigned w[2] = {0u, 0u};
        for (int j = 0; j < 4; ++j) {
            const int c = min(max(4 * k - phi + j, 0), NC - 1);
            const int rt = row_of(c, U);
            w[j >> 1] |= ((unsigned)(c - rowstart(rt, U)) | ((unsigned)rt << 8)) << (16 * (j & 1));
        }
        qs[t] = make_uint2(w[0], w[1]);
    }
    __syncthreads();

    const int cta_warps = blockDim.x >> 5;
    const long long nwarps = (long long)gridDim.x * cta_warps;
    // one warp per instance (validated once), its V streams in turn
    for (long long b = (long long)blockIdx.x * cta_warps + warp; b < d.n_inst; b += nwarps) {
        const bool ok = warp_instance_valid(p.t, b, V, nG, nL);
        if (!ok && lane == 0) flag_data_error(p.st);
        for (int v = 0; v < V; ++v) {
            const long long item = b * V + v;
            if (ok) {
                warp_load_stream(sin, p.t, item, nG, nL);
                warp_build_tables<GM, NGT, NLT, kSlots, 1, true, uint8_t>(sin, U, nG, nL, d.unit_gpu_seconds, d.a_min,
                                                                          T.lad, T.tvc);
            }
            // Flat write of the stream's cells [f0, f0 + NC) in aligned quads of 4
            // cells: one 16-B value store + one 4-B config store per quad (the
            // value and config arrays share the quad partition).  The quads at the
            // two ends may be shared with the neighbouring streams; only this
            // stream's cells of those are written, with scalar stores.
            const long long f0 = item * NC, f1 = f0 + NC;
            const int phi = (int)(f0 & 3);
            const long long q0 = f0 >> 2;
            const int nq = (int)(((f1 + 3) >> 2) - q0);
            const uint2* qst = qs + (size_t)phi * nq_tab;
            // one quad, any position / validity (edge quads shared with the neighbouring
            // streams, invalid instances, large U without the position table)
            auto quad_generic = [&](int k) {
                const long long fq = (q0 + k) << 2;
                const int c0 = 4 * k - phi;
                // (rt, ri) of the quad's four cells
                int ri[4], rt[4];
                if (use_qs) {
                    const uint2 s2 = qst[k];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const unsigned wj = j < 2 ? s2.x : s2.y;
                        ri[j] = (int)__byte_perm(wj, 0u, 0x4440u + 2u * (j & 1));
                        rt[j] = (int)__byte_perm(wj, 0u, 0x4441u + 2u * (j & 1));
                    }
                } else {
                    const int c = max(c0, 0);
                    int r_t = row_of(c, U);
                    int r_i = c - rowstart(r_t, U);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        rt[j] = r_t;
                        ri[j] = r_i;
                        if (c0 + j >= 0 && ++r_i > U - r_t) {
                            r_t = min(r_t + 1, U);   // past the last cell: stay in range (never stored)
                            r_i = 0;
                        }
                    }
                }
                float v4[4];
                unsigned cfg4 = 0;
                if (ok) {
                    // lad[] holds the byte offset of lambda*'s block: the entry of (rt, ri) is
                    // lad[ri] + rt * 8 bytes into tvc
                    const unsigned char* tv = reinterpret_cast<const unsigned char*>(T.tvc);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint2 vc = *reinterpret_cast<const uint2*>(tv + T.lad[ri[j]] * lblk + rt[j] * 8);
                        v4[j] = __uint_as_float(vc.x);
                        cfg4 |= vc.y << (8 * j);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) v4[j] = 0.0f;
                }
                if (c0 >= 0 && c0 + 4 <= NC) {
                    *reinterpret_cast<float4*>(p.out_grid + fq) = make_float4(v4[0], v4[1], v4[2], v4[3]);
                    if (p.out_grid_cfg) *reinterpret_cast<unsigned*>(p.out_grid_cfg + fq) = cfg4;
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int c = c0 + j;
                        if (c >= 0 && c < NC) {
                            p.out_grid[fq + j] = v4[j];
                            if (p.out_grid_cfg) p.out_grid_cfg[fq + j] = (uint8_t)(cfg4 >> (8 * j));
                        }
                    }
                }
            };
            // quads whose four cells all belong to this stream
            const int k_lo = phi ? 1 : 0, k_hi = (NC + phi) / 4;
            if (ok && use_qs) {
                // interior quads: table entry -> 4 x (lambda* byte offset, entry) through 32-bit
                // shared addresses, one 16-byte value store and one 4-byte config store, with
                // pointers advanced by 32 quads per step
                const unsigned lad_s = smem_addr(T.lad), tvc_s = smem_addr(T.tvc);
                int k = k_lo + lane;
                const uint2* qp = qst + k;
                float4* gp = reinterpret_cast<float4*>(p.out_grid + ((q0 + k) << 2));
                unsigned* cp = p.out_grid_cfg ? reinterpret_cast<unsigned*>(p.out_grid_cfg + ((q0 + k) << 2)) : nullptr;
                // one loop per config-output case: no per-quad null test of the config pointer
                auto interior = [&](auto with_cfg) {
                    for (; k < k_hi; k += 32, qp += 32, gp += 32) {
                        const uint2 s2 = *qp;
                        float v4[4];
                        unsigned cfg4 = 0;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const unsigned wj = j < 2 ? s2.x : s2.y;
                            const unsigned ri = __byte_perm(wj, 0u, 0x4440u + 2u * (j & 1));
                            const unsigned rt = __byte_perm(wj, 0u, 0x4441u + 2u * (j & 1));
                            const unsigned lo = ld_shared_u8(lad_s + ri) * (unsigned)lblk;
                            const uint2 vc = ld_shared_v2(tvc_s + lo + rt * 8);
                            v4[j] = __uint_as_float(vc.x);
                            if constexpr (decltype(with_cfg)::value) cfg4 |= vc.y << (8 * j);
                        }
                        *gp = make_float4(v4[0], v4[1], v4[2], v4[3]);
                        if constexpr (decltype(with_cfg)::value) {
                            *cp = cfg4;
                            cp += 32;
                        }
                    }
                };
                if (cp) interior(std::true_type{});
                else interior(std::false_type{});
                if (lane == 0 && k_lo > 0) quad_generic(0);
                for (int kk = k_hi + lane; kk < nq; kk += 32) quad_generic(kk);
            } else {
                for (int kk = lane; kk < nq; kk += 32) quad_generic(kk);
            }
            __syncwarp();
        }
    }
}

// ------------------------------------------------------------------------
// LIST
// ------------------------------------------------------------------------
// Sum of V LIST entries (Q32 | cfg << 56): low words by an add-with-carry chain
// into the high words; bits 0..23 of the high accumulator hold the Q32 bit-32
// count plus carries (< 2V), the config bytes land in bits 24..31 and are dropped.
struct Q32Sum {
    unsigned lo = 0, hi = 0;
    __device__ __forceinline__ void add(uint2 e) {
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"(e.x), "r"(e.y));
    }
    __device__ __forceinline__ unsigned long long value() const {
        return ((unsigned long long)(hi & 0xFFFFFFu) << 32) | lo;
    }
};

// VT > 0: compile-time stream count (fully unrolled rows); 0: runtime V.  NGT / NLT as GRID.
// UT > 0: the tables are laid out for U = UT (>= the runtime U), so every per-stream table
// offset is a compile-time constant.
template <int GM, int VT, int NGT, int NLT, int UT>
__global__ void __launch_bounds__(kListThreads, 1) list_kernel(EvalParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int U = d.units, nG = d.n_gamma, nL = d.n_lambda, V = VT > 0 ? VT : d.n_streams, J = 2 * V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const ListLayout& L = p.L;
    const InstLayout& IL = p.IL;
    const int tb = UT > 0 ? (int)tab_bytes(UT, kListRow) : (int)p.tb;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + L.bars);
    int* ctr = reinterpret_cast<int*>(smem + L.bars + 16);   // task counters, one per phase parity
    const int N = p.n_alloc;
    const long long B = d.n_inst, g = gridDim.x;

    // leader thread: TMA the inputs of instance b into input buffer k
    auto issue_inputs = [&](long long b, int k) {
        unsigned char* dst = smem + L.inst + k * L.inst_bytes;
        const Granules gs[5] = {granules(p.t.stale + b * V, (size_t)V * 4),
                                granules(p.t.cost + b * V * nG, (size_t)V * nG * 4),
                                granules(p.t.post + b * V * nG, (size_t)V * nG * 4),
                                granules(p.t.lam_min_units + b * V * nL, (size_t)V * nL * 2),
                                granules(p.t.lam_factor + b * V * nL, (size_t)V * nL * 4)};
        const size_t off[5] = {IL.stale, IL.cost, IL.post, IL.lmu, IL.lf};
        unsigned tot = 0;
        for (int i = 0; i < 5; ++i) tot += gs[i].bytes;
        mbar_arrive_expect_tx(&bar[k], tot);
        for (int i = 0; i < 5; ++i)
            if (gs[i].bytes) bulk_g2s(dst + off[i], gs[i].g0, gs[i].bytes, &bar[k]);
    };
    // leader thread: bulk-prefetch instance b's allocation rows into L2 (they are
    // then read with plain coalesced loads)
    auto prefetch_rows = [&](long long b) {
        const Granules gr = granules(p.alloc + b * N * J, (size_t)N * J * 2);
        for (unsigned o = 0; o < gr.bytes; o += (1u << 20)) bulk_prefetch_l2(gr.g0 + o, min(gr.bytes - o, 1u << 20));
    };

    // Staged inputs of instance b (the j-th of this CTA: buffer j & 1).
    struct Staged {
        const float *stale, *cost, *post, *lf;
        const uint16_t* lmu;
    };
    auto staged = [&](long long b, long long j) {
        unsigned char* ib = smem + L.inst + (j & 1) * L.inst_bytes;
        Staged S;
        S.stale = reinterpret_cast<const float*>(ib + IL.stale + granules(p.t.stale + b * V, 4).off);
        S.cost = reinterpret_cast<const float*>(ib + IL.cost + granules(p.t.cost + b * V * nG, 4).off);
        S.post = reinterpret_cast<const float*>(ib + IL.post + granules(p.t.post + b * V * nG, 4).off);
        S.lmu = reinterpret_cast<const uint16_t*>(ib + IL.lmu + granules(p.t.lam_min_units + b * V * nL, 2).off);
        S.lf = reinterpret_cast<const float*>(ib + IL.lf + granules(p.t.lam_factor + b * V * nL, 4).off);
        return S;
    };
    // Wait for instance b's inputs and test them (R-ERR): this thread's share.
    auto validate = [&](long long b, long long j) -> bool {
        mbar_wait(&bar[j & 1], (unsigned)((j >> 1) & 1));
        const Staged S = staged(b, j);
        bool vok = true;
        for (int t = threadIdx.x; t < V; t += blockDim.x) vok &= in01(S.stale[t]);
        for (int t = threadIdx.x; t < V * nG; t += blockDim.x) {
            const float c = S.cost[t];
            if (!(c >= 0.0f)) vok = false;
            else if (!isinf(c)) vok &= in01(S.post[t]);
        }
        for (int t = threadIdx.x; t < V * nL; t += blockDim.x)
            if (S.lmu[t] != kLmuPad) vok &= in01(S.lf[t]);
        return vok;
    };
    // Build task `task` = (stream v, block of 32 r_train rows) of instance b into
    // table set `tabs` (built regardless of validity: an invalid instance's rows
    // are zeroed, so its tables are never read).
    const int brows = p.build_rows, nblk = (U + brows) / brows;   // r_train rows per build task
    StreamIn* si = reinterpret_cast<StreamIn*>(smem + L.sin + (size_t)warp * a16(sizeof(StreamIn)));
    auto build_task = [&](long long b, long long j, unsigned char* tabs, int task) {
        const Staged S = staged(b, j);
        const int v = task / nblk, blk = task - v * nblk;
        if (lane < nG) {
            const float post = S.post[v * nG + lane];
            stream_in_put(si, lane, S.cost[v * nG + lane], post, fsub(post, S.stale[v]));
        }
        if (lane < nL) {
            si->lf[lane] = S.lf[v * nL + lane];
            si->lmu[lane] = S.lmu[v * nL + lane];
        }
        const bool f = lane >= nG || fast_dividend(S.cost[v * nG + lane]);
        const unsigned all = __ballot_sync(0xffffffffu, f);
        if (lane == 0) {
            si->stale = S.stale[v];
            si->fast = all == 0xffffffffu;
        }
        __syncwarp();
        unsigned char* tv = tabs + v * tb;
        const int r1 = min(U + 1, blk * brows + brows);
        warp_build_tables<GM, NGT, NLT, kListRow, 8>(si, U, nG, nL, d.unit_gpu_seconds, d.a_min, tv,
                              reinterpret_cast<unsigned long long*>(tv + a16((size_t)((UT > 0 ? UT : U) + 1))), blk * brows, r1,
                              blk == 0);
    };

    const unsigned UU = (unsigned)U | ((unsigned)U << 16);
    const bool pairs = (V % 2 == 0) && (reinterpret_cast<uintptr_t>(p.alloc) % 8 == 0) &&
                       (!p.out_cfg || reinterpret_cast<uintptr_t>(p.out_cfg) % 2 == 0);
    const int off_tvc = (int)a16((size_t)((UT > 0 ? UT : U) + 1));   // lad[] precedes the entries
    constexpr int kRowBytes = kListRow * 8;
    // Allocation row r of instance b: one thread per row, read straight from global (L2).
    auto row_one = [&](long long b, const unsigned char* tabs, bool ok, int r) {
        if (r >= N) return;
        const long long o = b * N + r;
        unsigned dev = 0;   // any bit set: some r_train / r_infer > U (clamped)
        int tot = 0;
        Q32Sum S;
        const unsigned char* tp = tabs;
        auto look = [&](unsigned pr, const unsigned char* t) -> uint2 {
            const unsigned pc = __vminu2(pr, UU);   // clamp both halves to U
            dev |= pr ^ pc;
            const int ri = (int)(pc & 0xFFFFu), rt = (int)(pc >> 16);
            tot += ri + rt;
            return *reinterpret_cast<const uint2*>(t + off_tvc + rt * kRowBytes + t[ri]);
        };
        bool fast_ok = false;
        if constexpr (VT > 0) {
            // V == VT (even): the whole row in registers, fully unrolled.  One SIMD max over
            // the row decides whether every entry is <= U; then no clamping is needed and the
            // unit total is one packed 16x2 sum (each half <= VT U < 2^16, host-checked).
            if (pairs) {
                constexpr int V2 = VT / 2;
                const uint2* row2 = reinterpret_cast<const uint2*>(p.alloc) + o * V2;
                uint2 pr[V2];
#pragma unroll
                for (int v2 = 0; v2 < V2; ++v2) pr[v2] = __ldg(row2 + v2);
                unsigned mx = 0;
#pragma unroll
                for (int v2 = 0; v2 < V2; ++v2) mx = __vmaxu2(mx, __vmaxu2(pr[v2].x, pr[v2].y));
                if ((mx & 0xFFFFu) <= (unsigned)U && (mx >> 16) <= (unsigned)U) {
                    unsigned acc = 0;
                    uint16_t* cr2 = p.out_cfg ? reinterpret_cast<uint16_t*>(p.out_cfg) + o * V2 : nullptr;
#pragma unroll
                    for (int v2 = 0; v2 < V2; ++v2) {
                        uint2 e[2];
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const unsigned w = hh ? pr[v2].y : pr[v2].x;
                            const unsigned char* t = tabs + (2 * v2 + hh) * tb;
                            acc += w;
                            e[hh] = *reinterpret_cast<const uint2*>(t + off_tvc + (w >> 16) * kRowBytes + t[w & 0xFFFFu]);
                            S.add(e[hh]);
                        }
                        if (cr2) cr2[v2] = (uint16_t)__byte_perm(e[0].y, e[1].y, 0x0073);
                    }
                    tot = (int)((acc & 0xFFFFu) + (acc >> 16));
                    fast_ok = true;
                }
            }
        }
        if (fast_ok) {
        } else if (pairs) {   // two streams per 8-byte row load and per 2-byte config store
            S = Q32Sum();
            tot = 0;
            const uint2* row2 = reinterpret_cast<const uint2*>(p.alloc) + o * (V / 2);
            uint16_t* cr2 = p.out_cfg ? reinterpret_cast<uint16_t*>(p.out_cfg) + o * (V / 2) : nullptr;
            for (int v2 = 0; v2 < V / 2; ++v2, tp += 2 * tb) {
                const uint2 pr = __ldg(row2 + v2);
                const uint2 e0 = look(pr.x, tp), e1 = look(pr.y, tp + tb);
                S.add(e0);
                S.add(e1);
                if (cr2) cr2[v2] = (uint16_t)__byte_perm(e0.y, e1.y, 0x0073);
            }
        } else {
            S = Q32Sum();
            tot = 0;
            const unsigned* row = reinterpret_cast<const unsigned*>(p.alloc) + o * V;
            uint8_t* cr = p.out_cfg ? p.out_cfg + o * V : nullptr;
            for (int v = 0; v < V; ++v, tp += tb) {
                const uint2 e = look(__ldg(row + v), tp);
                S.add(e);
                if (cr) cr[v] = (uint8_t)(e.y >> 24);
            }
        }
        const bool rok = ok && dev == 0 && tot <= U;   // Eq. 1 constraint 2
        unsigned long long s = S.value();
        if (!rok) {                                     // R-ERR: zero the row
            s = 0;
            if (p.out_cfg)
                for (int v = 0; v < V; ++v) p.out_cfg[o * V + v] = 0;
            if (ok) flag_data_error(p.st);
        }
        p.out_sum[o] = s;
        if (p.out_mean) {
            // mean = (float)((double)s / (V 2^32)): s / V by the correctly rounded
            // reciprocal rcp_v = RN(1/V) and one exact-residual correction (Markstein:
            // RN(q0 + r rcp_v) = RN(s / V) for q0 within 1 ulp; s < 2^53, no
            // over/underflow), then the exact power-of-two scale
            const double a = __ull2double_rn(s);
            const double q0 = __dmul_rn(a, p.rcp_v);
            const double q = __fma_rn(__fma_rn(-(double)V, q0, a), p.rcp_v, q0);
            p.out_mean[o] = rok ? __double2float_rn(__dmul_rn(q, 2.3283064365386963e-10)) : 0.0f;
        }
    };

    // Row task c: rows 64c + lane and 64c + 32 + lane (two rows per thread halve the
    // task-queue traffic per row)
    auto row_chunk = [&](long long b, const unsigned char* tabs, bool ok, int c) {
        row_one(b, tabs, ok, c * 64 + lane);
        row_one(b, tabs, ok, c * 64 + 32 + lane);
    };

    // Dynamic task queue of one phase: n_build build tasks of instance bb (into
    // table set tb_build) and n_rows row chunks of instance b, interleaved 1:1
    // while both last so that the issue-bound builds and the memory-bound row
    // chunks share the SM; warps pull tasks from a shared counter.
    int phase = 0;
    auto run_phase = [&](long long bb, long long jb, unsigned char* tabs_build, int n_build, long long b,
                         const unsigned char* tabs_rows, bool ok, int n_rows) {
        int* c = ctr + (phase & 1);
        if (threadIdx.x == 0) ctr[(phase + 1) & 1] = 0;   // used by the previous phase (ended by a barrier)
        ++phase;
        const int m = min(n_build, n_rows), total = n_build + n_rows;
        for (;;) {
            int t = 0;
            if (lane == 0) t = atomicAdd(c, 1);
            t = __shfl_sync(0xffffffffu, t, 0);
            if (t >= total) break;
            bool is_build;
            int idx;
            if (t < 2 * m) {
                is_build = (t & 1) == 0;
                idx = t >> 1;
            } else {
                is_build = n_build > n_rows;
                idx = t - m;
            }
            if (is_build) build_task(bb, jb, tabs_build, idx);
            else row_chunk(b, tabs_rows, ok, idx);
        }
    };

    if (threadIdx.x == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        ctr[0] = 0;
        ctr[1] = 0;
        fence_barrier_init();
    }
    __syncthreads();
    const long long b0 = blockIdx.x;
    if (b0 >= B) return;
    const int n_build = V * nblk, n_chunks = (N + 63) / 64;
    // Double-buffered table sets (ntabs == 2): the phase of step j builds
    // instance j+1's tables while instance j's rows stream; inputs are staged two
    // instances ahead.  Single set (large V x U): build j | barrier | rows j.
    // Step j = -1 (double buffering only) builds instance 0.
    const bool dbl = L.ntabs == 2;
    const int ahead = dbl ? 2 : 1;
    if (threadIdx.x == 0)
        for (int i = 0; i < ahead; ++i)
            if (b0 + i * g < B) issue_inputs(b0 + i * g, i);
    bool ok = true;
    for (long long j = dbl ? -1 : 0; b0 + j * g < B; ++j) {
        const long long b = b0 + j * g, jb = dbl ? j + 1 : j, bb = b0 + jb * g;   // rows of b, build of bb
        if (threadIdx.x == 0) {
            // inputs of instance jb+1 (unless the prologue staged them) into buffer (jb+1) & 1,
            // which held instance jb-1, built before the last barrier
            if (jb + 1 >= ahead && bb + g < B) issue_inputs(bb + g, (int)((jb + 1) & 1));
            if (bb < B) prefetch_rows(bb);
        }
        const bool has_next = bb < B;
        const bool vn = has_next ? validate(bb, jb) : true;
        unsigned char* tabs_b = smem + L.tabs + (dbl ? (jb & 1) : 0) * L.tabset;
        const unsigned char* tabs_r = smem + L.tabs + (dbl ? (j & 1) : 0) * L.tabset;
        if (dbl) {
            run_phase(bb, jb, tabs_b, has_next ? n_build : 0, b, tabs_r, ok, j >= 0 ? n_chunks : 0);
            ok = __syncthreads_and(vn) != 0;   // also frees table set j & 1 and input buffer jb & 1
            if (has_next && !ok && threadIdx.x == 0) flag_data_error(p.st);
        } else {
            run_phase(bb, jb, tabs_b, n_build, b, tabs_r, true, 0);
            ok = __syncthreads_and(vn) != 0;
            if (!ok && threadIdx.x == 0) flag_data_error(p.st);
            run_phase(bb, jb, tabs_b, 0, b, tabs_r, ok, n_chunks);
            __syncthreads();   // tables and input buffer j & 1 are free again
        }
    }
}

// ------------------------------------------------------------------------
// LIST for the paper's shape (V = 10, |Gamma| = 18, |Lambda| = 5, U <= 80), barrier-free
// ------------------------------------------------------------------------
// The same work as list_kernel -- per instance V stream-table builds and N rows -- but the
// CTA never synchronises as a whole.  Tasks come from ONE monotonic shared counter: phase p
// holds the row tasks of instance p-1 (64 rows each) and the build tasks of instance p (one
// stream, all r_train rows, each), interleaved.  Dependencies are mbarriers in rings of 8
// (instance i uses slot i & 7, phase parity (i >> 3) & 1):
//   full[s]  (32 V arrivals: every lane of each build)  the tables of instance i (table set
//            k = i & 1) are built -- each lane's arrive releases its own table writes;
//   empty[s] (32 C arrivals: every lane of each row task)  the rows of instance i are done
//            (set k may be rebuilt);
//   inbar[k] (TMA bytes)   the inputs of instance i are staged in input buffer k.
// A row task of instance i waits on full[i & 7]; a build task of instance i on empty of
// instance i-2 and then inbar[k] (unambiguous: the next copy into buffer k is issued only
// after the builds of i).  Every task waits only on tasks of earlier phases and tasks are
// taken in phase order, so the pipeline cannot deadlock.  Warps may run ahead of the oldest
// unfinished task, but not by 8 phases: every phase after a stalled build holds at least
// min(C, V) tasks blocked behind it, and 4 (C + V) > 32 warps, so a ring slot is never
// re-armed while a waiter of its previous use is pending.  The first row task of instance i (its
// tables are complete, so input buffer k is free) issues the TMA of instance i+2's inputs
// into buffer k and the L2 prefetch of instance i+1's rows.  A build task checks its stream
// (R-ERR) and marks the instance bad by writing i + 1 into bad[k] before it arrives.
constexpr int kL2V = 10, kL2G = 18, kL2L = 5;   // tables laid out for U = 80
constexpr int kL2Rows = 64;                       // rows per row task (two per thread; 32 / 128 / 256 measured slower)

struct List2Params {
    ekya_dims d;
    ekya_tables t;
    DevState* st;
    int n_alloc;
    const uint16_t* alloc;
    unsigned long long* out_sum;
    float* out_mean;
    uint8_t* out_cfg;
    ListLayout L;
    InstLayout IL;
    double rcp_v;
    int chunks;   // row tasks per instance (kL2Rows rows each)
    size_t rowbuf;     // per-warp row staging buffers (shared offset), kL2RowBuf bytes each
};
constexpr int kL2RowBuf = kL2Rows * 2 * kL2V * 2 + 32;   // one task's rows + granule slack

// One allocation row (one thread): V = 10 streams, rows 8-byte aligned, config bytes written
// in pairs; bit-identical to list_kernel's row evaluation.
__device__ __forceinline__ void list2_row(const List2Params& p, const unsigned char* tabs, bool ok, long long o,
                                          const uint2* row2) {
    constexpr int V = kL2V, V2 = kL2V / 2;
    constexpr int tb = 5936;                           // tab_bytes(kL2U, kListRow)
    constexpr int off_tvc = 96;                        // a16(kL2U + 1): lad[] precedes the entries
    constexpr int kRowBytes = kListRow * 8;
    const int U = p.d.units;
    const unsigned UU = (unsigned)U | ((unsigned)U << 16);
    uint2 pr[V2];
#pragma unroll
    for (int v2 = 0; v2 < V2; ++v2) pr[v2] = row2[v2];
    unsigned mx = 0;
#pragma unroll
    for (int v2 = 0; v2 < V2; ++v2) mx = __vmaxu2(mx, __vmaxu2(pr[v2].x, pr[v2].y));
    Q32Sum S;
    int tot;
    unsigned dev = 0;   // any bit set: some r_train / r_infer > U (clamped)
    uint16_t* cr2 = p.out_cfg ? reinterpret_cast<uint16_t*>(p.out_cfg) + o * V2 : nullptr;
    if ((mx & 0xFFFFu) <= (unsigned)U && (mx >> 16) <= (unsigned)U) {
        // every entry <= U: no clamping; the unit total is one packed 16x2 sum (<= V U < 2^16)
        unsigned acc = 0;
#pragma unroll
        for (int v2 = 0; v2 < V2; ++v2) {
            uint2 e[2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const unsigned w = hh ? pr[v2].y : pr[v2].x;
                const unsigned char* t = tabs + (2 * v2 + hh) * tb;
                acc += w;
                e[hh] = *reinterpret_cast<const uint2*>(t + off_tvc + (w >> 16) * kRowBytes + t[w & 0xFFFFu]);
                S.add(e[hh]);
            }
            if (cr2) cr2[v2] = (uint16_t)__byte_perm(e[0].y, e[1].y, 0x0073);
        }
        tot = (int)((acc & 0xFFFFu) + (acc >> 16));
    } else {
        // some entry > U: clamp to U, evaluate, and flag the row below (R-ERR)
        tot = 0;
#pragma unroll
        for (int v2 = 0; v2 < V2; ++v2) {
            uint2 e[2];
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                const unsigned w = hh ? pr[v2].y : pr[v2].x;
                const unsigned pc = __vminu2(w, UU);
                dev |= w ^ pc;
                const int ri = (int)(pc & 0xFFFFu), rt = (int)(pc >> 16);
                tot += ri + rt;
                const unsigned char* t = tabs + (2 * v2 + hh) * tb;
                e[hh] = *reinterpret_cast<const uint2*>(t + off_tvc + rt * kRowBytes + t[ri]);
                S.add(e[hh]);
            }
            if (cr2) cr2[v2] = (uint16_t)__byte_perm(e[0].y, e[1].y, 0x0073);
        }
    }
    const bool rok = ok && dev == 0 && tot <= U;   // Eq. 1 constraint 2
    unsigned long long s = S.value();
    if (!rok) {                                     // R-ERR: zero the row
        s = 0;
        if (p.out_cfg)
            for (int v = 0; v < V; ++v) p.out_cfg[o * V + v] = 0;
        if (ok) flag_data_error(p.st);
    }
    p.out_sum[o] = s;
    if (p.out_mean) {
        // mean = (float)((double)s / (V 2^32)) by the correctly rounded reciprocal and one
        // exact-residual correction (as list_kernel)
        const double a = __ull2double_rn(s);
        const double q0 = __dmul_rn(a, p.rcp_v);
        const double q = __fma_rn(__fma_rn(-(double)V, q0, a), p.rcp_v, q0);
        p.out_mean[o] = rok ? __double2float_rn(__dmul_rn(q, 2.3283064365386963e-10)) : 0.0f;
    }
}

__global__ void __launch_bounds__(kListThreads, 1) list2_kernel(const __grid_constant__ List2Params p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int V = kL2V, nG = kL2G, nL = kL2L;
    constexpr int tb = 5936;
    const ekya_dims& d = p.d;
    constexpr int RT = kL2Rows;
    const int U = d.units, N = p.n_alloc, C = p.chunks, T = C + V;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const ListLayout& L = p.L;
    const InstLayout& IL = p.IL;
    unsigned long long* inbar = reinterpret_cast<unsigned long long*>(smem + L.bars);
    unsigned long long* full = inbar + 2;    // [8]
    unsigned long long* empty = inbar + 10;  // [8]
    unsigned* ctr = reinterpret_cast<unsigned*>(inbar + 18);
    int* bad = reinterpret_cast<int*>(ctr + 1);   // bad[k] = i + 1: instance i (set k) is invalid
    const long long B = d.n_inst, g = gridDim.x, b0 = blockIdx.x;
    const long long n = B > b0 ? (B - 1 - b0) / g + 1 : 0;   // instances of this CTA
    if (n == 0) return;

    auto issue_inputs = [&](long long b, int k) {
        unsigned char* dst = smem + L.inst + k * L.inst_bytes;
        const Granules gs[5] = {granules(p.t.stale + b * V, (size_t)V * 4),
                                granules(p.t.cost + b * V * nG, (size_t)V * nG * 4),
                                granules(p.t.post + b * V * nG, (size_t)V * nG * 4),
                                granules(p.t.lam_min_units + b * V * nL, (size_t)V * nL * 2),
                                granules(p.t.lam_factor + b * V * nL, (size_t)V * nL * 4)};
        const size_t off[5] = {IL.stale, IL.cost, IL.post, IL.lmu, IL.lf};
        unsigned tot = 0;
        for (int i = 0; i < 5; ++i) tot += gs[i].bytes;
        mbar_arrive_expect_tx(&inbar[k], tot);
        for (int i = 0; i < 5; ++i)
            if (gs[i].bytes) bulk_g2s(dst + off[i], gs[i].g0, gs[i].bytes, &inbar[k]);
    };

    if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k) {
            mbar_init(&inbar[k], 1);
            bad[k] = 0;
        }
        for (int s = 0; s < 8; ++s) {
            mbar_init(&full[s], 32 * V);
            mbar_init(&empty[s], 32 * C);
        }
        for (int w = 0; w < kListThreads / 32; ++w) mbar_init(&inbar[20 + w], 1);
        *ctr = 0;
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        issue_inputs(b0, 0);
        if (n > 1) issue_inputs(b0 + g, 1);
    }

    StreamIn* si = reinterpret_cast<StreamIn*>(smem + L.sin + (size_t)warp * a16(sizeof(StreamIn)));
    // this warp's row staging buffer and its TMA barrier (phase = number of row tasks so far)
    unsigned char* rbuf = smem + p.rowbuf + (size_t)warp * kL2RowBuf;
    unsigned long long* rbar = inbar + 20 + warp;
    unsigned rphase = 0;
    const unsigned total = (unsigned)((n + 1) * T);
    // phase layout: R0 rows, then builds and rows alternating, then what is left -- the builds
    // of instance ph start once the rows of ph - 2 (previous phase) have had time to drain, and
    // end well before the rows of ph (next phase) need them
    const int R0 = C / 4, m = min(V, C - R0);
    long long ph = 0;        // this warp's phase (tasks are taken in increasing order)
    unsigned pstart = 0;     // first task of phase ph
    for (;;) {
        unsigned tau = 0;
        if (lane == 0) tau = atomicAdd(ctr, 1u);
        tau = __shfl_sync(0xffffffffu, tau, 0);
        if (tau >= total) break;
        while (tau >= pstart + (unsigned)T) {
            ++ph;
            pstart += (unsigned)T;
        }
        const int t = (int)(tau - pstart);
        bool is_build;
        int idx;
        if (t < R0) {
            is_build = false;
            idx = t;
        } else if (t < R0 + 2 * m) {
            is_build = ((t - R0) & 1) == 0;
            idx = is_build ? (t - R0) >> 1 : R0 + ((t - R0) >> 1);
        } else {
            is_build = V > C - R0;
            idx = is_build ? t - R0 - m : t - m;
        }
        if (is_build) {
            const long long i = ph;
            if (i >= n) continue;
            const int k = (int)(i & 1);
            const unsigned par = (unsigned)((i >> 1) & 1);
            if (i >= 2) mbar_wait_sleep(&empty[(i - 2) & 7], (unsigned)(((i - 2) >> 3) & 1));   // rows of i - 2 done
            mbar_wait_sleep(&inbar[k], par);
            const long long b = b0 + i * g;
            const unsigned char* ib = smem + L.inst + k * L.inst_bytes;
            const float* stale = reinterpret_cast<const float*>(ib + IL.stale + granules(p.t.stale + b * V, 4).off);
            const float* cost = reinterpret_cast<const float*>(ib + IL.cost + granules(p.t.cost + b * V * nG, 4).off);
            const float* post = reinterpret_cast<const float*>(ib + IL.post + granules(p.t.post + b * V * nG, 4).off);
            const uint16_t* lmu =
                reinterpret_cast<const uint16_t*>(ib + IL.lmu + granules(p.t.lam_min_units + b * V * nL, 2).off);
            const float* lf = reinterpret_cast<const float*>(ib + IL.lf + granules(p.t.lam_factor + b * V * nL, 4).off);
            const int v = idx;
            // stream v's profile into the warp's StreamIn, with its R-ERR checks
            const float st = stale[v];
            bool vok = in01(st);
            float c = 0.0f;
            if (lane < nG) {
                c = cost[v * nG + lane];
                const float po = post[v * nG + lane];
                if (!(c >= 0.0f)) vok = false;
                else if (!isinf(c)) vok &= in01(po);
                stream_in_put(si, lane, c, po, fsub(po, st));
            }
            if (lane < nL) {
                const float f = lf[v * nL + lane];
                const uint16_t mu = lmu[v * nL + lane];
                if (mu != kLmuPad) vok &= in01(f);
                si->lf[lane] = f;
                si->lmu[lane] = mu;
            }
            const bool allok = __all_sync(0xffffffffu, vok);
            const unsigned fastm = __ballot_sync(0xffffffffu, lane >= nG || fast_dividend(c));
            if (lane == 0) {
                si->stale = st;
                si->fast = fastm == 0xffffffffu;
                if (!allok) {
                    bad[k] = (int)(i + 1);
                    flag_data_error(p.st);
                }
            }
            __syncwarp();
            unsigned char* tv = smem + L.tabs + k * L.tabset + v * tb;
            warp_build_tables<19, kL2G, kL2L, kListRow, 8, false, uint8_t, true>(si, U, nG, nL, d.unit_gpu_seconds, d.a_min, tv,
                                                          reinterpret_cast<unsigned long long*>(tv + 96), 0, U + 1,
                                                          true);
            mbar_arrive(&full[i & 7]);
        } else {
            const long long i = ph - 1;
            if (i < 0) continue;
            const int k = (int)(i & 1);
            const long long b = b0 + i * g;
            // the task's rows (contiguous) into the warp's buffer by one bulk copy, issued before
            // the wait for the instance's tables so that the two latencies overlap
            const int rb = idx * RT, nr = min(RT, N - rb);
            const long long o0 = b * N + rb;   // first row of the task
            const uintptr_t ga = reinterpret_cast<uintptr_t>(p.alloc) + (uintptr_t)o0 * (2 * V * 2);
            const unsigned off = (unsigned)(ga & 15u), bytes = (off + (unsigned)nr * (2 * V * 2) + 15u) & ~15u;
            if (lane == 0) {
                mbar_arrive_expect_tx(rbar, bytes);
                bulk_g2s(rbuf, reinterpret_cast<const void*>(ga - off), bytes, rbar);
            }
            mbar_wait_sleep(&full[i & 7], (unsigned)((i >> 3) & 1));
            if (idx == 0 && lane == 0 && i + 2 < n)   // instance i's tables are complete: buffer k is free
                issue_inputs(b0 + (i + 2) * g, k);
            const bool ok = bad[k] != (int)(i + 1);
            const unsigned char* tabs = smem + L.tabs + k * L.tabset;
            mbar_wait_sleep(rbar, rphase & 1u);
            ++rphase;
            const uint2* rows = reinterpret_cast<const uint2*>(rbuf + off);
            if (lane < nr) list2_row(p, tabs, ok, o0 + lane, rows + lane * (V / 2));
            if (lane + 32 < nr) list2_row(p, tabs, ok, o0 + lane + 32, rows + (lane + 32) * (V / 2));
            __syncwarp();   // every lane's reads of the buffer precede the next task's copy
            mbar_arrive(&empty[i & 7]);
        }
    }
}

int resident_grid(ekya_handle* h, const void* fn, int threads, size_t smem, long long work) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem);
    per_sm = std::max(per_sm, 1);
    long long g = (long long)h->sm_count * per_sm;
    return (int)std::max(1LL, std::min(g, work));
}

}  // namespace

// register slots for {none} + Gamma: the paper's |Gamma| = 18 gets an exact fit
template <typename F>
F* pick_gm(int nG, F* k8, F* k16, F* k19, F* k24, F* k32) {
    const int g1 = nG + 1;
    return g1 <= 8 ? k8 : g1 <= 16 ? k16 : g1 <= 19 ? k19 : g1 <= 24 ? k24 : k32;
}

int launch_eval_grid(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, float* out_grid,
                     uint8_t* out_grid_cfg, cudaStream_t s) {
    if (d.units > 4094) return EKYA_ERR_SHAPE;   // rt * kSlots must fit 16 bits
    if ((reinterpret_cast<uintptr_t>(out_grid) & 15) || (reinterpret_cast<uintptr_t>(out_grid_cfg) & 3))
        return EKYA_ERR_ARG;
    EvalParams p{};
    p.d = d;
    p.t = t;
    p.st = h->dstate;
    p.out_grid = out_grid;
    p.out_grid_cfg = out_grid_cfg;
    p.warp_bytes = a16(sizeof(StreamIn)) + grid_tab_bytes(d.units);
    // the position table (16 B per 4 cells of a stream) is staged only while it
    // leaves room for all warps' tables; beyond that each quad locates its row
    // arithmetically, and large U runs fewer warps per CTA (>= 1)
    const size_t qsb = a16(4 * cellinfo_quads(d.units) * sizeof(uint2));
    p.grid_qs = d.units <= 255 && qsb + p.warp_bytes * kGridWarps <= h->smem_optin;
    const size_t avail = h->smem_optin - (p.grid_qs ? qsb : 0);
    const int warps = (int)std::min<size_t>(kGridWarps, avail / p.warp_bytes);
    if (warps < 1) return EKYA_ERR_SHAPE;
    const size_t smem = p.warp_bytes * warps + (p.grid_qs ? qsb : 0);
    if (d.n_inst == 0) return EKYA_OK;
    // the paper's shape (|Gamma| = 18, |Lambda| = 5) gets a guard-free table build
    auto kern = (d.n_gamma == 18 && d.n_lambda == 5)
                    ? grid_kernel<19, 18, 5>
                    : pick_gm(d.n_gamma, grid_kernel<8, 0, 0>, grid_kernel<16, 0, 0>, grid_kernel<19, 0, 0>,
                              grid_kernel<24, 0, 0>, grid_kernel<32, 0, 0>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    int grid = resident_grid(h, (const void*)kern, warps * 32, smem, (d.n_inst + warps - 1) / warps);
    kern<<<grid, warps * 32, smem, s>>>(p);
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
    if (reinterpret_cast<uintptr_t>(alloc) & 3) return EKYA_ERR_ARG;
    // the paper's shape (V = 10 streams, |Gamma| = 18, |Lambda| = 5, U <= 80) gets the
    // unrolled-row kernel with tables laid out for U = 80 (compile-time offsets)
    constexpr int kFastU = 80;
    const bool fast = d.n_streams == 10 && d.n_gamma == 18 && d.n_lambda == 5 && d.units <= kFastU;
    const int lu = fast ? kFastU : d.units;   // table layout
    p.L = list_layout(lu, d.n_streams, d.n_gamma, d.n_lambda, 2);
    if (p.L.total > h->smem_optin) p.L = list_layout(lu, d.n_streams, d.n_gamma, d.n_lambda, 1);
    p.IL = inst_layout(d.n_streams, d.n_gamma, d.n_lambda);
    p.tb = tab_bytes(lu, kListRow);
    p.rcp_v = 1.0 / (double)d.n_streams;
    // Many rows per instance: one build task per stream (staging and the lambda ladder done
    // once, all r_train rows in one warp) -- the row chunks keep every warp busy meanwhile.
    // Few rows: 32-row build tasks, so that the build itself spreads over the CTA's warps.
    p.build_rows = n_alloc >= 1024 ? ((d.units + 32) / 32) * 32 : 32;
    size_t smem = p.L.total;
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    if (d.n_inst == 0 || n_alloc == 0) return EKYA_OK;
    // the paper's shape with 8-byte aligned rows and 2-byte aligned config output: the
    // barrier-free pipeline (list2_kernel), its task counter bounded by 2^32
    const long long per_cta = (d.n_inst + h->sm_count - 1) / h->sm_count;
    const int chunks = (n_alloc + kL2Rows - 1) / kL2Rows;
    if (fast && p.L.ntabs == 2 && !(reinterpret_cast<uintptr_t>(alloc) & 7) &&
        !(reinterpret_cast<uintptr_t>(out_cfg) & 1) && (per_cta + 1) * (long long)(chunks + 10) < (1LL << 32) &&
        !getenv("EKYA_LIST_V1")) {
        List2Params q{};
        q.d = d;
        q.t = t;
        q.st = h->dstate;
        q.n_alloc = n_alloc;
        q.alloc = alloc;
        q.out_sum = p.out_sum;
        q.out_mean = out_mean;
        q.out_cfg = out_cfg;
        q.L = p.L;
        q.IL = p.IL;
        q.rcp_v = p.rcp_v;
        q.chunks = chunks;
        q.rowbuf = a16(smem);
        smem = q.rowbuf + (size_t)kL2RowBuf * (kListThreads / 32);
        if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
        cudaError_t e2 = cudaFuncSetAttribute(list2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e2 != cudaSuccess) return EKYA_ERR_CUDA;
        const int grid = (int)std::min<long long>(h->sm_count, d.n_inst);
        list2_kernel<<<grid, kListThreads, smem, s>>>(q);
        h->launches++;
        return cuda_status(cudaGetLastError());
    }
    auto kern = fast ? list_kernel<19, 10, 18, 5, kFastU>
                     : pick_gm(d.n_gamma, list_kernel<8, 0, 0, 0, 0>, list_kernel<16, 0, 0, 0, 0>,
                               list_kernel<19, 0, 0, 0, 0>, list_kernel<24, 0, 0, 0, 0>, list_kernel<32, 0, 0, 0, 0>);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    int grid = resident_grid(h, (const void*)kern, kListThreads, smem, d.n_inst);
    kern<<<grid, kListThreads, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
