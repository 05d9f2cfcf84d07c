// baselines.cu -- NEXT-3: the uniform scheduler the paper compares
// against (readings U1, U2 in DESIGN.md) and the Pareto
// frontier of a stream's retraining configurations (reading PR1).
//
// ekya_uniform_schedule: one warp per instance, lanes over streams: the static
// split (C9's per-stream share, inference weight w), the fixed retraining config
// (or each stream's highest-accuracy config), lambda* (rule 3) and the window
// average of rule 2 -- then the exact Q32 objective by a warp reduction.
// ekya_pareto: one thread per (instance, stream) set, its configs in registers,
// the O(n^2) dominance test sequential.
// ekya_prune_configs: history-based pruning, one warp per stream.
#include <algorithm>

#include "launch.h"
#include "stream_tables.cuh"

namespace ekya {

namespace {

constexpr int kBaseWarps = 8;

struct UniformParams {
    ekya_dims d;
    ekya_tables t;
    int fixed_gamma;
    float weight;
    uint16_t* out_alloc;
    uint8_t* out_cfg;
    unsigned long long* out_sum;
    float* out_mean;
    DevState* st;
};

constexpr int kUniStage = 512;   // staged (cost, post) floats per warp

// The instance's cost and post tables are read once, coalesced, for the validity test and
// kept in the warp's shared memory (V nG <= kUniStage) for the per-stream scans, so the
// lanes' scans hit shared memory instead of issuing dependent global loads.
__global__ void __launch_bounds__(kBaseWarps * 32) uniform_kernel(UniformParams p) {
    __shared__ float s_cost[kBaseWarps][kUniStage], s_post[kBaseWarps][kUniStage];
    const ekya_dims& d = p.d;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int V = d.n_streams, J = 2 * V, nG = d.n_gamma, nL = d.n_lambda, U = d.units;
    const float keep = fsub(1.0f, p.weight);
    const bool stage = V * nG <= kUniStage;
    for (long long b = (long long)blockIdx.x * kBaseWarps + warp; b < d.n_inst;
         b += (long long)gridDim.x * kBaseWarps) {
        // R-ERR validity (as warp_instance_valid), staging cost and post on the way
        bool vok = true;
        const long long v0 = b * V;
        for (int i = lane; i < V; i += 32) vok &= in01(__ldg(p.t.stale + v0 + i));
        __syncwarp();   // the previous instance's scans are done with the staging buffers
        for (int i = lane; i < V * nG; i += 32) {
            const float c = __ldg(p.t.cost + v0 * nG + i), po = __ldg(p.t.post + v0 * nG + i);
            if (!(c >= 0.0f)) vok = false;
            else if (!isinf(c)) vok &= in01(po);
            if (stage) {
                s_cost[warp][i] = c;
                s_post[warp][i] = po;
            }
        }
        for (int i = lane; i < V * nL; i += 32)
            if (__ldg(p.t.lam_min_units + v0 * nL + i) != kLmuPad) vok &= in01(__ldg(p.t.lam_factor + v0 * nL + i));
        const bool ok = __all_sync(0xffffffffu, vok);
        if (!ok && lane == 0) flag_data_error(p.st);
        __syncwarp();   // the staged tables are visible to every lane (a vote is not a fence)
        unsigned long long S = 0;
        for (int v = lane; v < V; v += 32) {
            // U1: static split
            const int share = U / V + (v < U % V ? 1 : 0);
            const int rt = (int)floorf(fmul(__int2float_rn(share), keep));
            const int ri = share - rt;
            const long long bv = b * V + v;
            const float stale = __ldg(p.t.stale + bv);
            const float* cost = stage ? s_cost[warp] + v * nG : p.t.cost + bv * nG;
            const float* post = stage ? s_post[warp] + v * nG : p.t.post + bv * nG;
            // U2: the fixed retraining config (1-based, 0 = none)
            int g = p.fixed_gamma;
            if (g < 0) {
                g = 0;
                float bp = 0.0f;
                for (int k = 0; k < nG; ++k) {
                    if (isinf(cost[k])) continue;   // padding
                    const float pk = post[k];
                    if (g == 0 || pk > bp) {
                        g = k + 1;
                        bp = pk;
                    }
                }
            }
            const int l = lambda_star(stale, p.t.lam_min_units + bv * nL, p.t.lam_factor + bv * nL, nL, ri, d.a_min);
            float val = 0.0f;
            uint8_t cfg = (uint8_t)(kLambdaNone << 5);
            if (l >= 0) {
                float acc = stale, w;
                if (g > 0 && window_acc(stale, post[g - 1], cost[g - 1], rt, d.unit_gpu_seconds, &w))
                    acc = w;
                val = fmul(__ldg(p.t.lam_factor + bv * nL + l), acc);
                cfg = (uint8_t)(g | (l << 5));
            }
            p.out_alloc[b * J + 2 * v] = ok ? (uint16_t)ri : 0;
            p.out_alloc[b * J + 2 * v + 1] = ok ? (uint16_t)rt : 0;
            p.out_cfg[bv] = ok ? cfg : 0;
            S += q32(val);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
        if (lane == 0) {
            p.out_sum[b] = ok ? S : 0ULL;
            if (p.out_mean) p.out_mean[b] = ok ? mean_q32(S, V) : 0.0f;
        }
    }
}

struct ParetoParams {
    long long n_sets;
    int n;
    const float* cost;
    const float* post;
    uint32_t* out_mask;
    DevState* st;
};

// one set per thread: the set's n <= 31 (cost, post) pairs in registers (NM = compile-time
// bound), the O(n^2) dominance test sequential -- far fewer instructions than a warp per set
template <int NM>
__global__ void __launch_bounds__(256) pareto_kernel(ParetoParams p) {
    const int n = p.n;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < p.n_sets;
         s += (long long)gridDim.x * blockDim.x) {
        float c[NM], q[NM];
        bool pad[NM];
        bool ok = true;   // R-ERR: costs >= 0 (+INF = padding), real accuracies in [0, 1]
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            c[k] = k < n ? __ldg(p.cost + s * n + k) : INFINITY;
            q[k] = k < n ? __ldg(p.post + s * n + k) : 0.0f;
            pad[k] = isinf(c[k]);
            ok &= c[k] >= 0.0f && (pad[k] || (q[k] >= 0.0f && q[k] <= 1.0f));
            // padding never dominates: its accuracy below every real one (>= any real q
            // fails); identical points never dominate each other, so j = k needs no test
            if (pad[k]) q[k] = -INFINITY;
        }
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            bool dom = pad[k];
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                if (j == k) continue;
                // branch-free: cost' <= cost, post' >= post, and not the same point
                dom |= (c[j] <= c[k]) & (q[j] >= q[k]) & ((c[j] != c[k]) | (q[j] != q[k]));
            }
            m |= dom ? 0u : (1u << k);
        }
        if (!ok) flag_data_error(p.st);
        p.out_mask[s] = ok ? m : 0u;
    }
}

struct PruneParams {
    long long n_query;
    int H, n;
    const float* cost;
    const float* acc;
    float margin;
    uint32_t* out_keep;
    DevState* st;
};

// PN1-PN3: one warp per stream (query).  The stream's real configs are ranked by (cost, index)
// once; per history window the Pareto boundary at every config's cost is then a prefix
// maximum in that order (equal costs share the value at their group's end), so a window
// costs one pass forward and one backward over n registers instead of n^2 comparisons.
// Lanes own windows: each warp stages 32 consecutive windows (n floats each, contiguous)
// with coalesced loads into shared memory and every lane reads its own row in cost order.
// Counts per config: measured in the low, far in the high 16 bits of one register (a lane
// sees at most ceil(H / 32) <= 32768 windows).
template <int NM>
__global__ void __launch_bounds__(kBaseWarps * 32) prune_kernel(PruneParams p) {
    __shared__ float rows[kBaseWarps][32 * 31];
    __shared__ uint8_t perm_s[kBaseWarps][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = p.H, n = p.n;
    float* sr = rows[warp];
    for (long long q = (long long)blockIdx.x * kBaseWarps + warp; q < p.n_query;
         q += (long long)gridDim.x * kBaseWarps) {
        const float ck = lane < n ? __ldg(p.cost + q * n + lane) : INFINITY;
        const bool cok = lane >= n || ck >= 0.0f;   // NaN or negative cost: R-ERR
        const bool real = lane < n && cok && !isinf(ck);
        // rank by (cost, index) among the real configs; group end = no later equal cost
        int rank = 0;
        bool later_tie = false;
        for (int k2 = 0; k2 < n; ++k2) {
            const float c2 = __shfl_sync(0xffffffffu, ck, k2);
            const bool r2 = __shfl_sync(0xffffffffu, real, k2);
            if (r2 && (c2 < ck || (c2 == ck && k2 < lane))) ++rank;
            if (r2 && c2 == ck && k2 > lane) later_tie = true;
        }
        const int nr = __popc(__ballot_sync(0xffffffffu, real));
        const unsigned ends = __reduce_or_sync(0xffffffffu, real && !later_tie ? 1u << rank : 0u);
        if (real) perm_s[warp][rank] = (uint8_t)lane;
        __syncwarp();
        int pi[NM];
#pragma unroll
        for (int i = 0; i < NM; ++i) pi[i] = i < nr ? perm_s[warp][i] : 0;
        unsigned cnt[NM];
#pragma unroll
        for (int i = 0; i < NM; ++i) cnt[i] = 0;
        bool aok = true;
        const float* A = p.acc + q * (long long)H * n;
        for (int j0 = 0; j0 < H; j0 += 32) {
            const int nw = min(32, H - j0);
            const float* src = A + (long long)j0 * n;
            __syncwarp();
            for (int e = lane; e < nw * n; e += 32) sr[e] = __ldg(src + e);
            __syncwarp();
            if (lane < nw) {
                const float* a = sr + lane * n;
                float av[NM], pm[NM];
                float m = -INFINITY;
#pragma unroll
                for (int i = 0; i < NM; ++i) {
                    if (i < nr) {
                        av[i] = a[pi[i]];
                        aok &= isnan(av[i]) || in01(av[i]);
                        m = fmaxf(m, av[i]);   // NaN (unmeasured) never wins
                        pm[i] = m;
                    }
                }
                float cur = -INFINITY;
#pragma unroll
                for (int i = NM - 1; i >= 0; --i) {
                    if (i < nr) {
                        if (ends >> i & 1) cur = pm[i];
                        if (!isnan(av[i])) cnt[i] += 1u + ((fsub(cur, av[i]) > p.margin) ? 0x10000u : 0u);
                    }
                }
            }
        }
        const bool ok = __all_sync(0xffffffffu, cok && aok);
        unsigned keep = 0;
#pragma unroll
        for (int i = 0; i < NM; ++i) {
            if (i < nr) {
                const unsigned meas = __reduce_add_sync(0xffffffffu, cnt[i] & 0xFFFFu);
                const unsigned far = __reduce_add_sync(0xffffffffu, cnt[i] >> 16);
                if (!(2ull * far > meas)) keep |= 1u << pi[i];
            }
        }
        if (lane == 0) {
            if (!ok) flag_data_error(p.st);
            p.out_keep[q] = ok ? keep : 0u;
        }
        __syncwarp();   // perm_s / rows are rewritten by the next query
    }
}

__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(K) : "memory"); }
constexpr int kPruneWarps = 4, kPruneStages = 3;

// The same for streams of exactly N configs (the paper's |Gamma| = 18).  Each warp copies its
// next 32 windows with cp.async while it evaluates the current 32 (two buffers), storing
// every row in cost order (column k to position rank(k); padding positions hold NaN, i.e.
// unmeasured), so a lane reads its row with 8-byte loads at compile-time offsets.  The
// accuracy range check folds into a NaN-ignoring minimum and the prefix maximum.  Without
// equal costs the boundary is the prefix maximum itself; with them (rare) the prefix maxima
// overwrite the row and the accuracies are re-read from global memory (L2).
template <int N>
__global__ void __launch_bounds__(kPruneWarps * 32, 8) prune_sorted_kernel(PruneParams p) {
    static_assert(N % 2 == 0, "8-byte row loads");
    __shared__ __align__(16) float rows[kPruneWarps][kPruneStages][32 * N];
    __shared__ int dst_s[kPruneWarps][N];   // column k -> position rank(k), or -1 (padding)
    __shared__ int col_s[kPruneWarps][N];   // position -> column, or -1 (padding)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int H = p.H;
    for (long long q = (long long)blockIdx.x * kPruneWarps + warp; q < p.n_query;
         q += (long long)gridDim.x * kPruneWarps) {
        const float ck = lane < N ? __ldg(p.cost + q * N + lane) : INFINITY;
        const bool cok = lane >= N || ck >= 0.0f;
        const bool real = lane < N && cok && !isinf(ck);
        int rank = 0;
        bool later_tie = false;
#pragma unroll
        for (int k2 = 0; k2 < N; ++k2) {
            const float c2 = __shfl_sync(0xffffffffu, ck, k2);
            const bool r2 = __shfl_sync(0xffffffffu, real, k2);
            if (r2 && (c2 < ck || (c2 == ck && k2 < lane))) ++rank;
            if (r2 && c2 == ck && k2 > lane) later_tie = true;
        }
        const unsigned rm = __ballot_sync(0xffffffffu, real);
        const int nr = __popc(rm);
        const unsigned ends = __reduce_or_sync(0xffffffffu, real && !later_tie ? 1u << rank : 0u);
        const bool ties = ends != (1u << nr) - 1u;
        __syncwarp();
        if (lane < N) {
            const int pos = real ? rank : nr + lane - __popc(rm & ((1u << lane) - 1u));
            dst_s[warp][lane] = real ? pos : -1;
            col_s[warp][pos] = real ? lane : -1;
        }
        for (int e = lane; e < 32 * (N - nr); e += 32) {   // padding positions: NaN in every buffer
            const int w = e / (N - nr), k = nr + (e - w * (N - nr));
#pragma unroll
            for (int sb = 0; sb < kPruneStages; ++sb) rows[warp][sb][w * N + k] = __int_as_float(0x7fc00000);
        }
        __syncwarp();
        const float* A = p.acc + q * (long long)H * N;
        auto issue = [&](int buf, int j0) {
            const int nw = min(32, H - j0);
            const float* src = A + (long long)j0 * N;
            float* dst = rows[warp][buf];
            int w = lane / N, col = lane - (lane / N) * N;   // element lane + 32 t = w N + col
#pragma unroll 6
            for (int t = 0; t < N; ++t) {
                if (w < nw) {
                    const int d = dst_s[warp][col];
                    if (d >= 0) cp_async4(dst + w * N + d, src + w * N + col);
                }
                col += 32 % N;
                w += 32 / N;
                if (col >= N) col -= N, ++w;
            }
            cp_async_commit();
        };
        unsigned cnt[N];
#pragma unroll
        for (int i = 0; i < N; ++i) cnt[i] = 0;
        float lo = 0.0f, hi = 0.0f;   // NaN-ignoring range of the measured accuracies
#pragma unroll
        for (int sb = 0; sb < kPruneStages - 1; ++sb) {
            if (32 * sb < H) issue(sb, 32 * sb);
            else cp_async_commit();
        }
        for (int j0 = 0, it = 0; j0 < H; j0 += 32, ++it) {
            const int jn = j0 + 32 * (kPruneStages - 1);
            if (jn < H) issue((it + kPruneStages - 1) % kPruneStages, jn);
            else cp_async_commit();
            cp_async_wait<kPruneStages - 1>();
            __syncwarp();
            float* sr = rows[warp][it % kPruneStages] + lane * N;
            if (lane < min(32, H - j0)) {
                const float2* a2 = reinterpret_cast<const float2*>(sr);
                float m = -INFINITY;
                if (!ties) {   // the boundary at position i is the prefix maximum
#pragma unroll
                    for (int i2 = 0; i2 < N / 2; ++i2) {
                        const float2 v2 = a2[i2];
#pragma unroll
                        for (int h2 = 0; h2 < 2; ++h2) {
                            const int i = 2 * i2 + h2;
                            const float v = h2 ? v2.y : v2.x;
                            lo = fminf(lo, v);
                            m = fmaxf(m, v);
                            cnt[i] += (v == v ? 1u : 0u) + (fsub(m, v) > p.margin ? 0x10000u : 0u);
                        }
                    }
                } else {       // equal costs: the prefix maximum at the group's end
#pragma unroll
                    for (int i = 0; i < N; ++i) {
                        const float v = sr[i];
                        lo = fminf(lo, v);
                        m = fmaxf(m, v);
                        // only the real positions: the padding ones must stay NaN for the
                        // buffer's next use (cp.async refills real positions only); an
                        // all-unmeasured row would leave -inf there and fail the range check
                        if (i < nr) sr[i] = m;
                    }
                    const float* arow = A + (long long)(j0 + lane) * N;
                    float cur = -INFINITY;
#pragma unroll
                    for (int i = N - 1; i >= 0; --i) {
                        if (ends >> i & 1) cur = sr[i];
                        const int c = col_s[warp][i];
                        const float v = c >= 0 ? __ldg(arow + c) : __int_as_float(0x7fc00000);
                        cnt[i] += (v == v ? 1u : 0u) + (fsub(cur, v) > p.margin ? 0x10000u : 0u);
                    }
                }
                hi = fmaxf(hi, m);
            }
            __syncwarp();   // this buffer is refilled by the next iteration's copy
        }
        const bool ok = __all_sync(0xffffffffu, cok && lo >= 0.0f && hi <= 1.0f);
        unsigned keep = 0;   // bit = position
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const unsigned meas = __reduce_add_sync(0xffffffffu, cnt[i] & 0xFFFFu);
            const unsigned far = __reduce_add_sync(0xffffffffu, cnt[i] >> 16);
            if (i < nr && !(2ull * far > meas)) keep |= 1u << i;
        }
        const unsigned kept_cols = __ballot_sync(0xffffffffu, real && (keep >> rank & 1));
        if (lane == 0) {
            if (!ok) flag_data_error(p.st);
            p.out_keep[q] = ok ? kept_cols : 0u;
        }
    }
}

}  // namespace

int launch_uniform(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int fixed_gamma, float weight,
                   uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean, cudaStream_t s) {
    if (d.n_inst == 0) return EKYA_OK;
    UniformParams p{d, t, fixed_gamma, weight, out_alloc, out_cfg,
                    reinterpret_cast<unsigned long long*>(out_sum), out_mean, h->dstate};
    const long long need = ((long long)d.n_inst + kBaseWarps - 1) / kBaseWarps;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    uniform_kernel<<<grid, kBaseWarps * 32, 0, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

int launch_pareto(ekya_handle* h, long long n_sets, int n, const float* cost, const float* post,
                  uint32_t* out_mask, cudaStream_t s) {
    if (n_sets == 0) return EKYA_OK;
    ParetoParams p{n_sets, n, cost, post, out_mask, h->dstate};
    const long long need = (n_sets + 255) / 256;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    auto k = n <= 8 ? pareto_kernel<8> : n <= 18 ? pareto_kernel<18> : pareto_kernel<31>;
    k<<<grid, 256, 0, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

int launch_prune(ekya_handle* h, long long n_query, int H, int n, const float* cost, const float* acc, float margin,
                 uint32_t* out_keep, cudaStream_t s) {
    if (n_query == 0) return EKYA_OK;
    PruneParams p{n_query, H, n, cost, acc, margin, out_keep, h->dstate};
    const long long need = (n_query + kBaseWarps - 1) / kBaseWarps;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    if (n == 18) {
        const long long need4 = (n_query + kPruneWarps - 1) / kPruneWarps;
        prune_sorted_kernel<18><<<(int)std::min<long long>(need4, (long long)h->sm_count * 16), kPruneWarps * 32, 0, s>>>(p);
        h->launches++;
        return cuda_status(cudaGetLastError());
    }
    auto k = n <= 8 ? prune_kernel<8> : n <= 18 ? prune_kernel<18> : prune_kernel<31>;
    k<<<grid, kBaseWarps * 32, 0, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya

// ------------------------------------------------------------------------
// NEXT-2: micro-profiler curve fit (readings CF1-CF3)
// ------------------------------------------------------------------------
// One thread per (stream, config) set.  For every grid value c_i = i/8 the
// regressor x_k = 1/(k + c_i) and its sums (sum x, sum x^2, n sum x^2 - (sum x)^2)
// do not depend on the data: each CTA computes them once into shared memory, in
// the oracle's operation order, so a set costs sum x y, the 2x2 solve and the
// residual sums only.  Everything is one binary32 rounding per operation.
namespace ekya {

namespace {

constexpr int kCfGrid = 257;
constexpr int kCfMaxPoints = 32;

struct CurveParams {
    long long n_sets;
    int np;
    const float* acc;
    const int* full_epochs;
    float* out_pred;
    float* out_params;
    DevState* st;
};

// One grid point's record in shared memory: x_0..x_{n-1}, then sum x, sum x^2, det, and the
// refined reciprocals of det and sum x^2 with a flag saying whether they may be used.
__host__ __device__ constexpr int cf_rec(int n) { return (n + 6 + 3) & ~3; }

// a / den, correctly rounded: the shared-reciprocal fast path (SharedDiv) when |a| and den
// lie in [2^-60, 2^60], else the full IEEE division (zeros keep their sign there)
__device__ __forceinline__ float cf_div(float a, float den, float rden, bool den_fast) {
    const float aa = fabsf(a);
    if (den_fast && aa >= 8.67361738e-19f && aa <= 1.15292150e18f) {
        const float q0 = __fmaf_rn(a, rden, 0.0f);
        const float e = __fmaf_rn(-den, q0, a);
        return __fmaf_rn(rden, e, q0);
    }
    return fdiv(a, den);
}

// NP: compile-time point count (5 = the paper's "say, 5" epochs), or kCfMaxPoints for a
// runtime count
template <int NP>
__global__ void __launch_bounds__(256) curve_fit_kernel(CurveParams p) {
    extern __shared__ __align__(16) float cs[];
    const int n = NP == kCfMaxPoints ? p.np : NP;
    const int R = cf_rec(n);
    const float fn = __int2float_rn(n);
    for (int i = threadIdx.x; i < kCfGrid; i += blockDim.x) {
        float* rec = cs + i * R;
        const float c = fmul(__int2float_rn(i), 0.125f);
        float sx = 0.0f, sxx = 0.0f;
        for (int k = 0; k < n; ++k) {
            const float x = fdiv(1.0f, fadd(__int2float_rn(k + 1), c));
            rec[k] = x;
            sx = fadd(sx, x);
            sxx = fadd(sxx, fmul(x, x));
        }
        const float det = fsub(fmul(fn, sxx), fmul(sx, sx));
        rec[n] = sx;
        rec[n + 1] = sxx;
        rec[n + 2] = det;
        // the reciprocals as SharedDiv refines them; usable for divisors in [2^-60, 2^60]
        const float dd = det > 0.0f ? det : 1.0f;
        const SharedDiv sd(dd), sq(sxx > 0.0f ? sxx : 1.0f);
        rec[n + 3] = sd.r;
        rec[n + 4] = sq.r;
        const bool fd = det > 0.0f && fast_dividend(det) && sxx > 0.0f && fast_dividend(sxx);
        rec[n + 5] = fd ? 1.0f : 0.0f;
    }
    __syncthreads();
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < p.n_sets;
         s += (long long)gridDim.x * blockDim.x) {
        const int K = p.full_epochs[s];
        bool ok = K >= 1;
        float y[NP];
        float sy = 0.0f;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            if (NP == kCfMaxPoints && k >= n) break;
            const float a = __ldg(p.acc + s * n + k);
            ok &= in01(a);
            y[k] = fsub(1.0f, a);
            sy = fadd(sy, y[k]);
        }
        // the alpha = 0 boundary solution does not depend on c: fl(0 x) + b0 = b0 exactly
        const float m = fdiv(sy, fn);
        const float b0 = m > 0.0f ? m : 0.0f;
        float e0 = 0.0f;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            if (NP == kCfMaxPoints && k >= n) break;
            const float d = fsub(b0, y[k]);
            e0 = fadd(e0, fmul(d, d));
        }
        float best = 0.0f, bal = 0.0f, bb = 0.0f;
        int bi = 0;
        for (int i = 0; i < kCfGrid; ++i) {
            const float* rec = cs + i * R;
            float x[NP];
            float sx, sxx, det, rdet, rsxx;
            bool fd;
            if constexpr (NP == 5) {
                const float4 r0 = *reinterpret_cast<const float4*>(rec);
                const float4 r1 = *reinterpret_cast<const float4*>(rec + 4);
                const float4 r2 = *reinterpret_cast<const float4*>(rec + 8);
                x[0] = r0.x, x[1] = r0.y, x[2] = r0.z, x[3] = r0.w, x[4] = r1.x;
                sx = r1.y, sxx = r1.z, det = r1.w, rdet = r2.x, rsxx = r2.y, fd = r2.z != 0.0f;
            } else {
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    if (NP == kCfMaxPoints && k >= n) break;
                    x[k] = rec[k];
                }
                sx = rec[n], sxx = rec[n + 1], det = rec[n + 2], rdet = rec[n + 3], rsxx = rec[n + 4];
                fd = rec[n + 5] != 0.0f;
            }
            float sxy = 0.0f;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (NP == kCfMaxPoints && k >= n) break;
                sxy = fadd(sxy, fmul(x[k], y[k]));
            }
            float al = 0.0f, b = 0.0f, e = 0.0f;
            bool done = false;
            if (det > 0.0f) {
                const float a1 = cf_div(fsub(fmul(fn, sxy), fmul(sx, sy)), det, rdet, fd);
                const float b1 = cf_div(fsub(fmul(sxx, sy), fmul(sx, sxy)), det, rdet, fd);
                if (a1 >= 0.0f && b1 >= 0.0f) {
                    al = a1;
                    b = b1;
#pragma unroll
                    for (int k = 0; k < NP; ++k) {
                        if (NP == kCfMaxPoints && k >= n) break;
                        const float d = fsub(fadd(fmul(al, x[k]), b), y[k]);
                        e = fadd(e, fmul(d, d));
                    }
                    done = true;
                }
            }
            if (!done) {
                const float q = sxx > 0.0f ? cf_div(sxy, sxx, rsxx, fd) : 0.0f;
                const float a0 = q > 0.0f ? q : 0.0f;
                // b = 0 boundary: fl(a0 x) + 0 = fl(a0 x) exactly (a0 x >= +0)
                float e1 = 0.0f;
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    if (NP == kCfMaxPoints && k >= n) break;
                    const float d = fsub(fmul(a0, x[k]), y[k]);
                    e1 = fadd(e1, fmul(d, d));
                }
                if (e1 < e0) {
                    al = a0;
                    b = 0.0f;
                    e = e1;
                } else {
                    al = 0.0f;
                    b = b0;
                    e = e0;
                }
            }
            if (i == 0 || e < best) {
                best = e;
                bal = al;
                bb = b;
                bi = i;
            }
        }
        const float bc = fmul(__int2float_rn(bi), 0.125f);
        float pr = fsub(1.0f, fadd(fdiv(bal, fadd(__int2float_rn(K), bc)), bb));
        pr = pr < 0.0f ? 0.0f : (pr > 1.0f ? 1.0f : pr);
        if (!ok) flag_data_error(p.st);
        p.out_pred[s] = ok ? pr : 0.0f;
        if (p.out_params) {
            p.out_params[s * 3] = ok ? bal : 0.0f;
            p.out_params[s * 3 + 1] = ok ? bc : 0.0f;
            p.out_params[s * 3 + 2] = ok ? bb : 0.0f;
        }
    }
}

}  // namespace

int launch_curve_fit(ekya_handle* h, long long n_sets, int np, const float* acc, const int* full_epochs,
                     float* out_pred, float* out_params, cudaStream_t s) {
    if (n_sets == 0) return EKYA_OK;
    CurveParams p{n_sets, np, acc, full_epochs, out_pred, out_params, h->dstate};
    const size_t smem = (size_t)kCfGrid * cf_rec(np) * 4;
    auto k = np == 5 ? curve_fit_kernel<5> : curve_fit_kernel<kCfMaxPoints>;
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    const long long need = (n_sets + 255) / 256;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    k<<<grid, 256, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
