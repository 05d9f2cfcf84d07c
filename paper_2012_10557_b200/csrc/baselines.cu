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

__global__ void __launch_bounds__(kBaseWarps * 32) uniform_kernel(UniformParams p) {
    const ekya_dims& d = p.d;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int V = d.n_streams, J = 2 * V, nG = d.n_gamma, nL = d.n_lambda, U = d.units;
    const float keep = fsub(1.0f, p.weight);
    for (long long b = (long long)blockIdx.x * kBaseWarps + warp; b < d.n_inst;
         b += (long long)gridDim.x * kBaseWarps) {
        const bool ok = warp_instance_valid(p.t, b, V, nG, nL);
        if (!ok && lane == 0) flag_data_error(p.st);
        unsigned long long S = 0;
        for (int v = lane; v < V; v += 32) {
            // U1: static split
            const int share = U / V + (v < U % V ? 1 : 0);
            const int rt = (int)floorf(fmul(__int2float_rn(share), keep));
            const int ri = share - rt;
            const long long bv = b * V + v;
            const float stale = __ldg(p.t.stale + bv);
            const float* cost = p.t.cost + bv * nG;
            const float* post = p.t.post + bv * nG;
            // U2: the fixed retraining config (1-based, 0 = none)
            int g = p.fixed_gamma;
            if (g < 0) {
                g = 0;
                float bp = 0.0f;
                for (int k = 0; k < nG; ++k) {
                    if (isinf(__ldg(cost + k))) continue;   // padding
                    const float pk = __ldg(post + k);
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
                if (g > 0 && window_acc(stale, __ldg(post + g - 1), __ldg(cost + g - 1), rt, d.unit_gpu_seconds, &w))
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
};

// one set per thread: the set's n <= 31 (cost, post) pairs in registers (NM = compile-time
// bound), the O(n^2) dominance test sequential -- far fewer instructions than a warp per set
template <int NM>
__global__ void __launch_bounds__(256) pareto_kernel(ParetoParams p) {
    const int n = p.n;
    for (long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x; s < p.n_sets;
         s += (long long)gridDim.x * blockDim.x) {
        float c[NM], q[NM];
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            c[k] = k < n ? __ldg(p.cost + s * n + k) : INFINITY;
            q[k] = k < n ? __ldg(p.post + s * n + k) : 0.0f;
        }
        unsigned m = 0;
#pragma unroll
        for (int k = 0; k < NM; ++k) {
            bool dom = isinf(c[k]);
#pragma unroll
            for (int j = 0; j < NM; ++j)
                if (j != k) dom |= !isinf(c[j]) && c[j] <= c[k] && q[j] >= q[k] && (c[j] < c[k] || q[j] > q[k]);
            m |= dom ? 0u : (1u << k);
        }
        p.out_mask[s] = m;
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
    ParetoParams p{n_sets, n, cost, post, out_mask};
    const long long need = (n_sets + 255) / 256;
    const int grid = (int)std::min<long long>(need, (long long)h->sm_count * 8);
    auto k = n <= 8 ? pareto_kernel<8> : n <= 18 ? pareto_kernel<18> : pareto_kernel<31>;
    k<<<grid, 256, 0, s>>>(p);
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
