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
