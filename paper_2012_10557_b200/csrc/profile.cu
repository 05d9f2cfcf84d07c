// profile.cu -- ekya_profile_estimate: the class-distribution-similarity
// accuracy estimator (draft appendix).
//
// RADIUS (HBM-bound): one CTA per query (grid-stride, 2 CTAs/SM).  The query's
// history histograms and history accuracies are staged into shared memory with
// 16-byte vector loads (chunks of Hc windows when a query does not fit), one
// thread per window computes the sequential squared distance (rule 5; row
// stride C words, conflict-free for odd C) and the <= tau test, then a fixed
// thread -> gamma mapping accumulates exact Q32 sums and counts over similar,
// measured windows; partials are combined in shared memory and divided once in
// double precision (rule 5), exactly as the oracle.
//
// CLUSTER (ALU-bound): one CTA per query holds the whole history in shared
// memory and runs Lloyd's algorithm (C19): thread-per-window assignment,
// thread-per-(cluster, class) exact Q32 centroid sums, convergence by block
// vote; the query joins its nearest centroid and the same per-gamma reduction
// follows.
#include <algorithm>
#include <cfloat>

#include "launch.h"

namespace ekya {

namespace {

constexpr int kProfThreads = 256;

struct ProfParams {
    ekya_profile_dims p;
    const float* cur;
    const float* hist;
    const float* acc;
    const float* fallback;
    float* out_est;
    int* out_n;
    int* out_cluster;
    DevState* st;
    int Hc;          // windows per staged chunk (RADIUS)
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// per-gamma partial sums: thread t owns gamma t % G and window residue t / G
struct GammaAcc {
    int g, grp, ngrp;
    unsigned long long s;
    int n;
};

__device__ __forceinline__ GammaAcc gamma_acc_init(int G) {
    GammaAcc a;
    a.ngrp = kProfThreads / G;
    a.g = threadIdx.x % G;
    a.grp = threadIdx.x / G;
    a.s = 0;
    a.n = 0;
    return a;
}

// accumulate windows [0, hn) of a staged accuracy tile; returns false on bad data
__device__ __forceinline__ bool gamma_acc_add(GammaAcc& a, const float* acc_s, const unsigned char* sim,
                                              int hn, int G) {
    bool ok = true;
    if (a.grp >= a.ngrp) return ok;
    for (int h = a.grp; h < hn; h += a.ngrp) {
        float x = acc_s[(size_t)h * G + a.g];
        bool nan = isnan(x);
        ok &= nan || in01(x);
        if (sim[h] && !nan) {
            a.s += q32(x);
            a.n += 1;
        }
    }
    return ok;
}

// combine partials and write est / n for query q
__device__ __forceinline__ void gamma_acc_finish(const GammaAcc& a, unsigned long long* ps, int* pn,
                                                 const ProfParams& P, long long q, bool ok) {
    const int G = P.p.n_gamma;
    if (a.grp < a.ngrp) {
        ps[threadIdx.x] = a.s;
        pn[threadIdx.x] = a.n;
    }
    __syncthreads();
    if (threadIdx.x < G) {
        unsigned long long s = 0;
        int n = 0;
        for (int r = 0; r < a.ngrp; ++r) {
            s += ps[r * G + threadIdx.x];
            n += pn[r * G + threadIdx.x];
        }
        float est;
        if (!ok) {
            est = 0.0f;
            n = 0;
        } else {
            est = n > 0 ? mean_q32(s, n) : __ldg(P.fallback + q * G + threadIdx.x);
        }
        P.out_est[q * G + threadIdx.x] = est;
        P.out_n[q * G + threadIdx.x] = n;
    }
}

__global__ void __launch_bounds__(kProfThreads) radius_kernel(ProfParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int H = P.p.n_hist, C = P.p.n_class, G = P.p.n_gamma, Hc = P.Hc;
    const float tau = P.p.tau;
    unsigned char* hbuf = smem;
    unsigned char* abuf = hbuf + al16((size_t)Hc * C * 4 + 16);
    float* cur_s = reinterpret_cast<float*>(abuf + al16((size_t)Hc * G * 4 + 16));
    unsigned char* sim = reinterpret_cast<unsigned char*>(cur_s + ((C + 3) & ~3));
    unsigned long long* ps = reinterpret_cast<unsigned long long*>(sim + al16(Hc));
    int* pn = reinterpret_cast<int*>(ps + kProfThreads);

    for (long long q = blockIdx.x; q < P.p.n_query; q += gridDim.x) {
        bool ok = true;
        for (int c = threadIdx.x; c < C; c += blockDim.x) {
            float x = __ldg(P.cur + q * C + c);
            ok &= in01(x);
            cur_s[c] = x;
        }
        GammaAcc a = gamma_acc_init(G);
        for (int h0 = 0; h0 < H; h0 += Hc) {
            const int hn = min(Hc, H - h0);
            const float* hs = reinterpret_cast<const float*>(
                stage_to_smem(hbuf, P.hist + ((size_t)q * H + h0) * C, (size_t)hn * C * 4));
            const float* as = reinterpret_cast<const float*>(
                stage_to_smem(abuf, P.acc + ((size_t)q * H + h0) * G, (size_t)hn * G * 4));
            __syncthreads();
            for (int h = threadIdx.x; h < hn; h += blockDim.x) {
                const float* row = hs + (size_t)h * C;
                float d2 = 0.0f;
                for (int c = 0; c < C; ++c) {
                    float x = row[c];
                    ok &= in01(x);
                    float diff = fsub(cur_s[c], x);
                    d2 = fadd(d2, fmul(diff, diff));
                }
                sim[h] = __fsqrt_rn(d2) <= tau;
            }
            __syncthreads();
            ok &= gamma_acc_add(a, as, sim, hn, G);
            __syncthreads();
        }
        ok = __syncthreads_and(ok) != 0;
        if (!ok && threadIdx.x == 0) flag_data_error(P.st);
        gamma_acc_finish(a, ps, pn, P, q, ok);
        __syncthreads();
    }
}

__device__ __forceinline__ float dist2(const float* x, const float* m, int C) {
    float s = 0.0f;
    for (int c = 0; c < C; ++c) {
        float diff = fsub(x[c], m[c]);
        s = fadd(s, fmul(diff, diff));
    }
    return s;
}

__device__ __forceinline__ int nearest(const float* x, const float* mu, int k, int C) {
    int best = 0;
    float bd = dist2(x, mu, C);
    for (int i = 1; i < k; ++i) {
        float di = dist2(x, mu + (size_t)i * C, C);
        if (di < bd) {
            bd = di;
            best = i;
        }
    }
    return best;
}

struct ClusterLayout {
    size_t hist, acc, cur, mu, assign, sim, ps, pn, total;
};

__host__ __device__ inline ClusterLayout cluster_layout(int H, int C, int G, int K) {
    ClusterLayout L;
    size_t o = 0;
    L.hist = o;   o += al16((size_t)H * C * 4 + 16);
    L.acc = o;    o += al16((size_t)H * G * 4 + 16);
    L.cur = o;    o += al16((size_t)C * 4);
    L.mu = o;     o += al16((size_t)K * C * 4);
    L.assign = o; o += al16((size_t)(H + 1) * 4);
    L.sim = o;    o += al16((size_t)H + 1);
    L.ps = o;     o += al16((size_t)kProfThreads * 8);
    L.pn = o;     o += al16((size_t)kProfThreads * 4);
    L.total = o;
    return L;
}

__global__ void __launch_bounds__(kProfThreads) cluster_kernel(ProfParams P) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int H = P.p.n_hist, C = P.p.n_class, G = P.p.n_gamma, K = P.p.k;
    ClusterLayout Lc = cluster_layout(H, C, G, K);
    unsigned char* hbuf = smem + Lc.hist;
    unsigned char* abuf = smem + Lc.acc;
    float* cur_s = reinterpret_cast<float*>(smem + Lc.cur);
    float* mu = reinterpret_cast<float*>(smem + Lc.mu);
    int* assign = reinterpret_cast<int*>(smem + Lc.assign);
    unsigned char* sim = smem + Lc.sim;
    unsigned long long* ps = reinterpret_cast<unsigned long long*>(smem + Lc.ps);
    int* pn = reinterpret_cast<int*>(smem + Lc.pn);
    __shared__ int s_qc;

    for (long long q = blockIdx.x; q < P.p.n_query; q += gridDim.x) {
        bool ok = true;
        for (int c = threadIdx.x; c < C; c += blockDim.x) {
            float x = __ldg(P.cur + q * C + c);
            ok &= in01(x);
            cur_s[c] = x;
        }
        const float* hs = reinterpret_cast<const float*>(
            stage_to_smem(hbuf, P.hist + (size_t)q * H * C, (size_t)H * C * 4));
        const float* as = reinterpret_cast<const float*>(
            stage_to_smem(abuf, P.acc + (size_t)q * H * G, (size_t)H * G * 4));
        __syncthreads();
        for (int i = threadIdx.x; i < H * C; i += blockDim.x) ok &= in01(hs[i]);
        if (H > 0) {
            for (int i = threadIdx.x; i < K * C; i += blockDim.x) {
                int ci = i / C, c = i - ci * C;
                mu[i] = hs[(size_t)((long long)ci * H / K) * C + c];
            }
            __syncthreads();
            for (int h = threadIdx.x; h < H; h += blockDim.x) assign[h] = nearest(hs + (size_t)h * C, mu, K, C);
            __syncthreads();
            for (int it = 0; it < P.p.max_iter; ++it) {
                for (int i = threadIdx.x; i < K * C; i += blockDim.x) {
                    int ci = i / C, c = i - ci * C;
                    unsigned long long s = 0;
                    int n = 0;
                    for (int h = 0; h < H; ++h) {
                        if (assign[h] == ci) {
                            s += q32(hs[(size_t)h * C + c]);
                            ++n;
                        }
                    }
                    if (n > 0) mu[i] = mean_q32(s, n);   // empty cluster keeps its centroid
                }
                __syncthreads();
                // reassign; writing in place is equivalent to the oracle's
                // "if unchanged stop, else assign = new" (both leave assign = new)
                int changed = 0;
                for (int h = threadIdx.x; h < H; h += blockDim.x) {
                    int x = nearest(hs + (size_t)h * C, mu, K, C);
                    changed |= x != assign[h];
                    assign[h] = x;
                }
                if (!__syncthreads_or(changed)) break;
            }
            if (threadIdx.x == 0) s_qc = nearest(cur_s, mu, K, C);
        } else if (threadIdx.x == 0) {
            s_qc = -1;
        }
        __syncthreads();
        const int qc = s_qc;
        for (int h = threadIdx.x; h < H; h += blockDim.x) sim[h] = assign[h] == qc;
        __syncthreads();
        GammaAcc a = gamma_acc_init(G);
        ok &= gamma_acc_add(a, as, sim, H, G);
        ok = __syncthreads_and(ok) != 0;
        if (!ok && threadIdx.x == 0) flag_data_error(P.st);
        if (P.out_cluster) {
            int* oc = P.out_cluster + q * (H + 1);
            for (int h = threadIdx.x; h < H; h += blockDim.x) oc[h] = ok ? assign[h] : 0;
            if (threadIdx.x == 0) oc[H] = ok ? qc : 0;
        }
        gamma_acc_finish(a, ps, pn, P, q, ok);
        __syncthreads();
    }
}

int resident(ekya_handle* h, const void* fn, size_t smem, long long work) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kProfThreads, smem);
    per_sm = std::max(per_sm, 1);
    long long g = (long long)h->sm_count * per_sm;
    return (int)std::max(1LL, std::min(g, work));
}

}  // namespace

int launch_profile(ekya_handle* h, const ekya_profile_dims& p, const float* cur, const float* hist,
                   const float* hist_acc, const float* fallback, float* out_est, int32_t* out_n,
                   int32_t* out_cluster, cudaStream_t s) {
    ProfParams P{};
    P.p = p;
    P.cur = cur;
    P.hist = hist;
    P.acc = hist_acc;
    P.fallback = fallback;
    P.out_est = out_est;
    P.out_n = out_n;
    P.out_cluster = out_cluster;
    P.st = h->dstate;
    const int C = p.n_class, G = p.n_gamma, H = p.n_hist, K = p.k;
    const size_t fixed = al16((size_t)C * 4 + 16) + al16((size_t)kProfThreads * 8) +
                         al16((size_t)kProfThreads * 4) + 256;
    if (p.n_query == 0) return EKYA_OK;
    if (p.mode == EKYA_PROFILE_RADIUS) {
        // two CTAs per SM: budget ~110 KB each
        const size_t per_window = (size_t)(C + G) * 4 + 1;
        size_t budget = std::min<size_t>(110 * 1024, h->smem_optin);
        long long hc = (long long)((budget - fixed - 64) / per_window);
        if (hc < 1) return EKYA_ERR_SHAPE;
        P.Hc = (int)std::max(1LL, std::min<long long>(hc, std::max(H, 1)));
        size_t smem = al16((size_t)P.Hc * C * 4 + 16) + al16((size_t)P.Hc * G * 4 + 16) +
                      al16((size_t)((C + 3) & ~3) * 4) + al16(P.Hc) + fixed;
        cudaError_t e = cudaFuncSetAttribute(radius_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return EKYA_ERR_CUDA;
        int grid = resident(h, (const void*)radius_kernel, smem, p.n_query);
        radius_kernel<<<grid, kProfThreads, smem, s>>>(P);
    } else {
        size_t smem = cluster_layout(H, C, G, K).total;
        if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
        cudaError_t e = cudaFuncSetAttribute(cluster_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return EKYA_ERR_CUDA;
        int grid = resident(h, (const void*)cluster_kernel, smem, p.n_query);
        cluster_kernel<<<grid, kProfThreads, smem, s>>>(P);
    }
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
