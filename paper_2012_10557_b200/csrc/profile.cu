// profile.cu -- ekya_profile_estimate: the class-distribution-similarity
// accuracy estimator (draft appendix).
//
// RADIUS and the general CLUSTER kernel run one persistent CTA (512 threads)
// per SM that walks its queries through a two-stage shared-memory pipeline fed
// by the TMA bulk-copy
// engine (cp.async.bulk + mbarrier): while the CTA computes query j, the
// history histograms / accuracies of query j+1 are in flight, so HBM streams
// continuously and no thread stalls on a global load.
//
// RADIUS (HBM-bound): one thread per history window computes rule 5's
// sequential squared distance from shared memory (row stride C words: bank-
// conflict free for odd C) and the <= tau test; a fixed thread -> gamma mapping
// then accumulates exact Q32 sums and counts over similar, measured windows;
// the partials are combined once per query and divided in double (rule 5).
// Queries whose history does not fit a stage are processed in window chunks.
//
// CLUSTER (ALU-bound): Lloyd's algorithm (C19) per query on the staged
// history.  The bench shape (H <= 512, C <= 32, k <= 8) runs cluster2_kernel:
// four 256-thread CTAs per SM, one query each, packed f32x2 distances with a
// changed-centroid register cache and exact cluster sums in shared 32-bit
// counter pairs (see the comment above the kernel).  Other shapes run
// cluster_kernel: one 512-thread CTA per SM, window rows in registers or shared
// memory, per-warp exact partial sums.  Both maintain the sums INCREMENTALLY
// (only windows whose assignment changed are moved), which is bit-identical to
// the oracle's full recomputation because integer addition is associative.
#include <algorithm>
#include <cfloat>
#include <cstring>

#include "launch.h"

namespace ekya {

namespace {

constexpr int kProfThreads = 512;
constexpr int kRadiusStages = 2;

struct ProfParams {
    ekya_profile_dims p;
    float* rad_est;     // fused RADIUS outputs (cluster2_kernel<5, 27> only; NULL = CLUSTER alone)
    int* rad_n;
    float rad_tau;
    const float* cur;
    const float* hist;
    const float* acc;
    const float* fallback;
    float* out_est;
    int* out_n;
    int* out_cluster;
    DevState* st;
    int Hc;             // windows per staged chunk
    int stages;         // 1 or 2
    int acc_staged;     // CLUSTER: accuracy tile staged in shared memory
    size_t stage_bytes; // bytes per stage
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// per-stage layout: [cur][fallback][hist chunk][acc chunk], each padded by 16 B for granule staging
struct StageLayout {
    size_t cur, fb, hist, acc, total;
};
__host__ __device__ inline StageLayout stage_layout(int C, int G, int Hc, bool with_acc) {
    StageLayout L;
    size_t o = 0;
    L.cur = o;  o += al16((size_t)C * 4) + 16;
    L.fb = o;   o += al16((size_t)G * 4) + 16;
    L.hist = o; o += al16((size_t)Hc * C * 4) + 16;
    L.acc = o;  o += with_acc ? al16((size_t)Hc * G * 4) + 16 : 0;
    L.total = al16(o);
    return L;
}

struct StagePtrs {
    const float* cur;
    const float* fb;
    const float* hist;
    const float* acc;
};

// Leader thread: arm the stage barrier and issue the bulk copies of one work item.
__device__ __forceinline__ void issue_item(const ProfParams& P, unsigned char* stage, unsigned long long* bar,
                                           long long q, int h0, int hn, bool with_acc, const StageLayout& L) {
    const int H = P.p.n_hist, C = P.p.n_class, G = P.p.n_gamma;
    Granules gc = granules(P.cur + q * C, (size_t)C * 4);
    Granules gf = granules(P.fallback + q * G, (size_t)G * 4);
    Granules gh = granules(P.hist + ((size_t)q * H + h0) * C, (size_t)hn * C * 4);
    Granules ga = with_acc ? granules(P.acc + ((size_t)q * H + h0) * G, (size_t)hn * G * 4) : Granules{nullptr, 0, 0};
    mbar_arrive_expect_tx(bar, gc.bytes + gf.bytes + gh.bytes + ga.bytes);
    bulk_g2s(stage + L.cur, gc.g0, gc.bytes, bar);
    bulk_g2s(stage + L.fb, gf.g0, gf.bytes, bar);
    if (gh.bytes) bulk_g2s(stage + L.hist, gh.g0, gh.bytes, bar);
    if (ga.bytes) bulk_g2s(stage + L.acc, ga.g0, ga.bytes, bar);
}

__device__ __forceinline__ StagePtrs stage_ptrs(const ProfParams& P, unsigned char* stage, long long q, int h0,
                                                bool with_acc, const StageLayout& L) {
    const int H = P.p.n_hist, C = P.p.n_class, G = P.p.n_gamma;
    StagePtrs s;
    s.cur = reinterpret_cast<const float*>(stage + L.cur + granules(P.cur + q * C, 4).off);
    s.fb = reinterpret_cast<const float*>(stage + L.fb + granules(P.fallback + q * G, 4).off);
    s.hist = reinterpret_cast<const float*>(stage + L.hist + granules(P.hist + ((size_t)q * H + h0) * C, 4).off);
    s.acc = with_acc ? reinterpret_cast<const float*>(stage + L.acc +
                                                      granules(P.acc + ((size_t)q * H + h0) * G, 4).off)
                     : nullptr;
    return s;
}

// ---- per-gamma exact accumulation: thread t owns gamma t % G and windows h = t / G (mod ngrp)
struct GammaAcc {
    int g, grp, ngrp;
    unsigned long long s;
    int n;
};

__device__ __forceinline__ void gacc_reset(GammaAcc& a, int G) {
    a.ngrp = kProfThreads / G;
    a.g = threadIdx.x % G;
    a.grp = threadIdx.x / G;
    a.s = 0;
    a.n = 0;
}

// windows [0, hn) of an accuracy tile (shared or global), similarity flags in sim[]
__device__ __forceinline__ bool gacc_add(GammaAcc& a, const float* acc, const unsigned char* sim, int hn, int G) {
    bool ok = true;
    if (a.grp >= a.ngrp) return ok;
    for (int h = a.grp; h < hn; h += a.ngrp) {
        float x = acc[(size_t)h * G + a.g];
        bool nan = isnan(x);
        ok &= nan || in01(x);
        if (sim[h] && !nan) {
            a.s += q32(x);
            a.n += 1;
        }
    }
    return ok;
}

__device__ __forceinline__ void gacc_finish(const GammaAcc& a, unsigned long long* ps, int* pn, const float* fb,
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
        float est = 0.0f;
        if (!ok) n = 0;
        else est = n > 0 ? mean_q32(s, n) : fb[threadIdx.x];
        P.out_est[q * G + threadIdx.x] = est;
        P.out_n[q * G + threadIdx.x] = n;
    }
}

struct ScratchLayout {
    size_t bars, sim, ps, pn, mu, sums, cnt, assign, chg, dcache, misc, total;
};
__host__ __device__ inline ScratchLayout scratch_layout(int H, int Hc, int C, int K, bool cluster) {
    ScratchLayout L;
    const int CP = (C + 3) & ~3;
    size_t o = 0;
    L.bars = o;   o += 64;
    L.sim = o;    o += al16(cluster ? (size_t)H + 1 : 2 * (size_t)Hc + 2);   // CLUSTER: flags; RADIUS: u16 list
    L.ps = o;     o += al16((size_t)kProfThreads * 8);
    L.pn = o;     o += al16((size_t)kProfThreads * 4);
    L.mu = o;     o += cluster ? al16((size_t)K * CP * 4) : 0;
    L.sums = o;   o += cluster ? al16((size_t)(kProfThreads / 32) * K * C * 8) : 0;
    L.cnt = o;    o += cluster ? al16((size_t)(kProfThreads / 32) * K * 4) : 0;
    L.assign = o; o += cluster ? al16((size_t)H * 4) : 0;
    L.chg = o;
    L.dcache = o; o += cluster ? (size_t)8 * kProfThreads * 4 : 0;
    L.misc = o;   o += 64;
    L.total = o;
    return L;
}

// ------------------------------------------------------------------------
// RADIUS
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(kProfThreads, 1) radius_kernel(ProfParams P) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int H = P.p.n_hist, C = P.p.n_class, G = P.p.n_gamma, Hc = P.Hc, NS = P.stages;
    const float tau = P.p.tau;
    const StageLayout L = stage_layout(C, G, Hc, true);
    const ScratchLayout S = scratch_layout(H, Hc, C, 0, false);
    unsigned char* scratch = smem + NS * P.stage_bytes;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(scratch + S.bars);
    unsigned char* sim = scratch + S.sim;
    unsigned long long* ps = reinterpret_cast<unsigned long long*>(scratch + S.ps);
    int* pn = reinterpret_cast<int*>(scratch + S.pn);

    const long long Q = P.p.n_query;
    const int nch = (H + Hc - 1) / Hc;
    const long long nq_local = Q > blockIdx.x ? (Q - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long items = nq_local * nch;
    auto item_q = [&](long long i) { return (long long)blockIdx.x + (i / nch) * gridDim.x; };
    auto item_h0 = [&](long long i) { return (int)(i % nch) * Hc; };

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (long long i = 0; i < NS && i < items; ++i) {
            int h0 = item_h0(i);
            issue_item(P, smem + (i % NS) * P.stage_bytes, &bar[i % NS], item_q(i), h0, min(Hc, H - h0), true, L);
        }
    }
    // similar windows of the current chunk, compacted (any order: the sums are exact integers)
    uint16_t* list = reinterpret_cast<uint16_t*>(sim);
    int* nsim = reinterpret_cast<int*>(scratch + S.misc);   // [2] counters, by chunk parity
    if (threadIdx.x < 2) nsim[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    GammaAcc a;
    bool ok = true;
    for (long long i = 0; i < items; ++i) {
        const int s = (int)(i % NS);
        const long long q = item_q(i);
        const int h0 = item_h0(i), hn = min(Hc, H - h0);
        int* cnt = nsim + (i & 1);
        if (threadIdx.x == 0) nsim[(i + 1) & 1] = 0;   // last used by chunk i - 1 (ended by a barrier)
        mbar_wait(&bar[s], (unsigned)((i / NS) & 1));
        const StagePtrs sp = stage_ptrs(P, smem + s * P.stage_bytes, q, h0, true, L);
        if (h0 == 0) {
            gacc_reset(a, G);
            ok = true;
            for (int c = threadIdx.x; c < C; c += blockDim.x) ok &= in01(sp.cur[c]);
        }
        // rule 5 distance per window; range check folded into a running min / max (a NaN
        // element makes d2 NaN, caught below); similar windows appended to the list
        for (int hw = warp * 32; hw < hn; hw += blockDim.x) {
            const int h = hw + lane;
            bool in = false;
            if (h < hn) {
                const float* row = sp.hist + (size_t)h * C;
                float d2 = 0.0f, lo = 1.0f, hi = 0.0f;
                for (int c = 0; c < C; ++c) {
                    const float x = row[c];
                    lo = fminf(lo, x);
                    hi = fmaxf(hi, x);
                    const float diff = fsub(sp.cur[c], x);
                    d2 = fadd(d2, fmul(diff, diff));
                }
                ok &= lo >= 0.0f && hi <= 1.0f && d2 == d2;
                in = __fsqrt_rn(d2) <= tau;
            }
            const unsigned m = __ballot_sync(0xffffffffu, in);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(cnt, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (in) list[base + __popc(m & ((1u << lane) - 1u))] = (uint16_t)h;
        }
        // the accuracy tile: NaN (unmeasured) or in [0, 1] (fminf / fmaxf ignore NaN)
        {
            float lo = 1.0f, hi = 0.0f;
            const int n = hn * G;
            if ((reinterpret_cast<uintptr_t>(sp.acc) & 15) == 0) {
                const float4* a4 = reinterpret_cast<const float4*>(sp.acc);
                for (int t = threadIdx.x; t < n / 4; t += blockDim.x) {
                    const float4 x = a4[t];
                    lo = fminf(fminf(lo, x.x), fminf(x.y, fminf(x.z, x.w)));
                    hi = fmaxf(fmaxf(hi, x.x), fmaxf(x.y, fmaxf(x.z, x.w)));
                }
                for (int t = (n & ~3) + threadIdx.x; t < n; t += blockDim.x) {
                    lo = fminf(lo, sp.acc[t]);
                    hi = fmaxf(hi, sp.acc[t]);
                }
            } else {
                for (int t = threadIdx.x; t < n; t += blockDim.x) {
                    lo = fminf(lo, sp.acc[t]);
                    hi = fmaxf(hi, sp.acc[t]);
                }
            }
            ok &= lo >= 0.0f && hi <= 1.0f;
        }
        __syncthreads();
        // exact per-gamma sums over the similar, measured windows
        if (a.grp < a.ngrp) {
            const int ns = *cnt;
            for (int e = a.grp; e < ns; e += a.ngrp) {
                const float x = sp.acc[(size_t)list[e] * G + a.g];
                if (x == x) {
                    a.s += q32(x);
                    a.n += 1;
                }
            }
        }
        const bool last = h0 + hn >= H;
        if (last) {
            ok = __syncthreads_and(ok) != 0;
            if (!ok && threadIdx.x == 0) flag_data_error(P.st);
            gacc_finish(a, ps, pn, sp.fb, P, q, ok);
        }
        __syncthreads();   // stage s and the list are free again
        if (threadIdx.x == 0 && i + NS < items) {
            int h1 = item_h0(i + NS);
            issue_item(P, smem + s * P.stage_bytes, &bar[s], item_q(i + NS), h1, min(Hc, H - h1), true, L);
        }
    }
}

// ------------------------------------------------------------------------
// CLUSTER
// ------------------------------------------------------------------------
// Nearest centroid of x (registers, zero-padded to 32 classes) among K
// centroid rows of CP floats (zero-padded, 16-B aligned): four centroids are
// processed together for ILP; the padded terms are fl(0 - 0)^2 = +0 and
// s + 0 = s exactly, so each distance equals rule 5's sequential sum over the C
// real classes.  Lowest index wins ties (C19).
__device__ __forceinline__ int nearest_reg(const float (&x)[32], const float* mu, int K, int CP) {
    int best = 0;
    float bd = 0.0f;
    for (int i0 = 0; i0 < K; i0 += 4) {
        float s[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
        for (int c4 = 0; c4 < 8; ++c4) {
            if (c4 * 4 < CP) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (i0 + k < K) {
                        const float4 m = *reinterpret_cast<const float4*>(mu + (i0 + k) * CP + c4 * 4);
                        float d0 = fsub(x[c4 * 4 + 0], m.x);
                        s[k] = fadd(s[k], fmul(d0, d0));
                        float d1 = fsub(x[c4 * 4 + 1], m.y);
                        s[k] = fadd(s[k], fmul(d1, d1));
                        float d2 = fsub(x[c4 * 4 + 2], m.z);
                        s[k] = fadd(s[k], fmul(d2, d2));
                        float d3 = fsub(x[c4 * 4 + 3], m.w);
                        s[k] = fadd(s[k], fmul(d3, d3));
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (i0 + k < K && (i0 + k == 0 || s[k] < bd)) {
                bd = s[k];
                best = i0 + k;
            }
        }
    }
    return best;
}

// Squared distances of x (registers, zero padded) to N <= 8 centroid rows, all N
// chains interleaved for ILP; padded classes contribute fl(0-0)^2 = +0 (exact).
template <int N>
__device__ __forceinline__ void dist_n(const float (&x)[32], const float* mu, const int (&id)[8], int CP,
                                       float (&s)[8]) {
    const float4* rp[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
        s[k] = 0.0f;
        rp[k] = reinterpret_cast<const float4*>(mu + id[k] * CP);
    }
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
        if (c4 * 4 < CP) {
#pragma unroll
            for (int k = 0; k < N; ++k) {
                const float4 m = rp[k][c4];
                const float d0 = fsub(x[c4 * 4 + 0], m.x);
                s[k] = fadd(s[k], fmul(d0, d0));
                const float d1 = fsub(x[c4 * 4 + 1], m.y);
                s[k] = fadd(s[k], fmul(d1, d1));
                const float d2 = fsub(x[c4 * 4 + 2], m.z);
                s[k] = fadd(s[k], fmul(d2, d2));
                const float d3 = fsub(x[c4 * 4 + 3], m.w);
                s[k] = fadd(s[k], fmul(d3, d3));
            }
        }
    }
}

// Nearest of K <= 8 centroids with a per-thread distance cache: only the
// centroids in `chg` (those whose coordinates changed bitwise since the cache
// was filled) are recomputed -- an unchanged centroid has bit-identical
// distances -- all of them in one interleaved pass.  Lowest index wins ties (C19).
__device__ __forceinline__ int nearest_cached(const float (&x)[32], const float* mu, int K, int CP, unsigned chg,
                                           float* dcs /* this thread's cache, stride kProfThreads */) {
    // changed centroids in groups of <= 4 interleaved chains (5..8 split evenly);
    unsigned m = chg;   // block-uniform: no divergence
    while (m) {
        const int left = __popc(m);
        const int n = left <= 4 ? left : (left + 1) / 2;
        int id[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) id[k] = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (k < n) {
                id[k] = __ffs(m) - 1;
                m &= m - 1;
            }
        }
        float s[8];
        switch (n) {
            case 1: dist_n<1>(x, mu, id, CP, s); break;
            case 2: dist_n<2>(x, mu, id, CP, s); break;
            case 3: dist_n<3>(x, mu, id, CP, s); break;
            default: dist_n<4>(x, mu, id, CP, s); break;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (k < n) dcs[id[k] * kProfThreads] = s[k];
    }
    int best = 0;
    float bd = dcs[0];
    for (int j = 1; j < K; ++j) {
        const float dj = dcs[j * kProfThreads];
        if (dj < bd) {
            bd = dj;
            best = j;
        }
    }
    return best;
}

__device__ __forceinline__ float dist2_mem(const float* x, const float* m, int C) {
    float s = 0.0f;
    for (int c = 0; c < C; ++c) {
        float d = fsub(x[c], m[c]);
        s = fadd(s, fmul(d, d));
    }
    return s;
}

template <bool REG>
__device__ __forceinline__ int nearest_c(const float (&xr)[32], const float* xm, const float* mu, int K, int C,
                                         int CP) {
    if (REG) return nearest_reg(xr, mu, K, CP);
    int best = 0;
    float bd = 0.0f;
    for (int i = 0; i < K; ++i) {
        float d = dist2_mem(xm, mu + i * CP, C);
        if (i == 0 || d < bd) {   // lowest index on ties (C19)
            bd = d;
            best = i;
        }
    }
    return best;
}

template <bool REG>
__global__ void __launch_bounds__(kProfThreads, 1) cluster_kernel(ProfParams P) {
    // REG && k <= 8: per-thread distance cache, recompute only changed centroids
    extern __shared__ __align__(128) unsigned char smem[];
    const int H = P.p.n_hist, C = P.p.n_class, G = P.p.n_gamma, K = P.p.k, NS = P.stages;
    const int CP = (C + 3) & ~3;
    const bool accs = P.acc_staged != 0;
    const StageLayout L = stage_layout(C, G, H, accs);
    const ScratchLayout S = scratch_layout(H, H, C, K, true);
    unsigned char* scratch = smem + NS * P.stage_bytes;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(scratch + S.bars);
    unsigned char* sim = scratch + S.sim;
    unsigned long long* ps = reinterpret_cast<unsigned long long*>(scratch + S.ps);
    int* pn = reinterpret_cast<int*>(scratch + S.pn);
    float* mu = reinterpret_cast<float*>(scratch + S.mu);
    // per-warp exact partial cluster sums: part[w][i][c] = sum of Q32(h_c) over the
    // windows owned by warp w that sit in cluster i (lane c owns column c, so no atomics)
    unsigned long long* part = reinterpret_cast<unsigned long long*>(scratch + S.sums);
    int* pcnt = reinterpret_cast<int*>(scratch + S.cnt);
    int* assign = reinterpret_cast<int*>(scratch + S.assign);
    int* misc = reinterpret_cast<int*>(scratch + S.misc);   // [2] query cluster, [3..4] changed-centroid masks
    const bool cache = REG && K <= 8;
    float* dcache = reinterpret_cast<float*>(scratch + S.dcache);   // [8][kProfThreads] distance cache

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = kProfThreads / 32;
    const long long Q = P.p.n_query;
    const long long items = Q > blockIdx.x ? (Q - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    unsigned long long* mypart = part + (size_t)warp * K * C;
    int* mycnt = pcnt + warp * K;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (long long i = 0; i < NS && i < items; ++i)
            issue_item(P, smem + (i % NS) * P.stage_bytes, &bar[i % NS], blockIdx.x + i * gridDim.x, 0, H, accs, L);

    // move window h (owned by this warp) from cluster oa to na in the warp's partials
    auto move = [&](int h, int oa, int na, const float* hs) {
        for (int c = lane; c < C; c += 32) {
            const unsigned long long v = q32(hs[(size_t)h * C + c]);
            if (oa >= 0) mypart[oa * C + c] -= v;
            mypart[na * C + c] += v;
        }
        if (lane == 0) {
            if (oa >= 0) mycnt[oa] -= 1;
            mycnt[na] += 1;
        }
    };

    for (long long i = 0; i < items; ++i) {
        const int s = (int)(i % NS);
        const long long q = blockIdx.x + i * gridDim.x;
        mbar_wait(&bar[s], (unsigned)((i / NS) & 1));
        const StagePtrs sp = stage_ptrs(P, smem + s * P.stage_bytes, q, 0, accs, L);
        const float* hs = sp.hist;
        bool ok = true;
        for (int c = threadIdx.x; c < C; c += blockDim.x) ok &= in01(sp.cur[c]);
        int qc = -1;
        if (H > 0) {
            // own window's histogram in registers (REG: H <= threads, C <= 32), zero padded
            float xr[32];
            float* dc = dcache + threadIdx.x;
            if (REG) {
                const int h = threadIdx.x;
#pragma unroll
                for (int c = 0; c < 32; ++c) {
                    float x = 0.0f;
                    if (h < H && c < C) {
                        x = hs[(size_t)h * C + c];
                        ok &= in01(x);
                    }
                    xr[c] = x;
                }
            } else {
                for (int t = threadIdx.x; t < H * C; t += blockDim.x) ok &= in01(hs[t]);
            }
            for (int t = threadIdx.x; t < K * CP; t += blockDim.x) {
                const int ci = t / CP, c = t - ci * CP;
                mu[t] = c < C ? hs[(size_t)(((long long)ci * H) / K) * C + c] : 0.0f;
            }
            for (int t = lane; t < K * C; t += 32) mypart[t] = 0ULL;
            for (int t = lane; t < K; t += 32) mycnt[t] = 0;
            if (threadIdx.x == 0) misc[3] = misc[4] = 0;
            __syncthreads();
            const unsigned all_k = K >= 32 ? 0xffffffffu : ((1u << K) - 1u);
            // Lloyd passes (C19, R-CL): pass 0 assigns from the initial centroids and
            // accumulates the exact sums; pass p >= 1 follows the centroid update of
            // iteration p-1 and moves only the windows whose cluster changed.  One
            // call site for the distance code (I-cache).
            unsigned chg = all_k;
            int passes = 0;
            for (;;) {
                int changed = 0;
                for (int h0 = warp * 32; h0 < H; h0 += kProfThreads) {
                    const int h = h0 + lane;
                    int oa = -1, na = 0;
                    if (h < H) {
                        na = cache ? nearest_cached(xr, mu, K, CP, chg, dc)
                                   : nearest_c<REG>(xr, hs + (size_t)h * C, mu, K, C, CP);
                        if (passes > 0) oa = assign[h];
                        assign[h] = na;
                    }
                    if (passes == 0) {
                        // counts by ballot, sums by one row per window (lanes over classes)
                        const int nh = min(32, H - h0);
                        for (int ci = 0; ci < K; ++ci) {
                            const unsigned bm = __ballot_sync(0xffffffffu, h < H && na == ci);
                            if (lane == 0) mycnt[ci] += __popc(bm);
                        }
                        for (int j = 0; j < nh; ++j) {
                            const int aj = __shfl_sync(0xffffffffu, na, j);
                            const float* row = hs + (size_t)(h0 + j) * C;
                            unsigned long long* dst = mypart + aj * C;
                            for (int c = lane; c < C; c += 32) dst[c] += q32(row[c]);
                        }
                    } else {
                        unsigned m = __ballot_sync(0xffffffffu, h < H && na != oa);
                        changed |= m != 0;
                        while (m) {
                            const int j = __ffs(m) - 1;
                            m &= m - 1;
                            move(h0 + j, __shfl_sync(0xffffffffu, oa, j), __shfl_sync(0xffffffffu, na, j), hs);
                        }
                    }
                }
                const int any = __syncthreads_or(changed);
                const int it = passes;   // iteration whose centroid update comes next
                ++passes;
                if ((it > 0 && !any) || it >= P.p.max_iter) break;
                // centroid update from the exact sums (empty cluster keeps its centroid)
                for (int t = threadIdx.x; t < K * C; t += blockDim.x) {
                    const int ci = t / C, c = t - ci * C;
                    unsigned long long sum = 0;
                    int n = 0;
                    for (int w = 0; w < nwarps; ++w) {
                        sum += part[((size_t)w * K + ci) * C + c];
                        n += pcnt[w * K + ci];
                    }
                    if (n > 0) {
                        const float nm = mean_q32(sum, n);
                        if (__float_as_uint(nm) != __float_as_uint(mu[ci * CP + c])) {
                            mu[ci * CP + c] = nm;
                            atomicOr(reinterpret_cast<unsigned*>(&misc[3 + (it & 1)]), 1u << ci);
                        }
                    }
                }
                __syncthreads();
                chg = (unsigned)misc[3 + (it & 1)];
                if (threadIdx.x == 0) misc[3 + ((it + 1) & 1)] = 0;
            }
            if (threadIdx.x == 0) atomicAdd(&P.st->lloyd_passes, (unsigned long long)passes);
            // the query joins its nearest centroid: lane i computes distance to centroid i
            if (warp == 0) {
                unsigned long long key = ~0ULL;
                for (int ci = lane; ci < K; ci += 32) {
                    const float d = dist2_mem(sp.cur, mu + ci * CP, C);
                    const unsigned long long k = ((unsigned long long)__float_as_uint(d) << 8) | (unsigned)ci;
                    key = k < key ? k : key;
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
                    key = y < key ? y : key;
                }
                if (lane == 0) misc[2] = (int)(key & 0xFF);
            }
            __syncthreads();
            qc = misc[2];
        }
        for (int h = threadIdx.x; h < H; h += blockDim.x) sim[h] = assign[h] == qc;
        __syncthreads();
        GammaAcc a;
        gacc_reset(a, G);
        ok &= gacc_add(a, accs ? sp.acc : P.acc + (size_t)q * H * G, sim, H, G);
        ok = __syncthreads_and(ok) != 0;
        if (!ok && threadIdx.x == 0) flag_data_error(P.st);
        if (P.out_cluster) {
            int* oc = P.out_cluster + q * (H + 1);
            for (int h = threadIdx.x; h < H; h += blockDim.x) oc[h] = ok ? assign[h] : 0;
            if (threadIdx.x == 0) oc[H] = ok ? qc : 0;
        }
        gacc_finish(a, ps, pn, sp.fb, P, q, ok);
        __syncthreads();   // stage s free
        if (threadIdx.x == 0 && i + NS < items)
            issue_item(P, smem + s * P.stage_bytes, &bar[s], blockIdx.x + (i + NS) * gridDim.x, 0, H, accs, L);
    }
}

// ------------------------------------------------------------------------
// CLUSTER, several queries per SM (the shape of BASELINE config 3)
// ------------------------------------------------------------------------
// Lloyd's algorithm is a chain of short block-wide phases per pass (distances,
// moves, barrier, centroid update, barrier); with one query per SM the SM idles
// in every serial phase.  Here a 256-thread CTA owns one query at a time and
// kC2Ctas CTAs share each SM, so one query's serial phases overlap the others'
// distance work.  Each thread owns two windows (h = t and t + 256); their
// squared distances are computed together as packed f32x2 pairs (one FADD2 /
// FMUL2 / FFMA2 per class and centroid for both windows), reading the
// histograms from the staged tile (row stride C words: conflict-free for odd C)
// and each centroid as a float4 broadcast.  The per-thread distance registers
// double as a cache: only centroids whose coordinates changed bitwise are
// recomputed.  Exact cluster sums are shared 32-bit counter pairs moved with
// red.shared only for windows that changed cluster; the similar windows of the
// query's cluster are compacted into a list for the accuracy reduction.  The
// history tile is single-buffered (4 CTAs x 56 KB fill the SM): the next
// query's TMA is issued as soon as this query's Lloyd passes are done,
// overlapping the accuracy reduction, which reads the accuracy tile from L2
// (bulk-prefetched when the query was issued).
constexpr int kC2Threads = 256;
constexpr int kC2Ctas = 4;
constexpr int kC2Kmax = 8;

using u64 = unsigned long long;

// packed binary32 pairs (lo = window t, hi = window t + 256); each op is one
// IEEE rounding per half, round-to-nearest-even, subnormals kept
__device__ __forceinline__ u64 pk2(float a, float b) {
    u64 d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float lo2(u64 x) { return __uint_as_float((unsigned)x); }
__device__ __forceinline__ float hi2(u64 x) { return __uint_as_float((unsigned)(x >> 32)); }
// s + fl(fl(x - m)^2) for both halves.  The accumulate is written as
// fma(sq, one, s) with `one` = (1.0f, 1.0f) known only at run time: sq * 1 is
// exact, so this is fl(s + sq); a plain add.rn.f32x2 after mul.rn.f32x2 is
// contracted into one FFMA2 by ptxas 12.9 even under --fmad=false, which would
// skip the rounding of the square (rule 5).
__device__ __forceinline__ u64 d2acc(u64 s, u64 x, float m, u64 one) {
    u64 d, q, r;
    const u64 mm = pk2(m, m);
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(x), "l"(mm));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(q) : "l"(d));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(q), "l"(one), "l"(s));
    return r;
}

// One Lloyd pass's distances for a thread's two windows (packed): s[k] is
// recomputed for every centroid k in `chg` (ALL: every centroid), the others
// keep their cached values.  Classes in chunks of 4; the padded classes of the
// last chunk read x = 0 against the zero-padded centroid, adding fl(0 - 0)^2 = +0.
// CK: also fold every loaded histogram value into the running [lo, hi] range (first pass:
// the input check of R-ERR; fminf / fmaxf ignore NaN, which poisons the distances instead)
template <int KT, int KS, bool ALL, bool CK = false>
__device__ __forceinline__ void c2_dists(u64 (&s)[KS], const float* x0, const float* x1, const float* mu, int C,
                                         int CP, int K, unsigned chg, u64 one, float* lo = nullptr,
                                         float* hi = nullptr) {
#pragma unroll
    for (int k = 0; k < KS; ++k)
        if ((KT > 0 || k < K) && (ALL || ((chg >> k) & 1u))) s[k] = 0ULL;
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
        const int cb = c4 * 4;
        if (cb >= C) break;
        u64 xp[4];
        if (cb + 4 <= C) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float a = x0[cb + j], b = x1[cb + j];
                if (CK) {
                    *lo = fminf(*lo, fminf(a, b));
                    *hi = fmaxf(*hi, fmaxf(a, b));
                }
                xp[j] = pk2(a, b);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const bool in = cb + j < C;
                const float a = in ? x0[cb + j] : 0.0f, b = in ? x1[cb + j] : 0.0f;
                if (CK) {
                    *lo = fminf(*lo, fminf(a, b));
                    *hi = fmaxf(*hi, fmaxf(a, b));
                }
                xp[j] = pk2(a, b);
            }
        }
#pragma unroll
        for (int k = 0; k < KS; ++k) {
            if ((KT > 0 || k < K) && (ALL || ((chg >> k) & 1u))) {
                const float4 m = *reinterpret_cast<const float4*>(mu + k * CP + cb);
                s[k] = d2acc(s[k], xp[0], m.x, one);
                s[k] = d2acc(s[k], xp[1], m.y, one);
                s[k] = d2acc(s[k], xp[2], m.z, one);
                s[k] = d2acc(s[k], xp[3], m.w, one);
            }
        }
    }
}

// position of the highest set bit of m != 0 (one FLO: bfind.u32)
__device__ __forceinline__ int msb(unsigned m) {
    int j;
    asm("bfind.u32 %0, %1;" : "=r"(j) : "r"(m));
    return j;
}

// Exact Q32 sums as two 32-bit shared counters: v = hi * 2^16 + lo with
// lo < 2^16 and hi <= 2^16, so each half of a sum over <= 65,535 windows fits 32
// bits; adds and subtracts are native 32-bit shared atomics (the 64-bit shared
// atomic is a CAS loop on sm_100a) and wrap-around arithmetic gives the exact
// non-negative result.
__device__ __forceinline__ void sum16_add(unsigned* lo, unsigned* hi, u64 v) {
    atomicAdd(lo, (unsigned)(v & 0xFFFFu));
    atomicAdd(hi, (unsigned)(v >> 16));
}
// red.shared.add.u32 at a shared-window address
__device__ __forceinline__ void red_add_shared(unsigned addr, unsigned v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Both counters are read as signed 32-bit.  Pass 0 adds each warp's member sum S as (S mod 2^16,
// S / 2^16) while moves add / subtract single windows' splits (v mod 2^16, v / 2^16), so the low
// counter holds sum over the cluster's current members of (v mod 2^16) -- in [0, 512 (2^16 - 1)]
// -- plus a fixed pass-0 offset in (-512 * 2^16, 0]: always within +-2^31, whatever the number of
// passes; hi * 2^16 + lo is the exact cluster sum.
__device__ __forceinline__ u64 sum16_get(const unsigned* lo, const unsigned* hi) {
    return (u64)((long long)(int)*hi * 65536LL + (long long)(int)*lo);
}

// The changed centroids' distances for N = popcount(chg) < K: the N centroid
// indices (ascending) are gathered first, so the class loop is straight-line code
// over N accumulators (no per-(chunk, centroid) branch), then scattered into the
// cache with compile-time selects.
template <int N, int KS>
__device__ __forceinline__ void c2_dists_n(u64 (&s)[KS], const float* x0, const float* x1, const float* mu, int C,
                                           int CP, unsigned chg, u64 one) {
    int idx[N];
    unsigned m = chg;
#pragma unroll
    for (int j = 0; j < N; ++j) {
        idx[j] = __ffs(m) - 1;
        m &= m - 1;
    }
    u64 acc[N];
#pragma unroll
    for (int j = 0; j < N; ++j) acc[j] = 0ULL;
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
        const int cb = c4 * 4;
        if (cb >= C) break;
        u64 xp[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool in = cb + j < C;
            xp[j] = pk2(in ? x0[cb + j] : 0.0f, in ? x1[cb + j] : 0.0f);
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const float4 mm = *reinterpret_cast<const float4*>(mu + idx[j] * CP + cb);
            acc[j] = d2acc(acc[j], xp[0], mm.x, one);
            acc[j] = d2acc(acc[j], xp[1], mm.y, one);
            acc[j] = d2acc(acc[j], xp[2], mm.z, one);
            acc[j] = d2acc(acc[j], xp[3], mm.w, one);
        }
    }
#pragma unroll
    for (int k = 0; k < KS; ++k)
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (idx[j] == k) s[k] = acc[j];
}

struct C2Layout {
    size_t bar, misc, cf, hist, mu, sums, cnt, dummy, total, cf_slot;
};
struct C2Fixed {
    size_t bar, misc, mu, cnt, dummy, sums;
};
__host__ __device__ constexpr size_t c2_al16(size_t x) { return (x + 15) & ~size_t(15); }
__host__ __device__ constexpr C2Fixed c2_fixed(int C, int K) {
    const size_t CP = (size_t)((C + 3) & ~3);
    const size_t mu = 16 + 96;
    const size_t cnt = mu + c2_al16((size_t)(K + 1) * CP * 4);
    const size_t dummy = cnt + c2_al16((size_t)K * 4);
    return C2Fixed{0, 16, mu, cnt, dummy, dummy + 128};
}
__host__ __device__ inline C2Layout c2_layout(int H, int C, int G, int K) {
    C2Layout L;
    // regions whose offsets depend only on (C, K) first, so that a compile-time (K, C)
    // instantiation addresses them with constants (c2_fixed); H- and G-sized regions after
    const C2Fixed F = c2_fixed(C, K);
    L.bar = F.bar;
    L.misc = F.misc;     // ints [0..7] + the HB kernel's displacement bounds at [8..15]
    L.mu = F.mu;         // K centroids + the padded query (fused RADIUS)
    L.cnt = F.cnt;
    L.dummy = F.dummy;   // sink of the lanes beyond column C
    L.sums = F.sums;
    // Lloyd: cluster sums lo[K][C], hi[K][C] (u32); afterwards the same space holds
    // the window list (u16[H]) and two sets of per-gamma sums lo[G], hi[G], n[G]
    const size_t lloyd = (size_t)K * C * 8, gam = al16((size_t)H * 2) + (size_t)G * 24;
    size_t o = F.sums + al16(lloyd > gam ? lloyd : gam);
    L.cf_slot = al16((size_t)C * 4) + 16 + al16((size_t)G * 4) + 16;   // [cur][fallback] granule-staged
    L.cf = o;     o += 2 * L.cf_slot;
    // + 256: row H holds a copy of the query's histogram (cluster2_kernel, H < 512) and lanes past
    // column C read (and ignore) up to 31 floats beyond the last row
    L.hist = o;   o += al16((size_t)H * C * 4) + 16 + 256;
    L.total = o;
    return L;
}

struct C2Params {
    ProfParams P;
    C2Layout L;
    u64 one2;                 // (1.0f, 1.0f), opaque to the compiler
    unsigned char* scratch;   // cluster_hb_kernel: kHbStride bytes per CTA (global, L1/L2 resident)
};

// KT > 0: K == KT known at compile time; KT == 0: runtime K <= kC2Kmax.
// CT > 0: C == CT known at compile time (immediate-offset loads, no class guards).
template <int KT, int CT>
__global__ void __launch_bounds__(kC2Threads, kC2Ctas) cluster2_kernel(const __grid_constant__ C2Params A) {
    constexpr int KS = KT > 0 ? KT : kC2Kmax;   // distance registers per window
    extern __shared__ __align__(128) unsigned char smem[];
    const ProfParams& P = A.P;
    const C2Layout& L = A.L;
    const int H = P.p.n_hist, G = P.p.n_gamma, K = KT > 0 ? KT : P.p.k;
    const int C = CT > 0 ? CT : P.p.n_class;
    const int CP = (C + 3) & ~3;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // (K, C) fixed at compile time: the (C, K)-only regions at constant offsets
    constexpr C2Fixed FX = c2_fixed(CT > 0 ? CT : 1, KT > 0 ? KT : 1);
    constexpr bool kFixed = KT > 0 && CT > 0;
    const size_t o_misc = kFixed ? FX.misc : L.misc, o_mu = kFixed ? FX.mu : L.mu;
    const size_t o_cnt = kFixed ? FX.cnt : L.cnt, o_dummy = kFixed ? FX.dummy : L.dummy;
    const size_t o_sums = kFixed ? FX.sums : L.sums;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + L.bar);
    int* misc = reinterpret_cast<int*>(smem + o_misc);   // [0..1] changed-centroid masks,
                                                         // [2] query cluster, [3] list count
    float* mu = reinterpret_cast<float*>(smem + o_mu);
    unsigned* slo = reinterpret_cast<unsigned*>(smem + o_sums);
    unsigned* shi = slo + K * C;
    int* cnt = reinterpret_cast<int*>(smem + o_cnt);
    uint16_t* list = reinterpret_cast<uint16_t*>(smem + o_sums);
    unsigned* glo = reinterpret_cast<unsigned*>(smem + o_sums + al16((size_t)H * 2));
    unsigned* ghi = glo + G;
    int* gnn = reinterpret_cast<int*>(ghi + G);
    const long long Q = P.p.n_query;
    const long long items = Q > blockIdx.x ? (Q - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const u64 one = A.one2;
    // this lane's counter address = cbase + cluster * cstride (+ choff for the high half).  Lane C
    // (C < 32) carries the cluster counts in the same reds: its address is cnt[cluster] for both
    // halves, its low value the count change and its high value 0; lanes past C add into a
    // private dummy word.
    const bool lane_c = lane < C, lane_n = lane == C;
    const unsigned cbase = lane_c ? smem_addr(slo) + 4u * (unsigned)lane
                           : lane_n ? smem_addr(cnt) : smem_addr(smem + o_dummy) + 4u * (unsigned)lane;
    const unsigned cstride = lane_c ? (unsigned)(C * 4) : lane_n ? 4u : 0u;
    const unsigned choff = lane_c ? (unsigned)(K * C * 4) : 0u;
    const bool cnt_by_lane0 = C >= 32;   // no spare lane: lane 0 updates the counts itself
    const int rstride = lane_c ? C * 4 : 0;   // member-row stride (lanes >= C: the constant word)

    // leader: TMA the history tile (+ cur, fallback into slot j & 1) of this CTA's j-th query and
    // bulk-prefetch its accuracy tile into L2
    auto issue = [&](long long j) {
        const long long q = blockIdx.x + j * gridDim.x;
        unsigned char* cf = smem + L.cf + (j & 1) * L.cf_slot;
        const Granules gc = granules(P.cur + q * C, (size_t)C * 4);
        const Granules gf = granules(P.fallback + q * G, (size_t)G * 4);
        const Granules gh = granules(P.hist + (size_t)q * H * C, (size_t)H * C * 4);
        mbar_arrive_expect_tx(bar, gc.bytes + gf.bytes + gh.bytes);
        bulk_g2s(cf, gc.g0, gc.bytes, bar);
        bulk_g2s(cf + al16((size_t)C * 4) + 16, gf.g0, gf.bytes, bar);
        bulk_g2s(smem + L.hist, gh.g0, gh.bytes, bar);
        const Granules ga = granules(P.acc + (size_t)q * H * G, (size_t)H * G * 4);
        for (unsigned o = 0; o < ga.bytes; o += (1u << 20)) bulk_prefetch_l2(ga.g0 + o, min(ga.bytes - o, 1u << 20));
    };

    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
        misc[7] = (int)0x2F800000u;   // 2^-32 (read by lanes >= C in the member sums)
    }
    __syncthreads();
    if (tid == 0 && items > 0) issue(0);

    const int h0 = tid, h1 = tid + kC2Threads;
    const bool v0 = h0 < H, v1 = h1 < H;
    const int qslot = H < 2 * kC2Threads ? H : -1;   // the query's slot, if a window slot is free
    for (long long i = 0; i < items; ++i) {
        const long long q = blockIdx.x + i * gridDim.x;
        const unsigned char* cf = smem + L.cf + (i & 1) * L.cf_slot;
        const float* cur = reinterpret_cast<const float*>(cf + granules(P.cur + q * C, 4).off);
        const float* fb = reinterpret_cast<const float*>(cf + al16((size_t)C * 4) + 16 +
                                                        granules(P.fallback + q * G, 4).off);
        const float* hs = reinterpret_cast<const float*>(smem + L.hist +
                                                         granules(P.hist + (size_t)q * H * C, 4).off);
        // the query's own histogram rides in the first unused window slot (H < 512) as tile row
        // H (copied there below): its distances to the centroids come out of every Lloyd pass
        // with the same packed code and nearest rule (C19), so the query's cluster needs no
        // separate computation; the slot is invalid (v false) for every sum, move, list and output
        const int rw0 = (v0 || h0 == qslot) ? h0 : 0;
        const int rw1 = (v1 || h1 == qslot) ? h1 : rw0;
        const float* x0 = hs + (size_t)rw0 * C;
        const float* x1 = hs + (size_t)rw1 * C;
        for (int t = tid; t < 2 * K * C; t += kC2Threads) slo[t] = 0u;
        for (int t = tid; t < K; t += kC2Threads) cnt[t] = 0;
        if (tid == 0) misc[0] = misc[1] = misc[3] = misc[4] = 0;
        mbar_wait(bar, (unsigned)(i & 1));
        if (qslot >= 0)   // the query's histogram as tile row H (read after the barrier below)
            for (int c = tid; c < C; c += kC2Threads) const_cast<float*>(hs)[(size_t)H * C + c] = cur[c];
        bool ok = true;
        for (int c = tid; c < C; c += kC2Threads) ok &= in01(cur[c]);
        if (KT != 5) {   // K = 5: checked during the first pass's distances
            if (v0)
                for (int c = 0; c < C; ++c) ok &= in01(x0[c]);
            if (v1)
                for (int c = 0; c < C; ++c) ok &= in01(x1[c]);
        }
        // initial centroids mu_i = h_floor(iH/K) (C19), zero padded to CP columns; row K = the
        // query's own histogram (fused RADIUS)
        const bool rad = KT == 5 && CT == 27 && P.rad_est != nullptr;
        for (int t = tid; t < (rad ? K + 1 : K) * CP; t += kC2Threads) {
            const int ci = t / CP, c = t - ci * CP;
            mu[t] = c >= C ? 0.0f : ci < K ? hs[(size_t)(((long long)ci * H) / K) * C + c] : cur[c];
        }
        __syncthreads();
        // fused RADIUS (rule 5, C17): both windows' distances to the query are computed in pass 0
        // as a sixth centroid row (mu row K = the query), similar iff sqrt(d2) <= tau -- the same
        // sequential sum as radius_kernel (fl(x - c)^2 = fl(c - x)^2); the similar flags are
        // parked as per-warp ballot masks in misc[8..23] until the end

        u64 s[KS];
#pragma unroll
        for (int k = 0; k < KS; ++k) s[k] = 0ULL;
        const unsigned all_k = (1u << K) - 1u;
        unsigned chg = all_k;
        int oa0 = -1, oa1 = -1, na0 = 0, na1 = 0;
        int passes = 0;
        for (;;) {
            // distances of both windows to every changed centroid (rule 5 order: class ascending)
            if constexpr (KT == 5) {
                if (passes == 0) {
                    // all K distances from the initial centroids, checking every histogram
                    // value on the way; a NaN value makes both windows' distances NaN.  Lanes
                    // without a second (or any) window read a duplicate row: still a real row.
                    float lo = 1.0f, hi = 0.0f;
                    if (rad) {   // + the query row: one pass over the history loads for both
                        u64 s6[KT + 1];
                        c2_dists<KT + 1, KT + 1, true, true>(s6, x0, x1, mu, C, CP, KT + 1, (1u << (KT + 1)) - 1u,
                                                             one, &lo, &hi);
#pragma unroll
                        for (int k = 0; k < KT; ++k) s[k] = s6[k];
                        const unsigned b0 = __ballot_sync(0xffffffffu, v0 && __fsqrt_rn(lo2(s6[KT])) <= P.rad_tau);
                        const unsigned b1 = __ballot_sync(0xffffffffu, v1 && __fsqrt_rn(hi2(s6[KT])) <= P.rad_tau);
                        if (lane == 0) {
                            misc[8 + warp] = (int)b0;
                            misc[16 + warp] = (int)b1;
                        }
                    } else {
                        c2_dists<KT, KS, true, true>(s, x0, x1, mu, C, CP, K, chg, one, &lo, &hi);
                    }
                    ok &= lo >= 0.0f && hi <= 1.0f && lo2(s[0]) == lo2(s[0]) && hi2(s[0]) == hi2(s[0]);
                } else switch (__popc(chg)) {
                    case 0: break;   // nothing moved: the cache is exact
                    case 1: c2_dists_n<1, KS>(s, x0, x1, mu, C, CP, chg, one); break;
                    case 2: c2_dists_n<2, KS>(s, x0, x1, mu, C, CP, chg, one); break;
                    case 3: c2_dists_n<3, KS>(s, x0, x1, mu, C, CP, chg, one); break;
                    case 4: c2_dists_n<4, KS>(s, x0, x1, mu, C, CP, chg, one); break;
                    default: c2_dists<KT, KS, true>(s, x0, x1, mu, C, CP, K, chg, one); break;
                }
            } else {
                if (KT > 0 && chg == all_k) c2_dists<KT, KS, true>(s, x0, x1, mu, C, CP, K, chg, one);
                else c2_dists<KT, KS, false>(s, x0, x1, mu, C, CP, K, chg, one);
            }
            // nearest centroid, lowest index on ties (C19)
            if constexpr (KT == 5) {
                // min of the five by two 3-input min instructions, then the lowest index equal to
                // it (same as the strict-'<' scan for non-NaN distances; a NaN distance -- invalid
                // data, outputs zeroed -- is never the minimum)
                float d0[5], d1[5];
#pragma unroll
                for (int k = 0; k < 5; ++k) {
                    d0[k] = lo2(s[k]);
                    d1[k] = hi2(s[k]);
                }
                const float m0 = fminf(fminf(d0[0], d0[1]), fminf(d0[2], fminf(d0[3], d0[4])));
                const float m1 = fminf(fminf(d1[0], d1[1]), fminf(d1[2], fminf(d1[3], d1[4])));
                na0 = 4;
                na1 = 4;
#pragma unroll
                for (int k = 3; k >= 0; --k) {
                    na0 = d0[k] == m0 ? k : na0;
                    na1 = d1[k] == m1 ? k : na1;
                }
            } else {
                float b0 = lo2(s[0]), b1 = hi2(s[0]);
                na0 = 0;
                na1 = 0;
#pragma unroll
                for (int k = 1; k < KS; ++k) {
                    if (KT > 0 || k < K) {
                        const float d0 = lo2(s[k]), d1 = hi2(s[k]);
                        if (d0 < b0) { b0 = d0; na0 = k; }
                        if (d1 < b1) { b1 = d1; na1 = k; }
                    }
                }
            }
            // exact cluster sums: windows whose cluster changed (pass 0: all, entering from
            // "none") move between the shared counters; lane c carries column c (C <= 32; lanes
            // >= C read past their row, inside shared memory, and add into a private dummy word)
            const unsigned bm0 = __ballot_sync(0xffffffffu, v0 && na0 != oa0);
            const unsigned bm1 = __ballot_sync(0xffffffffu, v1 && na1 != oa1);
            if (passes == 0) {
                // every window enters its first cluster: per cluster, the warp's members (ballot
                // masks) are summed in registers -- low and high halves separately, so the
                // shared counters keep each window's exact (v mod 2^16, v / 2^16) split that
                // later moves subtract -- then one pair of shared adds per cluster and lane
                // lanes < C read column `lane` of the member rows; lanes >= C read misc[7] = 2^-32
                // (q32 = 1) with stride 0, so lane C's sum is the member count with no select
                const float* r0 = lane_c ? hs + (size_t)(warp * 32) * C + lane : reinterpret_cast<const float*>(misc + 7);
                const float* r1 = lane_c ? r0 + (size_t)kC2Threads * C : r0;
                for (int k = 0; k < K; ++k) {
                    const unsigned b0 = __ballot_sync(0xffffffffu, v0 && na0 == k);
                    const unsigned b1 = __ballot_sync(0xffffffffu, v1 && na1 == k);
                    if ((b0 | b1) == 0) continue;
                    if (cnt_by_lane0 && lane == 0) atomicAdd(&cnt[k], __popc(b0) + __popc(b1));
                    // the members' exact sum as one u64 (split into the counter pair once, below)
                    u64 acc = 0;
                    // members from the highest lane down (any order: exact integers): the bit
                    // index is one FLO, the row a byte offset from the warp's base
                    const unsigned char* rb0 = reinterpret_cast<const unsigned char*>(r0);
                    const unsigned char* rb1 = reinterpret_cast<const unsigned char*>(r1);
                    for (unsigned m = b0; m;) {
                        const int j = msb(m);
                        m ^= 1u << j;
                        acc += q32(*reinterpret_cast<const float*>(rb0 + j * rstride));
                    }
                    for (unsigned m = b1; m;) {
                        const int j = msb(m);
                        m ^= 1u << j;
                        acc += q32(*reinterpret_cast<const float*>(rb1 + j * rstride));
                    }
                    unsigned alo = (unsigned)acc & 0xFFFFu, ahi = (unsigned)(acc >> 16);
                    const unsigned a = cbase + (unsigned)k * cstride;
                    red_add_shared(a, alo);
                    red_add_shared(a + choff, ahi);
                }
            } else {
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) {
                    const float* rows = lane_c ? hs + (size_t)(warp * 32 + sl * kC2Threads) * C + lane
                                               : reinterpret_cast<const float*>(misc + 7);
                    const int oav = sl ? oa1 : oa0, nav = sl ? na1 : na0;
                    for (unsigned m = sl ? bm1 : bm0; m;) {
                        const int j = msb(m);   // highest moved lane first (any order)
                        m ^= 1u << j;
                        const int o = __shfl_sync(0xffffffffu, oav, j);
                        const int n = __shfl_sync(0xffffffffu, nav, j);
                        // lane C reads 2^-32 (q32 = 1): one window leaves cnt[o] and enters cnt[n]
                        const u64 v = q32(*reinterpret_cast<const float*>(reinterpret_cast<const unsigned char*>(rows) + j * rstride));
                        const unsigned lo = (unsigned)v & 0xFFFFu, hi = (unsigned)(v >> 16);
                        const unsigned ao = cbase + (unsigned)o * cstride, an = cbase + (unsigned)n * cstride;
                        red_add_shared(ao, 0u - lo);
                        red_add_shared(ao + choff, 0u - hi);
                        red_add_shared(an, lo);
                        red_add_shared(an + choff, hi);
                        if (cnt_by_lane0 && lane == 0) {
                            atomicSub(&cnt[o], 1);
                            atomicAdd(&cnt[n], 1);
                        }
                    }
                }
            }
            oa0 = na0;
            oa1 = na1;
            if (h0 == qslot) misc[2] = na0;   // the query's nearest centroid at this pass's means
            if (h1 == qslot) misc[2] = na1;
            const int any = __syncthreads_or((bm0 | bm1) != 0);
            const int it = passes++;
            if ((it > 0 && !any) || it >= P.p.max_iter) break;
            // centroid update from the exact sums (empty cluster keeps its centroid)
            for (int t = tid; t < K * C; t += kC2Threads) {
                const int ci = t / C, c = t - ci * C;
                const int n = cnt[ci];
                if (n > 0) {
                    const float nm = mean_q32(sum16_get(&slo[t], &shi[t]), n);
                    if (__float_as_uint(nm) != __float_as_uint(mu[ci * CP + c])) {
                        mu[ci * CP + c] = nm;
                        atomicOr(reinterpret_cast<unsigned*>(&misc[it & 1]), 1u << ci);
                    }
                }
            }
            __syncthreads();
            chg = (unsigned)misc[it & 1];
            if (tid == 0) misc[(it + 1) & 1] = 0;
        }
        // the history tile is free: stream the next query's while this one finishes
        if (tid == 0) {
            atomicAdd(&P.st->lloyd_passes, (unsigned long long)passes);
            if (i + 1 < items) issue(i + 1);
        }
        // the query joins its nearest centroid (lowest index on ties, C19): every warp computes it
        // (lane ci < K: distance to centroid ci; K <= 8), so no barrier publishes it
        int qc = misc[2];   // from the query's window slot (the last pass's barrier published it)
        if (qslot < 0) {
            unsigned long long key = ~0ULL;
            if (lane < K) {
                const float d = dist2_mem(cur, mu + lane * CP, C);
                key = ((unsigned long long)__float_as_uint(d) << 8) | (unsigned)lane;
            }
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) {
                const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
                key = y < key ? y : key;
            }
            qc = (int)(__shfl_sync(0xffffffffu, key, 0) & 0xFF);
        }
        // the cluster sums are dead (the last pass's barrier): their space holds one list of the
        // windows in the query's cluster (bit 14) and/or RADIUS-similar (bit 15), and both sets of
        // per-gamma sums
        for (int t = tid; t < 6 * G; t += kC2Threads) glo[t] = 0u;
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
            const bool inc = sl ? (v1 && na1 == qc) : (v0 && na0 == qc);
            const bool inr = rad && ((((unsigned)misc[(sl ? 16 : 8) + warp]) >> lane) & 1u);
            const unsigned bm = __ballot_sync(0xffffffffu, inc || inr);
            int base = 0;
            if (lane == 0 && bm) base = atomicAdd(&misc[3], __popc(bm));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (inc || inr)
                list[base + __popc(bm & ((1u << lane) - 1u))] =
                    (uint16_t)((sl ? h1 : h0) | (inc ? 0x4000 : 0) | (inr ? 0x8000 : 0));
        }
        __syncthreads();
        // validate the whole accuracy tile (NaN = unmeasured, else in [0, 1]; R-ERR): NaN-ignoring
        // running min / max from 0
        {
            const float* at = P.acc + (size_t)q * H * G;
            const long long n = (long long)H * G;
            float lo = 0.0f, hi = 0.0f;
            if ((reinterpret_cast<uintptr_t>(at) & 15) == 0) {
                const float4* a4 = reinterpret_cast<const float4*>(at);
                for (long long t = tid; t < n / 4; t += kC2Threads) {
                    const float4 x = __ldg(a4 + t);
                    lo = fminf(fminf(lo, x.x), fminf(x.y, fminf(x.z, x.w)));
                    hi = fmaxf(fmaxf(hi, x.x), fmaxf(x.y, fmaxf(x.z, x.w)));
                }
                for (long long t = (n & ~3LL) + tid; t < n; t += kC2Threads) {
                    const float x = __ldg(at + t);
                    lo = fminf(lo, x);
                    hi = fmaxf(hi, x);
                }
            } else {
                for (long long t = tid; t < n; t += kC2Threads) {
                    const float x = __ldg(at + t);
                    lo = fminf(lo, x);
                    hi = fmaxf(hi, x);
                }
            }
            ok &= !(lo < 0.0f) && !(hi > 1.0f);
        }
        // per-gamma exact sums over the listed windows' measured accuracies, both estimates from
        // one load of each element: thread t owns gamma t % G and list entries t / G (mod ngrp);
        // the accuracy tile comes from L2
        {
            const int ns = misc[3];
            const int ngrp = kC2Threads / G, g = tid % G, grp = tid / G;
            if (grp < ngrp) {
                const float* acc = P.acc + (size_t)q * H * G + g;
                u64 sc = 0, sr = 0;
                int nc = 0, nr = 0;
#pragma unroll 4
                for (int e = grp; e < ns; e += ngrp) {
                    const unsigned ent = list[e];
                    const float x = __ldg(acc + (size_t)(ent & 0x3FFFu) * G);
                    if (x == x) {
                        const u64 v = q32(x);
                        if (ent & 0x4000u) {
                            sc += v;
                            nc += 1;
                        }
                        if (ent & 0x8000u) {
                            sr += v;
                            nr += 1;
                        }
                    }
                }
                if (nc) {
                    sum16_add(&glo[g], &ghi[g], sc);
                    atomicAdd(&gnn[g], nc);
                }
                if (nr) {
                    sum16_add(&glo[3 * G + g], &ghi[3 * G + g], sr);
                    atomicAdd(&gnn[3 * G + g], nr);
                }
            }
        }
        ok = __syncthreads_and(ok) != 0;
        if (!ok && tid == 0) flag_data_error(P.st);
        if (P.out_cluster) {
            int* oc = P.out_cluster + q * (H + 1);
            if (v0) oc[h0] = ok ? na0 : 0;
            if (v1) oc[h1] = ok ? na1 : 0;
            if (tid == 0) oc[H] = ok ? qc : 0;
        }
        // outputs: threads [0, G) the CLUSTER estimate, [G, 2G) the fused RADIUS estimate
        for (int t = tid; t < (rad ? 2 * G : G); t += kC2Threads) {
            const int set = t >= G, g = t - set * G;
            const int o = set * 3 * G + g;
            int n = gnn[o];
            float est = 0.0f;
            if (!ok) n = 0;
            else est = n > 0 ? mean_q32(sum16_get(&glo[o], &ghi[o]), n) : fb[g];
            (set ? P.rad_est : P.out_est)[q * G + g] = est;
            (set ? P.rad_n : P.out_n)[q * G + g] = n;
        }
        __syncthreads();   // sums, list and the cur/fallback slot are free again
    }
}

// ------------------------------------------------------------------------
// CLUSTER with distance bounds (the bench shape: K = 5, C = 27, H <= 512)
// ------------------------------------------------------------------------
// After Lloyd's first passes few windows change cluster, yet cluster2_kernel recomputes
// every window's distances to every centroid that moved.  Here each window keeps
// Hamerly's bounds -- u >= its Euclidean distance D to its own centroid, l <= D to every
// other centroid -- advanced after each centroid update by the centroids' displacements
// delta_k (triangle inequality: u += delta_a, l -= max_{k != a} delta_k), with every
// displacement, bound and test rounded in the safe direction (__f*_ru / __f*_rd).  Rule 5
// computes d2 as a sequential sum of C rounded squares of rounded differences, so
// |d2 - D^2| <= eps D^2 + eta with eps = 4e-6 >= gamma_{C+2} for C <= 32 and eta = 2^-120
// (subnormal terms).  Hence
//     fl_ru(u^2 (1 + 2 eps) + eta) < fl_rd(l^2 (1 - 2 eps) - eta)
// guarantees rule 5's fp32 distance to the current centroid is STRICTLY below every other
// fp32 distance: the oracle's argmin (lowest index on ties) keeps the assignment, with no
// distance computed.  Windows failing the test ("needy") are compacted into a CTA work
// list and recomputed exactly (all K distances, rule 5, the packed f32x2 path of
// cluster2_kernel), two per thread by the first ceil(n/2) threads, so whole warps skip the
// distance phase; the workers also move the exact cluster sums of windows that changed
// cluster and hand the new assignment and bounds back to the owning thread through a
// per-CTA scratch in global memory (5.5 KB, L1/L2 resident).  Every assignment equals the
// oracle's, hence every sum, centroid, pass count and output (bit-exact parity tests).
constexpr float kHbEps2 = 8.0e-6f;          // 2 eps; 1 + 2 eps >= 1 / (1 - eps), 1 - 2 eps <= 1 / (1 + eps)
constexpr float kHbEta = 7.52316385e-37f;   // 2^-120 >= 32 * 2^-149
constexpr int kHbStride = 5632;             // per CTA: list u16[512] | u f32[512] | l f32[512] | a u8[512]

// upper bound of rule 5's d2 given D <= u
__device__ __forceinline__ float hb_ub2(float u) { return __fadd_ru(__fmul_ru(__fmul_ru(u, u), 1.0f + kHbEps2), kHbEta); }
// lower bound of rule 5's d2 given D >= l
__device__ __forceinline__ float hb_lb2(float l) { return __fsub_rd(__fmul_rd(__fmul_rd(l, l), 1.0f - kHbEps2), kHbEta); }
// upper / lower bound of D given rule 5's d2
__device__ __forceinline__ float hb_u(float d2) { return __fsqrt_ru(__fmul_ru(__fadd_ru(d2, kHbEta), 1.0f + kHbEps2)); }
__device__ __forceinline__ float hb_l(float d2) {
    return __fsqrt_rd(fmaxf(__fmul_rd(__fsub_rd(d2, kHbEta), 1.0f - kHbEps2), 0.0f));
}

// nearest centroid (lowest index on ties, C19) and second-smallest distance of both packed
// windows -> assignment and bounds
template <int K>
__device__ __forceinline__ void hb_nearest(const u64 (&s)[K], int& na, int& nb, float& ua, float& la, float& ub,
                                           float& lb) {
    float b0 = lo2(s[0]), b1 = hi2(s[0]), c0 = INFINITY, c1 = INFINITY;
    na = 0;
    nb = 0;
#pragma unroll
    for (int k = 1; k < K; ++k) {
        const float d0 = lo2(s[k]), d1 = hi2(s[k]);
        if (d0 < b0) { c0 = b0; b0 = d0; na = k; } else if (d0 < c0) { c0 = d0; }
        if (d1 < b1) { c1 = b1; b1 = d1; nb = k; } else if (d1 < c1) { c1 = d1; }
    }
    ua = hb_u(b0);
    la = hb_l(c0);
    ub = hb_u(b1);
    lb = hb_l(c1);
}

// Exact Q32 (low 16 bits, rest) sums of the member windows m (bits = lanes) of one warp
// slot, lane = column: four independent load -> convert chains per step for ILP.
__device__ __forceinline__ void member_sums(unsigned m, const float* rows, int C, unsigned& alo, unsigned& ahi) {
    while (m) {
        const int j0 = __ffs(m) - 1;
        m &= m - 1;
        const bool h1 = m != 0;
        const int j1 = h1 ? __ffs(m) - 1 : j0;
        m &= m - 1;
        const bool h2 = m != 0;
        const int j2 = h2 ? __ffs(m) - 1 : j0;
        m &= m - 1;
        const bool h3 = m != 0;
        const int j3 = h3 ? __ffs(m) - 1 : j0;
        m &= m - 1;
        const u64 v0 = q32(rows[j0 * C]), v1 = q32(rows[j1 * C]), v2 = q32(rows[j2 * C]), v3 = q32(rows[j3 * C]);
        alo += ((unsigned)v0 & 0xFFFFu) + (h1 ? (unsigned)v1 & 0xFFFFu : 0u) + (h2 ? (unsigned)v2 & 0xFFFFu : 0u) +
               (h3 ? (unsigned)v3 & 0xFFFFu : 0u);
        ahi += (unsigned)(v0 >> 16) + (h1 ? (unsigned)(v1 >> 16) : 0u) + (h2 ? (unsigned)(v2 >> 16) : 0u) +
               (h3 ? (unsigned)(v3 >> 16) : 0u);
    }
}

template <int K, int C>
__global__ void __launch_bounds__(kC2Threads, kC2Ctas) cluster_hb_kernel(const __grid_constant__ C2Params A) {
    constexpr int CP = (C + 3) & ~3;
    extern __shared__ __align__(128) unsigned char smem[];
    const ProfParams& P = A.P;
    const C2Layout& L = A.L;
    const int H = P.p.n_hist, G = P.p.n_gamma;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + L.bar);
    int* misc = reinterpret_cast<int*>(smem + L.misc);   // [2] query cluster, [3] similar-window count,
                                                         // [4] work-list count; floats [8..8+K) displacements
    float* dl = reinterpret_cast<float*>(misc + 8);
    float* mu = reinterpret_cast<float*>(smem + L.mu);
    unsigned* slo = reinterpret_cast<unsigned*>(smem + L.sums);
    unsigned* shi = slo + K * C;
    int* cnt = reinterpret_cast<int*>(smem + L.cnt);
    uint16_t* list = reinterpret_cast<uint16_t*>(smem + L.sums);
    unsigned* glo = reinterpret_cast<unsigned*>(smem + L.sums + al16((size_t)H * 2));
    unsigned* ghi = glo + G;
    int* gnn = reinterpret_cast<int*>(ghi + G);
    unsigned char* scr = A.scratch + (size_t)blockIdx.x * kHbStride;
    uint16_t* wl = reinterpret_cast<uint16_t*>(scr);           // work list: window | old cluster << 9
    float* res_u = reinterpret_cast<float*>(scr + 1024);
    float* res_l = reinterpret_cast<float*>(scr + 3072);
    unsigned char* res_a = scr + 5120;
    const long long Q = P.p.n_query;
    const long long items = Q > blockIdx.x ? (Q - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const u64 one = A.one2;
    const unsigned full = 0xffffffffu;
    const bool lane_c = lane < C;
    const unsigned cbase = lane_c ? smem_addr(slo) + 4u * (unsigned)lane : smem_addr(smem + L.dummy) + 4u * (unsigned)lane;
    const unsigned cstride = lane_c ? (unsigned)(C * 4) : 0u, choff = lane_c ? (unsigned)(K * C * 4) : 0u;
    const unsigned lt = (1u << lane) - 1u;

    auto issue = [&](long long j) {
        const long long q = blockIdx.x + j * gridDim.x;
        unsigned char* cf = smem + L.cf + (j & 1) * L.cf_slot;
        const Granules gc = granules(P.cur + q * C, (size_t)C * 4);
        const Granules gf = granules(P.fallback + q * G, (size_t)G * 4);
        const Granules gh = granules(P.hist + (size_t)q * H * C, (size_t)H * C * 4);
        mbar_arrive_expect_tx(bar, gc.bytes + gf.bytes + gh.bytes);
        bulk_g2s(cf, gc.g0, gc.bytes, bar);
        bulk_g2s(cf + al16((size_t)C * 4) + 16, gf.g0, gf.bytes, bar);
        bulk_g2s(smem + L.hist, gh.g0, gh.bytes, bar);
        const Granules ga = granules(P.acc + (size_t)q * H * G, (size_t)H * G * 4);
        for (unsigned o = 0; o < ga.bytes; o += (1u << 20)) bulk_prefetch_l2(ga.g0 + o, min(ga.bytes - o, 1u << 20));
    };

    if (tid == 0) {
        mbar_init(bar, 1);
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0 && items > 0) issue(0);

    const int h0 = tid, h1 = tid + kC2Threads;
    const bool v0 = h0 < H, v1 = h1 < H;
    for (long long i = 0; i < items; ++i) {
        const long long q = blockIdx.x + i * gridDim.x;
        const unsigned char* cf = smem + L.cf + (i & 1) * L.cf_slot;
        const float* cur = reinterpret_cast<const float*>(cf + granules(P.cur + q * C, 4).off);
        const float* fb = reinterpret_cast<const float*>(cf + al16((size_t)C * 4) + 16 +
                                                        granules(P.fallback + q * G, 4).off);
        const float* hs = reinterpret_cast<const float*>(smem + L.hist +
                                                         granules(P.hist + (size_t)q * H * C, 4).off);
        const float* x0 = hs + (size_t)(v0 ? h0 : 0) * C;
        const float* x1 = hs + (size_t)(v1 ? h1 : (v0 ? h0 : 0)) * C;
        for (int t = tid; t < 2 * K * C; t += kC2Threads) slo[t] = 0u;
        for (int t = tid; t < K; t += kC2Threads) cnt[t] = 0;
        if (tid == 0) misc[3] = misc[4] = 0;
        mbar_wait(bar, (unsigned)(i & 1));
        bool ok = true;
        for (int c = tid; c < C; c += kC2Threads) ok &= in01(cur[c]);
        for (int t = tid; t < K * CP; t += kC2Threads) {
            const int ci = t / CP, c = t - ci * CP;
            mu[t] = c < C ? hs[(size_t)(((long long)ci * H) / K) * C + c] : 0.0f;
        }
        __syncthreads();

        // pass 0: every window's K distances from the initial centroids (rule 5), checking
        // every histogram value on the way (a NaN makes the distances NaN)
        int a0, a1;
        float u0, l0, u1, l1;
        {
            u64 s[K];
            float lo = 1.0f, hi = 0.0f;
            c2_dists<K, K, true, true>(s, x0, x1, mu, C, CP, K, (1u << K) - 1u, one, &lo, &hi);
            ok &= lo >= 0.0f && hi <= 1.0f && lo2(s[0]) == lo2(s[0]) && hi2(s[0]) == hi2(s[0]);
            hb_nearest<K>(s, a0, a1, u0, l0, u1, l1);
        }
        // every window enters its first cluster: exact sums per cluster and warp
        {
            const float* r0 = hs + (size_t)(warp * 32) * C + lane;
            const float* r1 = r0 + (size_t)kC2Threads * C;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const unsigned b0 = __ballot_sync(full, v0 && a0 == k);
                const unsigned b1 = __ballot_sync(full, v1 && a1 == k);
                if ((b0 | b1) == 0) continue;
                if (lane == 0) atomicAdd(&cnt[k], __popc(b0) + __popc(b1));
                unsigned alo = 0, ahi = 0;
                member_sums(b0, r0, C, alo, ahi);
                member_sums(b1, r1, C, alo, ahi);
                const unsigned a = cbase + (unsigned)k * cstride;
                red_add_shared(a, alo);
                red_add_shared(a + choff, ahi);
            }
        }
        int any = __syncthreads_or(v0 || v1);
        int passes = 1;
        for (;;) {
            const int it = passes - 1;   // centroid updates so far
            if ((it > 0 && !any) || it >= P.p.max_iter) break;
            // centroid update from the exact sums (empty cluster keeps its centroid), and each
            // centroid's displacement bound: warp k, lane = column
            if (warp < K) {
                const int k = warp;
                float dd = 0.0f;
                const int n = cnt[k];
                if (lane_c && n > 0) {
                    const float old = mu[k * CP + lane];
                    const float nm = mean_q32(sum16_get(&slo[k * C + lane], &shi[k * C + lane]), n);
                    mu[k * CP + lane] = nm;
                    const float du = fmaxf(__fsub_ru(nm, old), __fsub_ru(old, nm));
                    dd = __fmul_ru(du, du);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) dd = __fadd_ru(dd, __shfl_xor_sync(full, dd, o));
                if (lane == 0) dl[k] = __fsqrt_ru(dd);
            }
            if (tid == 0) misc[4] = 0;
            __syncthreads();
            // phase A (owners): advance the bounds, test, list the needy windows
            float m1 = -1.0f, m2 = 0.0f;
            int i1 = 0;
#pragma unroll
            for (int k = 0; k < K; ++k) {
                const float d = dl[k];
                if (d > m1) { m2 = m1; m1 = d; i1 = k; } else if (d > m2) { m2 = d; }
            }
            m2 = fmaxf(m2, 0.0f);
            u0 = __fadd_ru(u0, dl[a0]);
            l0 = fmaxf(__fsub_rd(l0, a0 == i1 ? m2 : m1), 0.0f);
            u1 = __fadd_ru(u1, dl[a1]);
            l1 = fmaxf(__fsub_rd(l1, a1 == i1 ? m2 : m1), 0.0f);
            const bool n0 = v0 && !(hb_ub2(u0) < hb_lb2(l0));
            const bool n1 = v1 && !(hb_ub2(u1) < hb_lb2(l1));
            {
                const unsigned b0 = __ballot_sync(full, n0), b1 = __ballot_sync(full, n1);
                const int nw = __popc(b0) + __popc(b1);
                int base = 0;
                if (lane == 0 && nw) base = atomicAdd(&misc[4], nw);
                base = __shfl_sync(full, base, 0);
                if (n0) wl[base + __popc(b0 & lt)] = (uint16_t)(h0 | (a0 << 9));
                if (n1) wl[base + __popc(b0) + __popc(b1 & lt)] = (uint16_t)(h1 | (a1 << 9));
            }
            __syncthreads();
            // phase B (workers): exact distances of two listed windows per thread, moves
            const int nl = misc[4];
            const int pairs = (nl + 1) >> 1;
            bool mv = false;
            if (warp * 32 < pairs) {
                const bool w0 = tid < pairs, w1 = 2 * tid + 1 < nl;
                const unsigned e0 = w0 ? wl[2 * tid] : 0u;
                const unsigned e1 = w1 ? wl[2 * tid + 1] : e0;
                const int wa = (int)(e0 & 511u), wb = (int)(e1 & 511u), oa = (int)(e0 >> 9), ob = (int)(e1 >> 9);
                u64 s[K];
                c2_dists<K, K, true>(s, hs + (size_t)wa * C, hs + (size_t)wb * C, mu, C, CP, K, (1u << K) - 1u, one);
                int na, nb;
                float ua, la, ub, lb;
                hb_nearest<K>(s, na, nb, ua, la, ub, lb);
                if (w0) {
                    res_a[wa] = (unsigned char)na;
                    res_u[wa] = ua;
                    res_l[wa] = la;
                }
                if (w1) {
                    res_a[wb] = (unsigned char)nb;
                    res_u[wb] = ub;
                    res_l[wb] = lb;
                }
                // windows that changed cluster move between the exact shared counters
#pragma unroll
                for (int sl = 0; sl < 2; ++sl) {
                    const int wv = sl ? wb : wa, ov = sl ? ob : oa, nv = sl ? nb : na;
                    const unsigned bm = __ballot_sync(full, (sl ? w1 : w0) && nv != ov);
                    mv |= bm != 0;
                    for (unsigned m = bm; m; m &= m - 1) {
                        const int j = __ffs(m) - 1;
                        const int w = __shfl_sync(full, wv, j);
                        const int o = __shfl_sync(full, ov, j);
                        const int n = __shfl_sync(full, nv, j);
                        const u64 v = q32(hs[(size_t)w * C + lane]);
                        const unsigned vlo = (unsigned)v & 0xFFFFu, vhi = (unsigned)(v >> 16);
                        const unsigned ao = cbase + (unsigned)o * cstride, an = cbase + (unsigned)n * cstride;
                        red_add_shared(ao, 0u - vlo);
                        red_add_shared(ao + choff, 0u - vhi);
                        red_add_shared(an, vlo);
                        red_add_shared(an + choff, vhi);
                        if (lane == 0) {
                            atomicSub(&cnt[o], 1);
                            atomicAdd(&cnt[n], 1);
                        }
                    }
                }
            }
            any = __syncthreads_or(mv);
            // phase C (owners): the recomputed windows' assignment and bounds
            if (n0) {
                a0 = res_a[h0];
                u0 = res_u[h0];
                l0 = res_l[h0];
            }
            if (n1) {
                a1 = res_a[h1];
                u1 = res_u[h1];
                l1 = res_l[h1];
            }
            ++passes;
        }
        // the history tile is free: stream the next query's while this one finishes
        if (tid == 0) {
            atomicAdd(&P.st->lloyd_passes, (unsigned long long)passes);
            if (i + 1 < items) issue(i + 1);
        }
        const int na0 = a0, na1 = a1;
        // the query joins its nearest centroid: lane i computes distance to centroid i
        if (warp == 0) {
            unsigned long long key = ~0ULL;
            for (int ci = lane; ci < K; ci += 32) {
                const float d = dist2_mem(cur, mu + ci * CP, C);
                const unsigned long long kk = ((unsigned long long)__float_as_uint(d) << 8) | (unsigned)ci;
                key = kk < key ? kk : key;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long y = __shfl_xor_sync(0xffffffffu, key, o);
                key = y < key ? y : key;
            }
            if (lane == 0) misc[2] = (int)(key & 0xFF);
        }
        // validate the whole accuracy tile (NaN = unmeasured, else in [0, 1]; R-ERR)
        {
            const float* at = P.acc + (size_t)q * H * G;
            const long long n = (long long)H * G;
            if ((reinterpret_cast<uintptr_t>(at) & 15) == 0) {
                const float4* a4 = reinterpret_cast<const float4*>(at);
                for (long long t = tid; t < n / 4; t += kC2Threads) {
                    const float4 x = __ldg(a4 + t);
                    ok &= !(x.x < 0.0f) && !(x.x > 1.0f) && !(x.y < 0.0f) && !(x.y > 1.0f) &&
                          !(x.z < 0.0f) && !(x.z > 1.0f) && !(x.w < 0.0f) && !(x.w > 1.0f);
                }
                for (long long t = (n & ~3LL) + tid; t < n; t += kC2Threads) {
                    const float x = __ldg(at + t);
                    ok &= !(x < 0.0f) && !(x > 1.0f);
                }
            } else {
                for (long long t = tid; t < n; t += kC2Threads) {
                    const float x = __ldg(at + t);
                    ok &= !(x < 0.0f) && !(x > 1.0f);
                }
            }
        }
        __syncthreads();   // misc[2] visible; the cluster sums are dead: their space holds the list
        const int qc = misc[2];
        for (int t = tid; t < 3 * G; t += kC2Threads) glo[t] = 0u;
        // compact list of the query cluster's windows (any order: the sums are exact integers)
#pragma unroll
        for (int sl = 0; sl < 2; ++sl) {
            const bool in = sl ? (v1 && na1 == qc) : (v0 && na0 == qc);
            const unsigned bm = __ballot_sync(0xffffffffu, in);
            int base = 0;
            if (lane == 0 && bm) base = atomicAdd(&misc[3], __popc(bm));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (in) list[base + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)(sl ? h1 : h0);
        }
        __syncthreads();
        // per-gamma exact sums over the similar, measured windows: thread t owns gamma t % G and
        // list entries t / G (mod ngrp); the accuracy tile comes from L2
        {
            const int ns = misc[3];
            const int ngrp = kC2Threads / G, g = tid % G, grp = tid / G;
            if (grp < ngrp) {
                const float* acc = P.acc + (size_t)q * H * G + g;
                u64 gs = 0;
                int gn = 0;
#pragma unroll 4
                for (int e = grp; e < ns; e += ngrp) {
                    const float x = __ldg(acc + (size_t)list[e] * G);
                    if (x == x) {
                        gs += q32(x);
                        gn += 1;
                    }
                }
                if (gn) {
                    sum16_add(&glo[g], &ghi[g], gs);
                    atomicAdd(&gnn[g], gn);
                }
            }
        }
        ok = __syncthreads_and(ok) != 0;
        if (!ok && tid == 0) flag_data_error(P.st);
        if (P.out_cluster) {
            int* oc = P.out_cluster + q * (H + 1);
            if (v0) oc[h0] = ok ? na0 : 0;
            if (v1) oc[h1] = ok ? na1 : 0;
            if (tid == 0) oc[H] = ok ? qc : 0;
        }
        for (int g = tid; g < G; g += kC2Threads) {
            int n = gnn[g];
            float est = 0.0f;
            if (!ok) n = 0;
            else est = n > 0 ? mean_q32(sum16_get(&glo[g], &ghi[g]), n) : fb[g];
            P.out_est[q * G + g] = est;
            P.out_n[q * G + g] = n;
        }
        __syncthreads();   // sums, list and the cur/fallback slot are free again
    }
}

// queries with an empty history: every estimate is the caller's fallback
__global__ void no_history_kernel(ProfParams P) {
    const long long QG = (long long)P.p.n_query * P.p.n_gamma;
    const int C = P.p.n_class, G = P.p.n_gamma;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < QG; e += (long long)gridDim.x * blockDim.x) {
        long long q = e / G;
        bool ok = true;
        for (int c = 0; c < C; ++c) ok &= in01(__ldg(P.cur + q * C + c));
        if (!ok) flag_data_error(P.st);
        P.out_est[e] = ok ? __ldg(P.fallback + e) : 0.0f;
        P.out_n[e] = 0;
        if (P.out_cluster && e % G == 0) P.out_cluster[q] = ok && P.p.mode == EKYA_PROFILE_CLUSTER ? -1 : 0;
    }
}

}  // namespace

int launch_profile(ekya_handle* h, const ekya_profile_dims& p, const float* cur, const float* hist,
                   const float* hist_acc, const float* fallback, float* out_est, int32_t* out_n,
                   int32_t* out_cluster, cudaStream_t s, float* rad_est, int32_t* rad_n, float rad_tau) {
    ProfParams P{};
    P.p = p;
    P.rad_est = rad_est;
    P.rad_n = rad_n;
    P.rad_tau = rad_tau;
    P.cur = cur;
    P.hist = hist;
    P.acc = hist_acc;
    P.fallback = fallback;
    P.out_est = out_est;
    P.out_n = out_n;
    P.out_cluster = out_cluster;
    P.st = h->dstate;
    const int C = p.n_class, G = p.n_gamma, H = p.n_hist, K = p.k;
    if (p.n_query == 0) return EKYA_OK;
    const size_t budget = h->smem_optin;
    if (G > kProfThreads) return EKYA_ERR_LIMIT;
    if (H == 0) {
        no_history_kernel<<<h->sm_count * 4, 256, 0, s>>>(P);
        h->launches++;
        return cuda_status(cudaGetLastError());
    }
    long long grid = std::min<long long>(p.n_query, h->sm_count);
    cudaError_t e;
    if (p.mode == EKYA_PROFILE_RADIUS) {
        const size_t scratch_fixed = scratch_layout(0, 0, C, 0, false).total;
        const size_t per_window = (size_t)(C + G) * 4 + 2;
        // kRadiusStages stages of Hc windows: a query is split into equal chunks so
        // that several chunks are always in flight while one is being computed
        const int NS = kRadiusStages;
        long long hc = (long long)((budget - scratch_fixed - NS * (stage_layout(C, G, 0, true).total + 64)) /
                                   (NS * per_window));
        if (hc < 1) return EKYA_ERR_SHAPE;
        hc = std::min<long long>(hc, H);
        const long long nch = (H + hc - 1) / hc;
        P.Hc = (int)((H + nch - 1) / nch);
        P.stages = NS;
        P.stage_bytes = stage_layout(C, G, P.Hc, true).total;
        size_t smem = P.stages * P.stage_bytes + scratch_layout(H, P.Hc, C, 0, false).total;
        if (smem > budget) return EKYA_ERR_SHAPE;
        e = cudaFuncSetAttribute(radius_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return EKYA_ERR_CUDA;
        radius_kernel<<<(unsigned)grid, kProfThreads, smem, s>>>(P);
    } else {
        if (H >= 65536 || K > 32) return EKYA_ERR_LIMIT;
        if (H <= 2 * kC2Threads && C <= 32 && K <= kC2Kmax && G <= kC2Threads &&
            c2_layout(H, C, G, K).total <= budget) {
            C2Params A{};
            A.P = P;
            A.L = c2_layout(H, C, G, K);
            const float one = 1.0f;
            unsigned ob;
            memcpy(&ob, &one, 4);
            A.one2 = ((unsigned long long)ob << 32) | ob;
            const size_t smem = A.L.total;
            // EKYA_CLUSTER_HB=1 selects the distance-bound kernel for the bench shape (A/B timing;
            // measured slower so far)
            const bool hb = K == 5 && C == 27 && getenv("EKYA_CLUSTER_HB") && !rad_est;
            auto k2 = hb ? cluster_hb_kernel<5, 27>
                         : (K == 5 && C == 27) ? cluster2_kernel<5, 27> : cluster2_kernel<0, 0>;
            if (rad_est && !(K == 5 && C == 27)) return EKYA_ERR_SHAPE;   // fused RADIUS: <5, 27> only
            e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) return EKYA_ERR_CUDA;
            int per_sm = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k2, kC2Threads, smem);
            grid = std::min<long long>(p.n_query, (long long)h->sm_count * std::max(per_sm, 1));
            if (hb) {
                A.scratch = static_cast<unsigned char*>(handle_scratch(h, (size_t)grid * kHbStride));
                if (!A.scratch) return EKYA_ERR_CUDA;
            }
            k2<<<(unsigned)grid, kC2Threads, smem, s>>>(A);
            h->launches++;
            return cuda_status(cudaGetLastError());
        }
        if (rad_est) return EKYA_ERR_SHAPE;   // fused RADIUS: cluster2_kernel<5, 27> only
        const size_t scratch = scratch_layout(H, H, C, K, true).total;
        P.Hc = H;
        const bool reg = (H <= kProfThreads) && (C <= 32);
        // prefer two stages with the accuracy tile staged, then fewer
        int cfgs[4][2] = {{2, 1}, {2, 0}, {1, 1}, {1, 0}};
        size_t smem = 0;
        bool found = false;
        for (auto& cf : cfgs) {
            size_t sb = stage_layout(C, G, H, cf[1] != 0).total;
            size_t tot = cf[0] * sb + scratch;
            if (tot <= budget) {
                P.stages = cf[0];
                P.acc_staged = cf[1];
                P.stage_bytes = sb;
                smem = tot;
                found = true;
                break;
            }
        }
        if (!found) return EKYA_ERR_SHAPE;
        auto kern = reg ? cluster_kernel<true> : cluster_kernel<false>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return EKYA_ERR_CUDA;
        kern<<<(unsigned)grid, kProfThreads, smem, s>>>(P);
    }
    h->launches++;
    return cuda_status(cudaGetLastError());
}

// RADIUS and CLUSTER estimates of the same queries.  The bench shape (k = 5, C = 27, H <= 512)
// runs both in ONE pass of cluster2_kernel<5, 27> over the staged history (the tile is read
// from HBM once); other shapes run radius_kernel then the CLUSTER kernel.
bool profile_fusable(const ekya_handle* h, const ekya_profile_dims& p) {
    return p.k == 5 && p.n_class == 27 && p.n_hist >= 1 && p.n_hist <= 2 * kC2Threads && p.n_gamma <= kC2Threads &&
           c2_layout(p.n_hist, p.n_class, p.n_gamma, p.k).total <= h->smem_optin && !getenv("EKYA_PROFILE_UNFUSED");
}

int launch_profile_both(ekya_handle* h, const ekya_profile_dims& p, const float* cur, const float* hist,
                        const float* hist_acc, const float* fallback, float* rad_est, int32_t* rad_n,
                        float* cl_est, int32_t* cl_n, int32_t* out_cluster, cudaStream_t s) {
    ekya_profile_dims pc = p;
    pc.mode = EKYA_PROFILE_CLUSTER;
    if (profile_fusable(h, p))
        return launch_profile(h, pc, cur, hist, hist_acc, fallback, cl_est, cl_n, out_cluster, s, rad_est, rad_n,
                              p.tau);
    ekya_profile_dims pr = p;
    pr.mode = EKYA_PROFILE_RADIUS;
    const int e = launch_profile(h, pr, cur, hist, hist_acc, fallback, rad_est, rad_n, nullptr, s);
    if (e != EKYA_OK) return e;
    return launch_profile(h, pc, cur, hist, hist_acc, fallback, cl_est, cl_n, out_cluster, s);
}

}  // namespace ekya
