// profile.cu -- ekya_profile_estimate: the class-distribution-similarity
// accuracy estimator (draft appendix).
//
// Both modes run one persistent CTA (512 threads) per SM that walks its
// queries through a two-stage shared-memory pipeline fed by the TMA bulk-copy
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
// history.  Each thread keeps its window's histogram in registers across
// iterations and reads centroids as float4 broadcasts; cluster sums are exact
// Q32 integers maintained INCREMENTALLY (only windows whose assignment changed
// are moved between clusters, with 64-bit shared atomics), which is
// bit-identical to the oracle's full recomputation because integer addition is
// associative.
#include <algorithm>
#include <cfloat>

#include "launch.h"

namespace ekya {

namespace {

constexpr int kProfThreads = 512;
constexpr int kRadiusStages = 2;

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
    L.sim = o;    o += al16((size_t)(cluster ? H : Hc) + 1);
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
    GammaAcc a;
    bool ok = true;
    for (long long i = 0; i < items; ++i) {
        const int s = (int)(i % NS);
        const long long q = item_q(i);
        const int h0 = item_h0(i), hn = min(Hc, H - h0);
        mbar_wait(&bar[s], (unsigned)((i / NS) & 1));
        const StagePtrs sp = stage_ptrs(P, smem + s * P.stage_bytes, q, h0, true, L);
        if (h0 == 0) {
            gacc_reset(a, G);
            ok = true;
            for (int c = threadIdx.x; c < C; c += blockDim.x) ok &= in01(sp.cur[c]);
        }
        for (int h = threadIdx.x; h < hn; h += blockDim.x) {
            const float* row = sp.hist + (size_t)h * C;
            float d2 = 0.0f;
            for (int c = 0; c < C; ++c) {
                float x = row[c];
                ok &= in01(x);
                float diff = fsub(sp.cur[c], x);
                d2 = fadd(d2, fmul(diff, diff));
            }
            sim[h] = __fsqrt_rn(d2) <= tau;
        }
        __syncthreads();
        ok &= gacc_add(a, sp.acc, sim, hn, G);
        const bool last = h0 + hn >= H;
        if (last) {
            ok = __syncthreads_and(ok) != 0;
            if (!ok && threadIdx.x == 0) flag_data_error(P.st);
            gacc_finish(a, ps, pn, sp.fb, P, q, ok);
        }
        __syncthreads();   // stage s and sim[] are free again
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
        const size_t per_window = (size_t)(C + G) * 4 + 1;
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

}  // namespace ekya
