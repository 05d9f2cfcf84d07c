// thief.cu -- ekya_thief_schedule: Algorithm 1, one warp per
// scheduling instance.
//
// A Delta-steal (thief t, victim w) changes at most the two streams s(t), s(w),
// so the objective change is an exact integer
//     dS(t, w) = up[t] + down[w]        if s(t) != s(w)
//     dS(t, w) = move[t]                if s(t) == s(w)  (w = t ^ 1)
// where, per stream, up/down/move are Q32 differences of the stream value at
// the seven splits {(rt,ri), (rt,ri+D), (rt+D,ri), (rt,ri-D), (rt-D,ri),
// (rt+D,ri-D), (rt-D,ri+D)}.  The arrays live in shared memory and only the
// touched streams are re-evaluated after a step: O(J) per step instead of the
// oracle's O(J^2) full PickConfigs recomputations, with bit-identical
// decisions (exact integers, identical tie rules).
//
// Stream evaluation is warp-parallel: lane g evaluates rule 2 for retraining
// config g (lane 0 = no retraining) at rt-D, rt, rt+D and a REDUX max gives
// G*(rt'); lambda*(ri') comes from a per-stream breakpoint table (lambda*
// changes only at the keep-up thresholds) via one REDUX + one shuffle; then
// value(rt', ri') = fl(f_lambda*(ri') G*(rt')) -- exact because x -> fl(c x) is
// monotone, and equal to the oracle's max over gamma of fl(f g_gamma).
//
// STEEPEST (C12): per step, per stream best down (value desc, index asc) ->
// top-2 by stream -> per thief its best victim -> argmax over thieves with
// lexicographic (t, w) ties; 64-bit keys reduced with two 32-bit REDUX
// passes.  Accept iff dS > 0.
// LITERAL: thieves in order; victims scanned 32 at a time with a warp ballot of
// "first steal improves" -- victims before the first set bit leave the state
// unchanged, exactly as the sequential loop -- then the steal chain on that
// victim, then the scan resumes after it.
#include <algorithm>
#include <cstdlib>
#include <climits>

#include "launch.h"
#include <type_traits>
#include "stream_tables.cuh"

namespace ekya {

namespace {

constexpr int kThiefThreads = 128;      // 4 warps = 4 instances per CTA
constexpr long long kInvalid = (long long)0x8000000000000000ULL;
constexpr long long kKeyOff = 1LL << 40;
constexpr unsigned FULL = 0xffffffffu;

struct ThiefParams {
    ekya_dims d;
    ekya_tables t;
    DevState* st;
    int mode;
    uint16_t* out_alloc;
    uint8_t* out_cfg;
    unsigned long long* out_sum;
    float* out_mean;
    uint32_t* out_steps;
    int warps;           // warps per CTA
    size_t warp_bytes;   // shared bytes per warp (state + staged tables)
    size_t state_bytes;  // shared bytes of the per-warp state
    int stage;           // stage stale/cost/post of the instance in shared memory
    int nsm;             // G* cache slots per stream - 1 (a power of two minus one)
    unsigned total_warps;   // warps launched (the claim counters' reset)
};

// Per-stream record rec[v][8] (Q32 units): [0] current value, [1] up (inference
// +D), [2] up (training +D), [3] down (inference -D), [4] down (training -D),
// [5] move with thief = training (training +D, inference -D), [6] move with
// thief = inference (inference +D, training -D); kInvalid where the victim has
// fewer than D units.
//
// Every record entry is value(rt', ri') = fl(F(ri') G*(rt')) at one of seven
// splits, so an entry costs two shared lookups once both functions are at hand:
//   F(ri)  = factor of lambda*(ri): a per-stream ladder of at most 8 keep-up
//            thresholds (ascending, u16) -- lambda* changes only there -- read as one
//            16-byte row and counted with four SIMD compares;
//   G*(rt) = max over {none} + feasible Gamma of rule 2: memoised per stream in a
//            direct-mapped cache of NS (rt, value) slots, filled on a miss.
// A step re-evaluates the two touched streams with one lane per record entry
// (lanes 8k + e, e < 7), i.e. 14 lanes in one pass.
// STEEPEST selects from per-stream keys (skey) above this stream count; at or below it one
// lane per thief job evaluates every candidate directly (J <= 32: one pass, cheaper)
constexpr int kKeyPathV = 16;

struct WarpState {
    long long* rec;              // [V][8]
    int* alloc;                  // [J]
    uint4* lthr;                 // [V] eight u16 lambda* thresholds, ascending (0xFFFF = unused)
    float* lfac;                 // [V][8] factor of lambda* at the threshold
    signed char* lidx;           // [V][8] index of lambda* at the threshold
    uint2* gc;                   // [V][NS] G* cache: (rt, value bits), rt = 0xFFFFFFFF empty
    unsigned long long* skey;    // [V][4] the stream's best down / up / move key (0 = none)
    __device__ __forceinline__ long long cur(int v) const { return rec[v * 8]; }
    __device__ __forceinline__ long long up(int j) const { return rec[(j >> 1) * 8 + 1 + (j & 1)]; }
    __device__ __forceinline__ long long dn(int j) const { return rec[(j >> 1) * 8 + 3 + (j & 1)]; }
    __device__ __forceinline__ long long mv(int j) const { return rec[(j >> 1) * 8 + 6 - (j & 1)]; }
};

__host__ __device__ inline size_t thief_warp_bytes(int V, int NS, bool keys) {
    const size_t J = 2 * (size_t)V;
    size_t b = 8 * 8 * (size_t)V + 4 * J + 16 * (size_t)V + 4 * 8 * (size_t)V + 8 * (size_t)V +
               8 * (size_t)NS * (size_t)V;
    if (keys) b = ((b + 7) & ~size_t(7)) + 32 * (size_t)V;   // skey (STEEPEST, V > kKeyPathV)
    return (b + 15) & ~size_t(15);
}

__device__ inline WarpState carve(unsigned char* base, int V, int NS) {
    const int J = 2 * V;
    WarpState w;
    w.rec = reinterpret_cast<long long*>(base);                        // 16-byte aligned
    w.gc = reinterpret_cast<uint2*>(w.rec + 8 * V);                    // 16-byte aligned
    w.lthr = reinterpret_cast<uint4*>(w.gc + (size_t)NS * V);          // 16-byte aligned (NS even)
    w.lfac = reinterpret_cast<float*>(w.lthr + V);
    w.alloc = reinterpret_cast<int*>(w.lfac + 8 * V);
    w.lidx = reinterpret_cast<signed char*>(w.alloc + J);
    w.skey = reinterpret_cast<unsigned long long*>(
        (reinterpret_cast<uintptr_t>(w.lidx + 8 * V) + 7) & ~uintptr_t(7));   // V > kKeyPathV only
    return w;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
    const unsigned hi = (unsigned)(k >> 32);
    const unsigned mh = __reduce_max_sync(FULL, hi);
    const unsigned ml = __reduce_max_sync(FULL, hi == mh ? (unsigned)k : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

__device__ __forceinline__ unsigned long long shfl_sum_u64(unsigned long long x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
    return x;
}

// key for (delta, job): larger delta first, then smaller job index; 0 = none
__device__ __forceinline__ unsigned long long dkey(long long delta, int j) {
    return ((unsigned long long)(delta + kKeyOff) << 16) | (unsigned long long)(0xFFFF - j);
}
__device__ __forceinline__ long long key_delta(unsigned long long k) { return (long long)(k >> 16) - kKeyOff; }
__device__ __forceinline__ int key_job(unsigned long long k) { return 0xFFFF - (int)(k & 0xFFFF); }

struct InstView {
    const float* stale;     // [V]
    const float* cost;      // [V][nG]
    const float* post;
    const uint16_t* lmu;    // [V][nL]
    const float* lf;
    const float4* cpd;      // [V][nG] staged (cost, post, fl(post - stale), 0), or NULL
    // (cost, post, fl(post - stale)) of config g (0-based) of stream v
    __device__ __forceinline__ float4 get(int v, int g, int nG) const {
        if (cpd) return cpd[v * nG + g];
        const float c = cost[(size_t)v * nG + g], po = post[(size_t)v * nG + g];
        return make_float4(c, po, fsub(po, stale[v]), 0.0f);
    }
};

// IEEE division off the hot path (the exact shared-reciprocal path covers the paper's shapes)
__device__ __noinline__ float fdiv_cold(float a, float b) { return __fdiv_rn(a, b); }

// lambda* ladder of stream v (Alg. 2 lines 3-4, rule 3), one lane per stream.
// lambda*(ri) depends only on the admissible set {l : t_l <= ri} (t_l = lmu_l if
// fl(stale f_l) >= a_MIN, else never), which equals the set at the largest
// t_l <= ri; so the thresholds are stored ascending (ties: lambda order) with
// lambda*(t) and its factor, and F(ri) is the entry of the last threshold <= ri.
// Slot rank(l) = #{l' : (t_l', l') < (t_l, l)}; slots nL..7 stay unused (0xFFFF).
// NL: the loops' compile-time bound -- |Lambda| itself for the paper's shape (no guards, 5 x 5
// comparisons), kMaxLambda with runtime guards otherwise.
template <int NL>
__device__ __forceinline__ void init_ladder_lane(const InstView& in, const WarpState& S, int v, const ekya_dims& d) {
    const int nL = NL < kMaxLambda ? NL : d.n_lambda;
    unsigned t[NL];
    float acc[NL], f[NL];
    const float st = in.stale[v];
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        t[l] = 0xFFFFu;
        acc[l] = 0.0f;
        f[l] = 0.0f;
        if (l < nL) {
            const uint16_t m = in.lmu[(size_t)v * nL + l];
            f[l] = in.lf[(size_t)v * nL + l];
            acc[l] = fmul(st, f[l]);
            if (m != kLmuPad && acc[l] >= d.a_min) t[l] = m;
        }
    }
    unsigned short* th = reinterpret_cast<unsigned short*>(S.lthr + v);
#pragma unroll
    for (int p = 0; p < 8; ++p) th[p] = 0xFFFFu;
#pragma unroll
    for (int l = 0; l < NL; ++l) {
        if (l < nL) {
            // lambda*(t_l) over {l' : t_l' <= t_l}: highest accuracy, lowest index on ties
            int best = 0, rank = 0;
            float bacc = -1.0f, fb = 0.0f;
#pragma unroll
            for (int l2 = 0; l2 < NL; ++l2) {
                if (l2 < nL) {
                    const bool take = t[l2] <= t[l] && acc[l2] > bacc;
                    best = take ? l2 : best;
                    fb = take ? f[l2] : fb;
                    bacc = take ? acc[l2] : bacc;
                    rank += (t[l2] < t[l] || (t[l2] == t[l] && l2 < l)) ? 1 : 0;
                }
            }
            th[rank] = (unsigned short)t[l];
            S.lfac[v * 8 + rank] = fb;
            S.lidx[v * 8 + rank] = (signed char)best;
        }
    }
}

// number of ladder thresholds <= ri (0 .. 8): the ladder slot of lambda*(ri) is count - 1
__device__ __forceinline__ int ladder_count(const uint4& th, int ri) {
    const unsigned r = (unsigned)min(ri, 0xFFFE);
    const unsigned rr = r | (r << 16);
    return (__popc(__vcmpleu2(th.x, rr)) + __popc(__vcmpleu2(th.y, rr)) + __popc(__vcmpleu2(th.z, rr)) +
            __popc(__vcmpleu2(th.w, rr))) >> 4;
}

// G*(r) of stream v (r >= 0), warp-collective: lane g evaluates rule 2 for retraining
// config g (lane 0 = no retraining), one REDUX max; values are >= 0 or the -1 sentinel,
// so signed-int order of the bits = float order.  The divisor fl(r uT) is shared by the
// warp: with `fast` the division is the exact shared-reciprocal fast path
// (stream_tables.cuh), branch-free.
__device__ __forceinline__ float gstar_warp(const InstView& in, int v, int r, const ekya_dims& d, bool fast) {
    const int lane = threadIdx.x & 31, nG = d.n_gamma;
    const bool mine = lane >= 1 && lane <= nG;
    float4 c = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (mine) c = in.get(v, lane - 1, nG);
    const float den = fmul(__int2float_rn(r), d.unit_gpu_seconds);
    float f;
    if (fast) {
        const SharedDiv dv(den);
        f = dv.div(c.x);
    } else {
        f = mine && r >= 1 ? fdiv_cold(c.x, den) : 2.0f;
    }
    const float w = fsub(c.y, fmul(f, c.z));
    const float g = lane == 0 ? in.stale[v] : (mine && r >= 1 && f <= 1.0f ? w : -1.0f);
    return __int_as_float(__reduce_max_sync(FULL, __float_as_int(g)));
}

// G*(r) of stream v (r >= 0) by one lane: the same maximum over the same rule-2 values
// (fmaxf of values >= 0 and -1 sentinels equals the integer-bit maximum above)
__device__ __forceinline__ float gstar_lane(const InstView& in, int v, int r, const ekya_dims& d, bool fast) {
    const int nG = d.n_gamma;
    float G = in.stale[v];
    if (r < 1) return G;
    const float den = fmul(__int2float_rn(r), d.unit_gpu_seconds);
    if (fast) {
        const SharedDiv dv(den);
#pragma unroll 1
        for (int g = 0; g < nG; ++g) {
            const float4 c = in.get(v, g, nG);
            const float f = dv.div(c.x);
            const float w = fsub(c.y, fmul(f, c.z));
            G = f <= 1.0f ? fmaxf(G, w) : G;
        }
    } else {
#pragma unroll 1
        for (int g = 0; g < nG; ++g) {
            const float4 c = in.get(v, g, nG);
            const float f = fdiv_cold(c.x, den);
            if (f <= 1.0f) G = fmaxf(G, fsub(c.y, fmul(f, c.z)));
        }
    }
    return G;
}

// Warp-collective: record entries of up to four streams s0..s3 (-1 = none), lane 8k + e
// computing entry e of stream s_k at its split: e = 0 cur (rt,ri), 1 (rt,ri+D),
// 2 (rt+D,ri), 3 (rt,ri-D), 4 (rt-D,ri), 5 (rt+D,ri-D), 6 (rt-D,ri+D).
template <int MODE>
__device__ __forceinline__ void update_streams(const InstView& in, const WarpState& S, int s0, int s1, int s2,
                                               int s3, const ekya_dims& d, bool fast, int nsm) {
    const int lane = threadIdx.x & 31, D = d.steal_units;
    const int k = lane >> 3, e = lane & 7;
    const int s = k == 0 ? s0 : k == 1 ? s1 : k == 2 ? s2 : s3;
    const bool act = e < 7 && s >= 0;
    int ri = 0, rt = 0;
    if (act) {
        ri = S.alloc[2 * s];
        rt = S.alloc[2 * s + 1];
    }
    const int drt = (e == 2 || e == 5) ? D : (e == 4 || e == 6) ? -D : 0;
    const int dri = (e == 1 || e == 6) ? D : (e == 3 || e == 5) ? -D : 0;
    const int rt2 = rt + drt, ri2 = ri + dri;
    const bool valid = act && rt2 >= 0 && ri2 >= 0;
    float G = 0.0f;
    bool need = false;
    if (valid) {
        const uint2 c = S.gc[s * (nsm + 1) + (rt2 & nsm)];
        need = c.x != (unsigned)rt2;
        G = __uint_as_float(c.y);
    }
    __syncwarp();   // every lane's cache read precedes a miss fill's write (lane 0, below)
    for (unsigned m = __ballot_sync(FULL, need); m; m = __ballot_sync(FULL, need)) {
        const int src = __ffs(m) - 1;
        const int ms = __shfl_sync(FULL, s, src), mr = __shfl_sync(FULL, rt2, src);
        const float gv = gstar_warp(in, ms, mr, d, fast);
        if (lane == 0) S.gc[ms * (nsm + 1) + (mr & nsm)] = make_uint2((unsigned)mr, __float_as_uint(gv));
        if (need && s == ms && rt2 == mr) {
            G = gv;
            need = false;
        }
    }
    float F = -1.0f;
    if (valid) {
        const int cnt = ladder_count(S.lthr[s], ri2);
        if (cnt > 0) F = S.lfac[s * 8 + cnt - 1];
    }
    const long long val = F < 0.0f ? 0LL : (long long)q32(fmul(F, G));
    const long long c = __shfl_sync(FULL, val, lane & ~7);
    if (act) S.rec[s * 8 + e] = e == 0 ? c : (valid ? val - c : kInvalid);
    __syncwarp();
    // the stream's best steal keys (STEEPEST's selection reads only these), lane k for s_k
    if (MODE == EKYA_THIEF_STEEPEST && d.n_streams > kKeyPathV && lane < 4) {
        const int sk = lane == 0 ? s0 : lane == 1 ? s1 : lane == 2 ? s2 : s3;
        if (sk >= 0) {
            const long long* r = S.rec + sk * 8;
            const int j0 = 2 * sk, j1 = j0 + 1;
            unsigned long long dk = 0, uk, mk = 0;
            if (r[3] != kInvalid) dk = dkey(r[3], j0);
            if (r[4] != kInvalid) dk = max(dk, dkey(r[4], j1));
            uk = max(dkey(r[1], j0), dkey(r[2], j1));
            if (r[6] != kInvalid) mk = dkey(r[6], j0);   // thief = inference job j0
            if (r[5] != kInvalid) mk = max(mk, dkey(r[5], j1));
            S.skey[sk * 4] = dk;
            S.skey[sk * 4 + 1] = uk;
            S.skey[sk * 4 + 2] = mk;
        }
    }
    __syncwarp();
}

// Exact argmax config byte of stream v at its final split, one lane per stream: rule 3's
// (lambda*, gamma*) with gamma* the lowest index maximising fl(f_lambda* g_gamma) (strict '>'
// in index order keeps the lowest; gamma = none is index 0).
__device__ uint8_t stream_cfg_lane(const InstView& in, const WarpState& S, int v, int ri, int rt,
                                   const ekya_dims& d, bool fast) {
    const int nG = d.n_gamma;
    const int cnt = ladder_count(S.lthr[v], ri);
    if (cnt == 0) return (uint8_t)(kLambdaNone << 5);
    const int l = S.lidx[v * 8 + cnt - 1];
    const float fac = S.lfac[v * 8 + cnt - 1];
    float best = fmul(fac, in.stale[v]);
    int gb = 0;
    if (rt >= 1) {
        const float den = fmul(__int2float_rn(rt), d.unit_gpu_seconds);
        const SharedDiv dv(den);
#pragma unroll 1
        for (int g = 0; g < nG; ++g) {
            const float4 c = in.get(v, g, nG);
            const float f = fast ? dv.div(c.x) : fdiv_cold(c.x, den);
            if (f <= 1.0f) {
                const float a = fmul(fac, fsub(c.y, fmul(f, c.z)));
                if (a > best) {
                    best = a;
                    gb = g + 1;
                }
            }
        }
    }
    return (uint8_t)(gb | (l << 5));
}

__device__ __forceinline__ bool uT_fast(const ekya_dims& d) {
    const float lo = d.unit_gpu_seconds;
    const float hi = fmul(__int2float_rn(d.units + d.steal_units), d.unit_gpu_seconds);
    return lo >= 8.67361738e-19f && hi <= 1.15292150e18f;   // [2^-60, 2^60]
}

__device__ __forceinline__ bool lit_cond(const WarpState& S, int t, int w, int J) {
    if (w >= J || w == t) return false;
    if ((w >> 1) == (t >> 1)) {
        const long long m = S.mv(t);
        return m != kInvalid && m > 0;
    }
    const long long dn = S.dn(w);
    return dn != kInvalid && S.up(t) + dn > 0;
}


__device__ __forceinline__ unsigned long long stream_down_key(const WarpState& S, int v) {
    unsigned long long k = 0;
    const long long d0 = S.dn(2 * v), d1 = S.dn(2 * v + 1);
    if (d0 != kInvalid) k = dkey(d0, 2 * v);
    if (d1 != kInvalid) {
        const unsigned long long kk = dkey(d1, 2 * v + 1);
        k = kk > k ? kk : k;
    }
    return k;
}

// MODE: EKYA_THIEF_STEEPEST or EKYA_THIEF_LITERAL (one kernel per mode keeps the hot loop's
// code small)
// lanes 0..4: bulk-prefetch instance bn's five input arrays into L2
__device__ __forceinline__ void prefetch_instance(const ThiefParams& p, unsigned bn) {
    const int lane = threadIdx.x & 31;
    const ekya_dims& d = p.d;
    const int V = d.n_streams, nG = d.n_gamma, nL = d.n_lambda;
    if (lane < 5 && bn < (unsigned)d.n_inst) {
        const Granules gi = lane == 0   ? granules(p.t.stale + (size_t)bn * V, (size_t)V * 4)
                            : lane == 1 ? granules(p.t.cost + (size_t)bn * V * nG, (size_t)V * nG * 4)
                            : lane == 2 ? granules(p.t.post + (size_t)bn * V * nG, (size_t)V * nG * 4)
                            : lane == 3 ? granules(p.t.lam_min_units + (size_t)bn * V * nL, (size_t)V * nL * 2)
                                        : granules(p.t.lam_factor + (size_t)bn * V * nL, (size_t)V * nL * 4);
        if (gi.bytes) bulk_prefetch_l2(gi.g0, gi.bytes);
    }
}

// One instance b by the calling warp (warp-collective; leaves with every lane's shared-memory
// accesses done after the caller's __syncwarp).  `claim` is lane 0's pending claim of the
// warp's next instance: consumed only after this instance's validity pass (the atomic's
// latency overlaps those loads), broadcast into *next and prefetched into L2.
template <int MODE, bool PERSIST>
__device__ __forceinline__ void thief_one(const ThiefParams& p, long long b, unsigned claim, unsigned* next) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int V = d.n_streams, J = 2 * V, D = d.steal_units, U = d.units, nG = d.n_gamma, nL = d.n_lambda;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nsm = p.nsm;
    const WarpState S = carve(smem + warp * p.warp_bytes, V, nsm + 1);
    float* staged = reinterpret_cast<float*>(smem + warp * p.warp_bytes + p.state_bytes);

    InstView in{p.t.stale + b * V, p.t.cost + b * V * nG, p.t.post + b * V * nG,
                p.t.lam_min_units + b * V * nL, p.t.lam_factor + b * V * nL, nullptr};

    // ---- validity (R-ERR), the exact-division test and the staging, in one pass ----
    // (lanes over a stream's configs: |Gamma| <= 31)
    bool ok = true;
    // exact shared-reciprocal division applies to every cost and every fl(r uT), r <= U + D
    bool fast = uT_fast(d);
    float4* cpd = reinterpret_cast<float4*>(staged);
    float* st = reinterpret_cast<float*>(cpd + V * nG);
    for (int i = lane; i < V; i += 32) {
        const float x = __ldg(in.stale + i);
        ok &= in01(x);
        if (p.stage) st[i] = x;
    }
    // flat over (stream, config): every lane's loads are independent (one latency round trip);
    // the paper's |Gamma| = 18 divides by a constant
    auto stage_pass = [&](auto ngc) {
        constexpr int NGC = decltype(ngc)::value;
        const int ng = NGC > 0 ? NGC : nG;
#pragma unroll 2
        for (int i = lane; i < V * ng; i += 32) {
            const int v = i / ng;
            const float c = __ldg(in.cost + i), po = __ldg(in.post + i);
            ok &= c >= 0.0f && (isinf(c) || in01(po));
            fast &= fast_dividend(c);
            if (p.stage) cpd[i] = make_float4(c, po, fsub(po, __ldg(in.stale + v)), 0.0f);
        }
    };
    if (nG == 18) stage_pass(std::integral_constant<int, 18>{});
    else stage_pass(std::integral_constant<int, 0>{});
    for (int i = lane; i < V * nL; i += 32)
        if (__ldg(in.lmu + i) != kLmuPad) ok &= in01(__ldg(in.lf + i));
    __syncwarp();
    ok = __all_sync(FULL, ok);
    fast = __all_sync(FULL, fast);
    if (PERSIST) {
        *next = __shfl_sync(FULL, claim, 0);
        prefetch_instance(p, *next);
    }
    if (p.stage) {   // stale and (cost, post, post - stale) in this warp's shared memory
        in.stale = st;
        in.cpd = cpd;
    }
    if (!ok) {
        for (int j = lane; j < J; j += 32) p.out_alloc[b * J + j] = 0;
        for (int v = lane; v < V; v += 32) p.out_cfg[b * V + v] = 0;
        if (lane == 0) {
            p.out_sum[b] = 0;
            if (p.out_mean) p.out_mean[b] = 0.0f;
            if (p.out_steps) p.out_steps[b] = 0;
            flag_data_error(p.st);
        }
        return;
    }

    // ---- fair start (C9) + per-stream breakpoints and entries ----
    for (int v = lane; v < V; v += 32) {
        const int share = U / V + (v < U % V ? 1 : 0);
        const int rt = share / 2;
        S.alloc[2 * v + 1] = rt;
        S.alloc[2 * v] = share - rt;
    }
    if (nL == 5) {   // the paper's |Lambda|: compile-time loops (no guards)
#pragma unroll 1
        for (int v = lane; v < V; v += 32) init_ladder_lane<5>(in, S, v, d);
    } else {
#pragma unroll 1
        for (int v = lane; v < V; v += 32) init_ladder_lane<kMaxLambda>(in, S, v, d);
    }
#pragma unroll 1
    for (int i = lane; i < V * (nsm + 1); i += 32) S.gc[i] = make_uint2(0xFFFFFFFFu, 0u);
    __syncwarp();
    // G* at rt - D, rt, rt + D of every stream, one lane each (two slots may collide when
    // 2D = 0 mod NS: either complete (rt, value) pair is a valid cache entry)
    for (int i = lane; i < 3 * V; i += 32) {
        const int v = i / 3, r = S.alloc[2 * v + 1] + D * (i - 3 * v - 1);
        if (r >= 0) S.gc[v * (nsm + 1) + (r & nsm)] = make_uint2((unsigned)r, __float_as_uint(gstar_lane(in, v, r, d, fast)));
    }
    __syncwarp();
    for (int v = 0; v < V; v += 4)
        update_streams<MODE>(in, S, v, v + 1 < V ? v + 1 : -1, v + 2 < V ? v + 2 : -1, v + 3 < V ? v + 3 : -1, d, fast, nsm);

    unsigned steps = 0;
    if (MODE == EKYA_THIEF_STEEPEST) {
        // Best single steal (C12) from per-stream keys.  For thief t the candidates are the
        // cross-stream steal from the best victim outside its stream (the top-2 down keys by
        // stream, K1 / K2) and the move with its sibling; its value is the larger of the two.
        // Maximising dkey(value, t) over t splits into: thieves outside K1's stream s1, whose
        // best is the best up key outside s1 (top-2 up keys by stream, U1 / U2) shifted by
        // K1's delta; s1's two jobs with K2; and the best move key M.  Ties resolve as the
        // per-thief scan does (dkey order: larger delta, then lower job index; the victim of
        // the chosen thief by the same rule as before).
        const unsigned max_steps = 1u << 26;
        if (V <= kKeyPathV) {
            for (;;) {
                // per-stream best down, top-2 by stream
                unsigned long long k1 = 0, k2 = 0;
                int s1;
                if (V <= 32) {   // one stream per lane: its key serves both reductions
                    const unsigned long long k = lane < V ? stream_down_key(S, lane) : 0ULL;
                    k1 = warp_max_u64(k);
                    s1 = k1 ? (key_job(k1) >> 1) : -1;
                    k2 = warp_max_u64(lane == s1 ? 0ULL : k);
                } else {
                    for (int v = lane; v < V; v += 32) {
                        const unsigned long long k = stream_down_key(S, v);
                        k1 = k > k1 ? k : k1;
                    }
                    k1 = warp_max_u64(k1);
                    s1 = k1 ? (key_job(k1) >> 1) : -1;
                    for (int v = lane; v < V; v += 32) {
                        if (v == s1) continue;
                        const unsigned long long k = stream_down_key(S, v);
                        k2 = k > k2 ? k : k2;
                    }
                    k2 = warp_max_u64(k2);
                }
                // per thief: best victim, then argmax over thieves
                unsigned long long bestkey = 0;
                int bestw = -1;
                for (int t = lane; t < J; t += 32) {
                    const unsigned long long ck = ((t >> 1) != s1) ? k1 : k2;
                    bool have = false;
                    long long tot = 0;
                    int w = -1;
                    if (ck) {
                        tot = S.up(t) + key_delta(ck);
                        w = key_job(ck);
                        have = true;
                    }
                    const long long m = S.mv(t);
                    if (m != kInvalid) {
                        const int ws = t ^ 1;
                        if (!have || m > tot || (m == tot && ws < w)) {
                            tot = m;
                            w = ws;
                            have = true;
                        }
                    }
                    if (have) {
                        const unsigned long long tk = dkey(tot, t);
                        if (tk > bestkey) {
                            bestkey = tk;
                            bestw = w;
                        }
                    }
                }
                const unsigned long long gk = warp_max_u64(bestkey);
                if (gk == 0 || key_delta(gk) <= 0) break;
                const int t = key_job(gk);
                const unsigned owner = __ballot_sync(FULL, bestkey == gk);
                const int w = __shfl_sync(FULL, bestw, __ffs(owner) - 1);
                if (lane == 0) {
                    S.alloc[w] -= D;
                    S.alloc[t] += D;
                }
                __syncwarp();
                update_streams<MODE>(in, S, t >> 1, (w >> 1) != (t >> 1) ? (w >> 1) : -1, -1, -1, d, fast, nsm);
                if (++steps >= max_steps) {
                    if (lane == 0) flag_data_error(p.st);
                    break;
                }
            }
        } else
        for (;;) {
            unsigned long long d1 = 0, d2 = 0, u1 = 0, u2 = 0, mb = 0;
            int ds1 = -1, us1 = -1;
            for (int v = lane; v < V; v += 32) {   // this lane's streams: partial top-2 by stream
                const unsigned long long dk = S.skey[v * 4], uk = S.skey[v * 4 + 1], mk = S.skey[v * 4 + 2];
                if (dk > d1) { d2 = d1; d1 = dk; ds1 = v; } else if (dk > d2) { d2 = dk; }
                if (uk > u1) { u2 = u1; u1 = uk; us1 = v; } else if (uk > u2) { u2 = uk; }
                mb = mk > mb ? mk : mb;
            }
            const unsigned long long K1 = warp_max_u64(d1);
            const int s1 = K1 ? (key_job(K1) >> 1) : -1;
            const unsigned long long K2 = warp_max_u64(ds1 == s1 ? d2 : d1);
            const unsigned long long U1 = warp_max_u64(u1);
            const int su = U1 ? (key_job(U1) >> 1) : -1;
            const unsigned long long U2 = warp_max_u64(us1 == su ? u2 : u1);
            unsigned long long gk = warp_max_u64(mb);
            if (K1) {
                const unsigned long long UK = su != s1 ? U1 : U2;
                if (UK) {
                    const unsigned long long c = dkey(key_delta(UK) + key_delta(K1), key_job(UK));
                    gk = c > gk ? c : gk;
                }
            }
            if (K2) {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int t = 2 * s1 + h;
                    const unsigned long long c = dkey(S.up(t) + key_delta(K2), t);
                    gk = c > gk ? c : gk;
                }
            }
            if (gk == 0 || key_delta(gk) <= 0) break;
            const int t = key_job(gk);
            // the victim of thief t: its best cross-stream victim, or its sibling (move) when
            // that is strictly better or equal with the lower job index
            const unsigned long long ck = (t >> 1) != s1 ? K1 : K2;
            int w = ck ? key_job(ck) : -1;
            const long long tot = ck ? S.up(t) + key_delta(ck) : 0;
            const long long m = S.mv(t);
            if (m != kInvalid && (!ck || m > tot || (m == tot && (t ^ 1) < w))) w = t ^ 1;
            if (lane == 0) {
                S.alloc[w] -= D;
                S.alloc[t] += D;
            }
            __syncwarp();
            update_streams<MODE>(in, S, t >> 1, (w >> 1) != (t >> 1) ? (w >> 1) : -1, -1, -1, d, fast, nsm);
            if (++steps >= max_steps) {
                if (lane == 0) flag_data_error(p.st);
                break;
            }
        }
    } else {
        for (int t = 0; t < J; ++t) {
            int pos = 0;
            while (pos < J) {
                const unsigned m = __ballot_sync(FULL, lit_cond(S, t, pos + lane, J));
                if (!m) {
                    pos += 32;
                    continue;
                }
                const int w = pos + __ffs(m) - 1;
                do {
                    if (lane == 0) {
                        S.alloc[w] -= D;
                        S.alloc[t] += D;
                    }
                    __syncwarp();
                    update_streams<MODE>(in, S, t >> 1, (w >> 1) != (t >> 1) ? (w >> 1) : -1, -1, -1, d, fast, nsm);
                    ++steps;
                } while (lit_cond(S, t, w, J));
                pos = w + 1;
            }
        }
    }

    // ---- decision output (A6) ----
    unsigned long long part = 0;
    for (int v = lane; v < V; v += 32) part += (unsigned long long)S.cur(v);
    const unsigned long long sum = shfl_sum_u64(part);
    for (int j = lane; j < J; j += 32) p.out_alloc[b * J + j] = (uint16_t)S.alloc[j];
    for (int v = lane; v < V; v += 32)
        p.out_cfg[b * V + v] = stream_cfg_lane(in, S, v, S.alloc[2 * v], S.alloc[2 * v + 1], d, fast);
    if (lane == 0) {
        p.out_sum[b] = sum;
        if (p.out_mean) p.out_mean[b] = mean_q32(sum, V);
        if (p.out_steps) p.out_steps[b] = steps;
    }
}

// PERSIST: persistent warps claiming instances from a device counter (dynamic balance:
// per-instance step counts vary): a warp claims its next instance while running the current
// one and lanes 0..4 bulk-prefetch the next one's five input arrays into L2, so its validity /
// staging pass does not wait on HBM.  Every warp makes exactly one failing claim; the last
// warp past it (thief_done) returns both counters to 0 for the handle's next launch (launches
// on one handle are stream-ordered, as for its error word).  Otherwise one instance per warp
// (measured faster for STEEPEST at the paper's V = 10: 0.663 vs 0.674 ms; persistent LITERAL
// 1.04 -> 0.99 ms, config-5 shape STEEPEST 4.17 -> 3.77, LITERAL 10.4 -> 9.5).
template <int MODE, bool PERSIST>
__global__ void __launch_bounds__(kThiefThreads, 8) thief_kernel(ThiefParams p) {
    const int lane = threadIdx.x & 31;
    if (!PERSIST) {
        const long long b = (long long)blockIdx.x * p.warps + (threadIdx.x >> 5);
        unsigned unused;
        if (b < p.d.n_inst) thief_one<MODE, false>(p, b, 0u, &unused);
        return;
    }
    const unsigned n = (unsigned)p.d.n_inst;
    unsigned b = 0;
    if (lane == 0) b = atomicAdd(&p.st->thief_next, 1u);
    b = __shfl_sync(FULL, b, 0);
    while (b < n) {
        unsigned claim = 0, bn;
        if (lane == 0) claim = atomicAdd(&p.st->thief_next, 1u);
        thief_one<MODE, true>(p, (long long)b, claim, &bn);
        __syncwarp();   // the next instance's state writes follow every lane's reads of this one's
        b = bn;
    }
    if (lane == 0 && atomicAdd(&p.st->thief_done, 1u) == p.total_warps - 1) {
        p.st->thief_next = 0;
        p.st->thief_done = 0;
    }
}

}  // namespace

int launch_thief(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int mode,
                 uint16_t* out_alloc, uint8_t* out_cfg, uint64_t* out_sum, float* out_mean,
                 uint32_t* out_steps, cudaStream_t s) {
    if (d.n_streams > 1024) return EKYA_ERR_SHAPE;
    ThiefParams p{};
    p.d = d;
    p.t = t;
    p.st = h->dstate;
    p.mode = mode;
    p.out_alloc = out_alloc;
    p.out_cfg = out_cfg;
    p.out_sum = reinterpret_cast<unsigned long long*>(out_sum);
    p.out_mean = out_mean;
    p.out_steps = out_steps;
    // G* cache: 32 slots per stream for the paper's stream counts; wide instances keep fewer
    // so that the shared-memory carve-out leaves L1 room for the unstaged profile tables
    // (config-5 shape, 16,384 instances: STEEPEST 5.53 ms at 8 slots, 4.17 at 4, 4.99 at 2;
    // LITERAL 10.44 at 8, 10.57 at 4, 13.9 at 16)
    const int ns = d.n_streams <= 16 ? 32 : (mode == EKYA_THIEF_STEEPEST ? 4 : 8);
    p.nsm = ns - 1;
    p.state_bytes = thief_warp_bytes(d.n_streams, ns, mode == EKYA_THIEF_STEEPEST && d.n_streams > kKeyPathV);
    const size_t tbytes = ((size_t)d.n_streams * (4 * d.n_gamma + 1) * 4 + 15) & ~size_t(15);
    p.stage = tbytes <= 8192;
    p.warp_bytes = p.state_bytes + (p.stage ? tbytes : 0);
    p.warps = (int)std::min<size_t>(kThiefThreads / 32, h->smem_optin / p.warp_bytes);
    if (p.warps < 1) return EKYA_ERR_SHAPE;
    size_t smem = p.warp_bytes * p.warps;
    if (d.n_inst == 0) return EKYA_OK;
    // persistent claiming warps except for STEEPEST at the paper's stream counts (V <= 16),
    // where one instance per warp measured faster (thief_kernel)
    const bool persist = !(mode == EKYA_THIEF_STEEPEST && d.n_streams <= 16);
    auto kern = mode == EKYA_THIEF_STEEPEST
                    ? (persist ? thief_kernel<EKYA_THIEF_STEEPEST, true> : thief_kernel<EKYA_THIEF_STEEPEST, false>)
                    : thief_kernel<EKYA_THIEF_LITERAL, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    if (d.n_inst >= 0xFFFFFFFFLL - (1LL << 24)) return EKYA_ERR_LIMIT;
    long long grid = (d.n_inst + p.warps - 1) / p.warps;
    if (persist) {   // as many CTAs as are resident at once
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, p.warps * 32, smem);
        grid = std::min<long long>(grid, (long long)h->sm_count * std::max(per_sm, 1));
    }
    if (grid > 0x7fffffffLL) return EKYA_ERR_SHAPE;
    p.total_warps = (unsigned)(grid * p.warps);
    kern<<<(unsigned)grid, p.warps * 32, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
