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
#include <climits>

#include "launch.h"
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
};

// Per-stream record rec[v][8] (Q32 units): [0] current value, [1] up (inference
// +D), [2] up (training +D), [3] down (inference -D), [4] down (training -D),
// [5] move with thief = training (training +D, inference -D), [6] move with
// thief = inference (inference +D, training -D); kInvalid where the victim has
// fewer than D units.
struct WarpState {
    long long* rec;              // [V][8]
    int* alloc;                  // [J]
    int* lthr;                   // [V][8] lambda* breakpoints, ascending (INT_MAX = unused)
    float* lfac;                 // [V][8] factor of lambda* at the breakpoint
    int* lidx;                   // [V][8] index of lambda* at the breakpoint
    float* gc;                   // [V][4] G*(rt-D), G*(rt), G*(rt+D) cached for rt = grt[v]
    int* grt;                    // [V]    (-1 = empty)
    __device__ __forceinline__ long long cur(int v) const { return rec[v * 8]; }
    __device__ __forceinline__ long long up(int j) const { return rec[(j >> 1) * 8 + 1 + (j & 1)]; }
    __device__ __forceinline__ long long dn(int j) const { return rec[(j >> 1) * 8 + 3 + (j & 1)]; }
    __device__ __forceinline__ long long mv(int j) const { return rec[(j >> 1) * 8 + 6 - (j & 1)]; }
};

__host__ __device__ inline size_t thief_warp_bytes(int V) {
    const size_t J = 2 * (size_t)V;
    size_t b = 8 * 8 * (size_t)V + 4 * J + 3 * 4 * 8 * (size_t)V + 4 * 4 * (size_t)V + 4 * (size_t)V;
    return (b + 15) & ~size_t(15);
}

__device__ inline WarpState carve(unsigned char* base, int V) {
    const int J = 2 * V;
    WarpState w;
    w.rec = reinterpret_cast<long long*>(base);
    w.alloc = reinterpret_cast<int*>(w.rec + 8 * V);
    w.lthr = w.alloc + J;
    w.lfac = reinterpret_cast<float*>(w.lthr + 8 * V);
    w.lidx = reinterpret_cast<int*>(w.lfac + 8 * V);
    w.gc = reinterpret_cast<float*>(w.lidx + 8 * V);
    w.grt = reinterpret_cast<int*>(w.gc + 4 * V);
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

// Warp-collective, once per stream: lambda* ladder (Alg. 2 lines 3-4, rule 3).
// lambda*(ri) depends only on the admissible set {l : t_l <= ri} (t_l = lmu_l if
// fl(stale f_l) >= a_MIN, else never), which equals the set at the largest
// t_l <= ri; so the thresholds are stored ascending (ties: lambda order) with
// lambda*(t) and its factor, and a lookup is one ballot over lanes 0..7: the
// lanes with t <= ri form a prefix and its last lane holds lambda*(ri).
__device__ void init_ladder(const InstView& in, const WarpState& S, int v, const ekya_dims& d) {
    const int lane = threadIdx.x & 31, nL = d.n_lambda;
    int t = INT_MAX;
    float acc = 0.0f, f = 0.0f;
    if (lane < nL) {
        const uint16_t m = in.lmu[(size_t)v * nL + lane];
        f = in.lf[(size_t)v * nL + lane];
        acc = fmul(in.stale[v], f);
        if (m != kLmuPad && acc >= d.a_min) t = m;
    }
    // lambda*(t) over {l : t_l <= t}: highest accuracy, lowest index on ties
    int best = -1, rank = 0;
    float bacc = 0.0f;
    for (int l = 0; l < nL; ++l) {
        const int tl = __shfl_sync(FULL, t, l);
        const float al = __shfl_sync(FULL, acc, l);
        if (tl <= t && (best < 0 || al > bacc)) {
            best = l;
            bacc = al;
        }
        rank += (tl < t || (tl == t && l < lane)) ? 1 : 0;
    }
    const float fb = __shfl_sync(FULL, f, best < 0 ? 0 : best);
    if (lane < 8) {
        // unused / inadmissible lambdas sort last (t = INT_MAX) and are never reached
        const int pos = lane < nL ? rank : lane;
        S.lthr[v * 8 + pos] = t;
        S.lfac[v * 8 + pos] = fb;
        S.lidx[v * 8 + pos] = best;
    }
}

// lambda* ladder lookup of stream v at ri: slot of lambda*(ri) in the ladder, -1 if none
__device__ __forceinline__ int ladder_slot(int tk, int ri) {
    const unsigned m = __ballot_sync(FULL, (threadIdx.x & 31) < 8 && tk <= ri);
    return 31 - __clz(m);   // -1 when m == 0
}

// Warp-collective update of stream v's entries in the state arrays.
__device__ __forceinline__ void update_stream(const InstView& in, const WarpState& S, int v, const ekya_dims& d,
                                              bool fast) {
    const int lane = threadIdx.x & 31;
    const int D = d.steal_units, nG = d.n_gamma;
    const int ri = S.alloc[2 * v], rt = S.alloc[2 * v + 1];
    const float stale = in.stale[v];
    float cost = 0.0f, post = 0.0f, diff = 0.0f;
    if (lane >= 1 && lane <= nG) {
        const float4 c = in.get(v, lane - 1, nG);
        cost = c.x;
        post = c.y;
        diff = c.z;
    }
    const int tk = lane < 8 ? S.lthr[v * 8 + lane] : INT_MAX;
    const float fk = lane < 8 ? S.lfac[v * 8 + lane] : -1.0f;
    const bool mine = lane >= 1 && lane <= nG;
    // G*(r): lane g evaluates rule 2 for config g, REDUX max; values are >= 0 or
    // the -1 sentinel, so signed-int order of the bits = float order.  The divisor
    // fl(r uT) is shared by the warp: with `fast` the division is the exact
    // shared-reciprocal fast path (stream_tables.cuh), branch-free.
    auto gstar = [&](int r) -> float {
        const float den = fmul(__int2float_rn(r), d.unit_gpu_seconds);
        float f;
        if (fast) {
            const SharedDiv dv(den);
            f = dv.div(cost);
        } else {
            f = mine && r >= 1 ? fdiv(cost, den) : 2.0f;
        }
        const float w = fsub(post, fmul(f, diff));
        const float g = lane == 0 ? stale : (mine && r >= 1 && f <= 1.0f ? w : -1.0f);
        const int m = __reduce_max_sync(FULL, __float_as_int(g));
        return r < 0 ? -1.0f : __int_as_float(m);
    };
    // G* at rt-D, rt, rt+D, reusing the stream's cached values when rt moved by D
    const int crt = S.grt[v];
    float G[3];
    if (crt == rt) {
        G[0] = S.gc[v * 4]; G[1] = S.gc[v * 4 + 1]; G[2] = S.gc[v * 4 + 2];
    } else if (crt >= 0 && crt == rt - D) {
        G[0] = S.gc[v * 4 + 1]; G[1] = S.gc[v * 4 + 2]; G[2] = gstar(rt + D);
    } else if (crt >= 0 && crt == rt + D) {
        G[2] = S.gc[v * 4 + 1]; G[1] = S.gc[v * 4]; G[0] = gstar(rt - D);
    } else {
        G[0] = gstar(rt - D); G[1] = gstar(rt); G[2] = gstar(rt + D);
    }
    float fac[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int ri2 = ri + D * (k - 1);
        const int sl = ladder_slot(tk, ri2);   // ri2 < 0 never reaches a threshold (t >= 0)
        const float f = __shfl_sync(FULL, fk, sl < 0 ? 0 : sl);
        fac[k] = sl >= 0 ? f : -1.0f;
    }
    __syncwarp();
    if (lane == 0) {
        S.gc[v * 4] = G[0]; S.gc[v * 4 + 1] = G[1]; S.gc[v * 4 + 2] = G[2];
        S.grt[v] = rt;
    }
    // lanes 0..6 each produce one of the seven record entries, no divergence:
    // lane: 0 cur (rt,ri) 1 (rt,ri+D) 2 (rt+D,ri) 3 (rt,ri-D) 4 (rt-D,ri) 5 (rt+D,ri-D) 6 (rt-D,ri+D)
    const float Ga = (lane == 2 || lane == 5) ? G[2] : (lane == 4 || lane == 6) ? G[0] : G[1];
    const float fb = (lane == 1 || lane == 6) ? fac[2] : (lane == 3 || lane == 5) ? fac[0] : fac[1];
    const long long val = fb < 0.0f ? 0LL : (long long)q32(fmul(fb, Ga));
    const long long c = fac[1] < 0.0f ? 0LL : (long long)q32(fmul(fac[1], G[1]));
    const bool valid = (lane == 3 || lane == 5) ? ri >= D : (lane == 4 || lane == 6) ? rt >= D : true;
    const long long out = lane == 0 ? c : (valid ? val - c : kInvalid);
    if (lane < 7) S.rec[v * 8 + lane] = out;
    __syncwarp();
}

// Warp-collective: exact argmax config byte of stream v at its final split.
__device__ uint8_t stream_cfg(const InstView& in, const WarpState& S, int v, int ri, int rt, const ekya_dims& d) {
    const int lane = threadIdx.x & 31, nG = d.n_gamma;
    const int tk = lane < 8 ? S.lthr[v * 8 + lane] : INT_MAX;
    const int sl = ladder_slot(tk, ri);
    if (sl < 0) return (uint8_t)(kLambdaNone << 5);
    const int l = S.lidx[v * 8 + sl];
    const float fac = S.lfac[v * 8 + sl];
    const float stale = in.stale[v];
    float a = -1.0f;
    if (lane == 0) a = fmul(fac, stale);
    else if (lane <= nG) {
        const float4 c = in.get(v, lane - 1, nG);
        float w;
        if (window_acc(stale, c.y, c.x, rt, d.unit_gpu_seconds, &w)) a = fmul(fac, w);
    }
    const int m = __reduce_max_sync(FULL, __float_as_int(a));
    const unsigned hits = __ballot_sync(FULL, __float_as_int(a) == m);
    return (uint8_t)((__ffs(hits) - 1) | (l << 5));
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
template <int MODE>
__global__ void __launch_bounds__(kThiefThreads, 8) thief_kernel(ThiefParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const ekya_dims& d = p.d;
    const int V = d.n_streams, J = 2 * V, D = d.steal_units, U = d.units, nG = d.n_gamma, nL = d.n_lambda;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const WarpState S = carve(smem + warp * p.warp_bytes, V);
    float* staged = reinterpret_cast<float*>(smem + warp * p.warp_bytes + p.state_bytes);
    const long long b = (long long)blockIdx.x * p.warps + warp;
    if (b >= d.n_inst) return;

    InstView in{p.t.stale + b * V, p.t.cost + b * V * nG, p.t.post + b * V * nG,
                p.t.lam_min_units + b * V * nL, p.t.lam_factor + b * V * nL, nullptr};

    // ---- validity (R-ERR) ----
    bool ok = true;
    for (int i = lane; i < V; i += 32) ok &= in01(__ldg(in.stale + i));
    for (int i = lane; i < V * nG; i += 32) {
        const float c = __ldg(in.cost + i);
        if (!(c >= 0.0f)) ok = false;
        else if (!isinf(c)) ok &= in01(__ldg(in.post + i));
    }
    for (int i = lane; i < V * nL; i += 32)
        if (__ldg(in.lmu + i) != kLmuPad) ok &= in01(__ldg(in.lf + i));
    ok = __all_sync(FULL, ok);
    // exact shared-reciprocal division applies to every cost and every fl(r uT), r <= U + D
    bool fast = uT_fast(d);
    for (int i = lane; i < V * nG; i += 32) fast &= fast_dividend(__ldg(in.cost + i));
    fast = __all_sync(FULL, fast);
    if (p.stage && ok) {   // stale and (cost, post, post - stale) into this warp's shared memory
        float4* cpd = reinterpret_cast<float4*>(staged);
        float* st = reinterpret_cast<float*>(cpd + V * nG);
        for (int i = lane; i < V; i += 32) st[i] = __ldg(in.stale + i);
        for (int i = lane; i < V * nG; i += 32) {
            const float c = __ldg(in.cost + i), po = __ldg(in.post + i);
            cpd[i] = make_float4(c, po, fsub(po, __ldg(in.stale + i / nG)), 0.0f);
        }
        __syncwarp();
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
    for (int v = 0; v < V; ++v) init_ladder(in, S, v, d);
    for (int v = lane; v < V; v += 32) S.grt[v] = -1;
    __syncwarp();
    for (int v = 0; v < V; ++v) update_stream(in, S, v, d, fast);

    unsigned steps = 0;
    if (MODE == EKYA_THIEF_STEEPEST) {
        const unsigned max_steps = 1u << 26;
        for (;;) {
            // per-stream best down, top-2 by stream
            unsigned long long k1 = 0;
            for (int v = lane; v < V; v += 32) {
                const unsigned long long k = stream_down_key(S, v);
                k1 = k > k1 ? k : k1;
            }
            k1 = warp_max_u64(k1);
            const int s1 = k1 ? (key_job(k1) >> 1) : -1;
            unsigned long long k2 = 0;
            for (int v = lane; v < V; v += 32) {
                if (v == s1) continue;
                const unsigned long long k = stream_down_key(S, v);
                k2 = k > k2 ? k : k2;
            }
            k2 = warp_max_u64(k2);
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
            update_stream(in, S, t >> 1, d, fast);
            if ((w >> 1) != (t >> 1)) update_stream(in, S, w >> 1, d, fast);
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
                    update_stream(in, S, t >> 1, d, fast);
                    if ((w >> 1) != (t >> 1)) update_stream(in, S, w >> 1, d, fast);
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
    for (int v = 0; v < V; ++v) {
        const uint8_t c = stream_cfg(in, S, v, S.alloc[2 * v], S.alloc[2 * v + 1], d);
        if (lane == 0) p.out_cfg[b * V + v] = c;
    }
    if (lane == 0) {
        p.out_sum[b] = sum;
        if (p.out_mean) p.out_mean[b] = mean_q32(sum, V);
        if (p.out_steps) p.out_steps[b] = steps;
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
    p.warps = kThiefThreads / 32;
    p.state_bytes = thief_warp_bytes(d.n_streams);
    const size_t tbytes = ((size_t)d.n_streams * (4 * d.n_gamma + 1) * 4 + 15) & ~size_t(15);
    p.stage = tbytes <= 8192;
    p.warp_bytes = p.state_bytes + (p.stage ? tbytes : 0);
    size_t smem = p.warp_bytes * p.warps;
    if (smem > h->smem_optin) return EKYA_ERR_SHAPE;
    if (d.n_inst == 0) return EKYA_OK;
    auto kern = mode == EKYA_THIEF_STEEPEST ? thief_kernel<EKYA_THIEF_STEEPEST> : thief_kernel<EKYA_THIEF_LITERAL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return EKYA_ERR_CUDA;
    long long grid = (d.n_inst + p.warps - 1) / p.warps;
    if (grid > 0x7fffffffLL) return EKYA_ERR_SHAPE;
    kern<<<(unsigned)grid, kThiefThreads, smem, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
