// window.cu -- NEXT-1: the retraining window as a timeline, with
// the thief re-invoked at every retraining completion (
// readings W1-W6 in DESIGN.md).
//
// All instances advance in lock-step invocations driven from the host: each of
// the V + 1 rounds is (1) window_prepare: the residual tables of every instance
// (new model accuracy of finished streams, remaining work of retraining streams
// and the remaining window folded into the costs); (2) the thief kernel itself
// (thief.cu) on those tables; (3) window_advance: one thread per instance finds
// the next completion, accumulates the realized inference accuracy and updates
// the remaining work -- in the oracle's operation order, one binary32 rounding
// per operation.  Instances whose window has ended are left untouched.
#include <algorithm>

#include "launch.h"

namespace ekya {

namespace {

struct WinState {
    // residual tables (thief inputs) and thief outputs
    float* stale;        // [B][V]
    float* cost;         // [B][V][nG]
    uint16_t* alloc;     // [B][2V]
    uint8_t* cfg;        // [B][V]
    unsigned long long* sum;   // [B]
    // timeline state
    float* tau;          // [B]
    uint32_t* ev;        // [B]
    int* valid;          // [B]
    float* m;            // [B][V] model accuracy
    float* R;            // [B][V] remaining work (cost units)
    float* A;            // [B][V] accumulated accuracy x window fraction
    int8_t* stt;         // [B][V] 0 idle, 1 retraining, 2 done
    int8_t* g;           // [B][V] config being retrained (1-based)
};

inline size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

struct WinLayout {
    size_t stale, cost, alloc, cfg, sum, tau, ev, valid, m, R, A, stt, g, total;
};
inline WinLayout win_layout(long long B, int V, int nG) {
    WinLayout L;
    size_t o = 0;
    const size_t BV = (size_t)B * V;
    L.stale = o; o += a256(BV * 4);
    L.cost = o;  o += a256(BV * (size_t)(nG > 1 ? nG : 1) * 4);
    L.alloc = o; o += a256(BV * 4);
    L.cfg = o;   o += a256(BV);
    L.sum = o;   o += a256((size_t)B * 8);
    L.tau = o;   o += a256((size_t)B * 4);
    L.ev = o;    o += a256((size_t)B * 4);
    L.valid = o; o += a256((size_t)B * 4);
    L.m = o;     o += a256(BV * 4);
    L.R = o;     o += a256(BV * 4);
    L.A = o;     o += a256(BV * 4);
    L.stt = o;   o += a256(BV);
    L.g = o;     o += a256(BV);
    L.total = o;
    return L;
}

struct WinParams {
    ekya_dims d;
    ekya_tables t;   // the caller's tables
    WinState w;
    float* out_avg;
    uint32_t* out_events;
    float* out_done;
    DevState* st;
};

// W2/W3: residual tables at the instance's current tau (thread per instance)
__global__ void window_prepare_kernel(WinParams p, int round) {
    const ekya_dims& d = p.d;
    const int V = d.n_streams, nG = d.n_gamma, nL = d.n_lambda;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < d.n_inst;
         b += (long long)gridDim.x * blockDim.x) {
        if (round == 0) {
            // R-ERR: validity exactly as the thief's (the thief zeroes invalid instances)
            bool ok = true;
            for (int v = 0; v < V; ++v) {
                ok &= in01(p.t.stale[b * V + v]);
                for (int k = 0; k < nG; ++k) {
                    const float c = p.t.cost[(b * V + v) * nG + k];
                    if (!(c >= 0.0f)) ok = false;
                    else if (!isinf(c)) ok &= in01(p.t.post[(b * V + v) * nG + k]);
                }
                for (int l = 0; l < nL; ++l)
                    if (p.t.lam_min_units[(b * V + v) * nL + l] != kLmuPad) ok &= in01(p.t.lam_factor[(b * V + v) * nL + l]);
            }
            p.w.valid[b] = ok;
            p.w.tau[b] = 0.0f;
            p.w.ev[b] = 0;
            for (int v = 0; v < V; ++v) {
                p.w.m[b * V + v] = p.t.stale[b * V + v];
                p.w.R[b * V + v] = 0.0f;
                p.w.A[b * V + v] = 0.0f;
                p.w.stt[b * V + v] = 0;
                p.w.g[b * V + v] = 0;
                p.out_done[b * V + v] = ok ? 1.0f : 0.0f;
            }
        }
        const float tau = p.w.tau[b];
        const float sc = fdiv(1.0f, fsub(1.0f, tau));
        for (int v = 0; v < V; ++v) {
            const long long bv = b * V + v;
            p.w.stale[bv] = p.w.valid[b] ? p.w.m[bv] : p.t.stale[bv];
            const int s = p.w.stt[bv], gv = p.w.g[bv];
            for (int k = 0; k < nG; ++k) {
                const float c = p.t.cost[bv * nG + k];
                float cs = INFINITY;
                if (!p.w.valid[b]) cs = c;   // keep the caller's (invalid) data: the thief flags it
                else if (tau >= 1.0f) cs = INFINITY;
                else if (s == 0) cs = isinf(c) ? c : fmul(c, sc);
                else if (s == 1 && k + 1 == gv) cs = fmul(p.w.R[bv], sc);
                p.w.cost[bv * nG + k] = cs;
            }
        }
    }
}

// W4-W6: one invocation's outcome (thread per instance)
__global__ void window_advance_kernel(WinParams p) {
    const ekya_dims& d = p.d;
    const int V = d.n_streams, nG = d.n_gamma, nL = d.n_lambda;
    const float uT = d.unit_gpu_seconds;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < d.n_inst;
         b += (long long)gridDim.x * blockDim.x) {
        const float tau = p.w.tau[b];
        if (!p.w.valid[b] || !(tau < 1.0f) || p.w.ev[b] > (unsigned)V) continue;
        const float rem = fsub(1.0f, tau);
        const uint16_t* al = p.w.alloc + b * 2 * V;
        const uint8_t* cf = p.w.cfg + b * V;
        auto tdone = [&](int v, int gv) -> float {
            const float den = fmul(__int2float_rn((int)al[2 * v + 1]), uT);
            const float f = fdiv(p.w.cost[(b * V + v) * nG + gv - 1], den);
            return fadd(tau, fmul(f, rem));
        };
        float tnext = 1.0f;
        for (int v = 0; v < V; ++v) {
            const int gv = cf[v] & 31;
            if (gv > 0) {
                const float tv = tdone(v, gv);
                if (tv < tnext) tnext = tv;
            }
        }
        const float span = fsub(tnext, tau);
        for (int v = 0; v < V; ++v) {
            const int l = cf[v] >> 5;
            const float fac = l == kLambdaNone ? 0.0f : p.t.lam_factor[(b * V + v) * nL + l];
            const float acc = fmul(fac, p.w.m[b * V + v]);
            p.w.A[b * V + v] = fadd(p.w.A[b * V + v], fmul(span, acc));
        }
        for (int v = 0; v < V; ++v) {
            const int gv = cf[v] & 31;
            if (gv == 0) continue;
            const long long bv = b * V + v;
            const float tv = tdone(v, gv);
            if (tv <= tnext) {
                p.w.stt[bv] = 2;
                p.w.m[bv] = p.t.post[bv * nG + gv - 1];
                p.out_done[bv] = tv;
            } else {
                const float base = p.w.stt[bv] == 1 ? p.w.R[bv] : p.t.cost[bv * nG + gv - 1];
                const float q = fdiv(span, fsub(tv, tau));
                p.w.R[bv] = fmul(base, fsub(1.0f, q));
                p.w.stt[bv] = 1;
                p.w.g[bv] = (int8_t)gv;
            }
        }
        p.w.tau[b] = tnext;
        p.w.ev[b] += 1;
    }
}

__global__ void window_finish_kernel(WinParams p) {
    const ekya_dims& d = p.d;
    const int V = d.n_streams;
    for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < d.n_inst;
         b += (long long)gridDim.x * blockDim.x) {
        if (!p.w.valid[b]) {
            p.out_avg[b] = 0.0f;
            p.out_events[b] = 0;
            continue;
        }
        float s = 0.0f;
        for (int v = 0; v < V; ++v) s = fadd(s, p.w.A[b * V + v]);
        p.out_avg[b] = fdiv(s, __int2float_rn(V));
        p.out_events[b] = p.w.ev[b];
    }
}

}  // namespace

size_t window_workspace_bytes(const ekya_dims& d) { return win_layout(d.n_inst, d.n_streams, d.n_gamma).total; }

int launch_window(ekya_handle* h, const ekya_dims& d, const ekya_tables& t, int mode, void* ws, size_t ws_bytes,
                  float* out_avg, uint32_t* out_events, float* out_done, cudaStream_t s) {
    const WinLayout L = win_layout(d.n_inst, d.n_streams, d.n_gamma);
    if (ws_bytes < L.total || !ws) return EKYA_ERR_ARG;
    if (d.n_inst == 0) return EKYA_OK;
    unsigned char* base = static_cast<unsigned char*>(ws);
    WinParams p{};
    p.d = d;
    p.t = t;
    p.w.stale = reinterpret_cast<float*>(base + L.stale);
    p.w.cost = reinterpret_cast<float*>(base + L.cost);
    p.w.alloc = reinterpret_cast<uint16_t*>(base + L.alloc);
    p.w.cfg = base + L.cfg;
    p.w.sum = reinterpret_cast<unsigned long long*>(base + L.sum);
    p.w.tau = reinterpret_cast<float*>(base + L.tau);
    p.w.ev = reinterpret_cast<uint32_t*>(base + L.ev);
    p.w.valid = reinterpret_cast<int*>(base + L.valid);
    p.w.m = reinterpret_cast<float*>(base + L.m);
    p.w.R = reinterpret_cast<float*>(base + L.R);
    p.w.A = reinterpret_cast<float*>(base + L.A);
    p.w.stt = reinterpret_cast<int8_t*>(base + L.stt);
    p.w.g = reinterpret_cast<int8_t*>(base + L.g);
    p.out_avg = out_avg;
    p.out_events = out_events;
    p.out_done = out_done;
    p.st = h->dstate;
    ekya_tables rt = t;   // the residual tables: stale and cost from the workspace
    rt.stale = p.w.stale;
    rt.cost = d.n_gamma > 0 ? p.w.cost : t.cost;
    const int grid = (int)std::min<long long>((d.n_inst + 255) / 256, (long long)h->sm_count * 4);
    for (int r = 0; r <= d.n_streams; ++r) {
        window_prepare_kernel<<<grid, 256, 0, s>>>(p, r);
        h->launches++;
        int e = launch_thief(h, d, rt, mode, p.w.alloc, p.w.cfg, reinterpret_cast<uint64_t*>(p.w.sum), nullptr,
                             nullptr, s);
        if (e != EKYA_OK) return e;
        window_advance_kernel<<<grid, 256, 0, s>>>(p);
        h->launches++;
    }
    window_finish_kernel<<<grid, 256, 0, s>>>(p);
    h->launches++;
    return cuda_status(cudaGetLastError());
}

}  // namespace ekya
