// ekya_common.cuh -- device helpers shared by the sm_100a kernels of libekya.
//
// Arithmetic contract: every floating-point operation
// that can influence a result is ONE IEEE binary32 rounding (nearest-even),
// written with explicit __f*_rn intrinsics so nvcc can never contract it into
// an FMA; the objective is summed exactly as Q32 integers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/ekya.h"

namespace ekya {

constexpr int kLambdaNone = 7;
constexpr uint16_t kLmuPad = 0xFFFFu;
constexpr int kMaxGamma = 31;   // real configs; index 0 = "no retraining"
constexpr int kMaxLambda = 7;

// device-side error word bits (handle workspace)
constexpr unsigned kErrData = 1u;

struct DevState {
    unsigned int err;                   // OR of kErr* bits
    unsigned int pad0;
    unsigned long long lloyd_passes;    // CLUSTER assignment passes (telemetry)
    unsigned int thief_next;            // thief: next instance to claim (0 between launches)
    unsigned int thief_done;            // thief: warps past their last claim (0 between launches)
    unsigned int pad[10];
};

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }

// Rule 4: Q32(x) = round-to-nearest-even integer of fl(x * 2^32)
__device__ __forceinline__ unsigned long long q32(float x) {
    return __float2ull_rn(__fmul_rn(x, 4294967296.0f));
}

// mean = (float)((double)S / (n * 2^32))
__device__ __forceinline__ float mean_q32(unsigned long long s, int n) {
    double num = __ull2double_rn(s);
    double den = __dmul_rn((double)n, 4294967296.0);
    return __double2float_rn(__ddiv_rn(num, den));
}

__device__ __forceinline__ bool in01(float x) { return x >= 0.0f && x <= 1.0f; }

// Rule 1: feasibility of retraining with cost c at rt units; on success *g
// receives rule 2's window-average accuracy factor g(gamma, rt).
__device__ __forceinline__ bool window_acc(float stale, float post, float cost, int rt, float uT,
                                           float* g) {
    if (rt < 1) return false;
    float den = fmul(__int2float_rn(rt), uT);
    float f = fdiv(cost, den);
    if (!(f <= 1.0f)) return false;
    float diff = fsub(post, stale);
    float prod = fmul(f, diff);
    *g = fsub(post, prod);
    return true;
}

// Alg. 2 lines 3-4 (rule 3): admissible lambda with the highest accuracy,
// lowest index on ties; -1 if none.
__device__ __forceinline__ int lambda_star(float stale, const uint16_t* lmu, const float* lf, int nl,
                                           int ri, float a_min) {
    int best = -1;
    float bacc = 0.0f;
    for (int l = 0; l < nl; ++l) {
        unsigned m = lmu[l];
        if (m == kLmuPad || ri < (int)m) continue;
        float acc = fmul(stale, lf[l]);
        if (!(acc >= a_min)) continue;
        if (best < 0 || acc > bacc) {
            best = l;
            bacc = acc;
        }
    }
    return best;
}

__device__ __forceinline__ void flag_data_error(DevState* st) {
    atomicOr(&st->err, kErrData);
}

// Block-cooperative copy of `bytes` from global `src` to shared `dst_base`
// placed at dst_base + (src % 16) so 16-byte vector loads line up; returns the
// shared pointer that corresponds to src.  dst_base must be 16-byte aligned
// and have room for bytes + 16.
__device__ __forceinline__ unsigned char* stage_to_smem(unsigned char* dst_base, const void* src,
                                                        size_t bytes) {
    const unsigned char* s = static_cast<const unsigned char*>(src);
    size_t mis = reinterpret_cast<uintptr_t>(s) & 15u;
    unsigned char* d = dst_base + mis;
    size_t head = mis ? (16 - mis) : 0;
    if (head > bytes) head = bytes;
    size_t body = ((bytes - head) / 16) * 16;
    for (size_t i = threadIdx.x; i < head; i += blockDim.x) d[i] = __ldg(s + i);
    const uint4* sv = reinterpret_cast<const uint4*>(s + head);
    uint4* dv = reinterpret_cast<uint4*>(d + head);
    for (size_t i = threadIdx.x; i < body / 16; i += blockDim.x) dv[i] = __ldg(sv + i);
    for (size_t i = head + body + threadIdx.x; i < bytes; i += blockDim.x) d[i] = __ldg(s + i);
    return d;
}

// Block-cooperative copy from shared `src` (which sits at the same address
// offset modulo 16 as `dst`) to global `dst`.
__device__ __forceinline__ void store_from_smem(void* dst, const unsigned char* src, size_t bytes) {
    unsigned char* d = static_cast<unsigned char*>(dst);
    size_t mis = reinterpret_cast<uintptr_t>(d) & 15u;
    size_t head = mis ? (16 - mis) : 0;
    if (head > bytes) head = bytes;
    size_t body = ((bytes - head) / 16) * 16;
    for (size_t i = threadIdx.x; i < head; i += blockDim.x) d[i] = src[i];
    const uint4* sv = reinterpret_cast<const uint4*>(src + head);
    uint4* dv = reinterpret_cast<uint4*>(d + head);
    for (size_t i = threadIdx.x; i < body / 16; i += blockDim.x) dv[i] = sv[i];
    for (size_t i = head + body + threadIdx.x; i < bytes; i += blockDim.x) d[i] = src[i];
}

}  // namespace ekya

// ---------------------------------------------------------------------------
// sm_90+/sm_100a asynchronous bulk copies (TMA bulk engine) and mbarriers
// ---------------------------------------------------------------------------
namespace ekya {

__device__ __forceinline__ unsigned smem_addr(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

// make mbarrier initialisation visible to the async proxy
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

// order generic-proxy shared-memory writes before subsequent async-proxy reads
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

// plain arrival (release at CTA scope: this thread's prior shared writes are visible to
// every thread whose wait observes the phase completion)
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// shared-memory counters with release / acquire semantics at CTA scope (monotonic
// dependency counters that never alias, unlike a parity-tracked mbarrier phase)
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {
    asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(smem_addr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
    return v;
}
// warp-uniform wait until *p >= target
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
    while (ld_acquire(p) < target) {
    }
}

__device__ __forceinline__ bool mbar_try_wait(unsigned long long* bar, unsigned parity) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}

// try_wait with a suspend-time hint: the waiting warp is parked (no issue slots spent
// spinning) until the phase completes or about `ns` nanoseconds pass
__device__ __forceinline__ bool mbar_try_wait_hint(unsigned long long* bar, unsigned parity, unsigned ns) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(parity), "r"(ns)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, unsigned parity, unsigned ns = 20000) {
    while (!mbar_try_wait_hint(bar, parity, ns)) {
    }
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    while (!mbar_try_wait(bar, parity)) {
    }
}

// global -> shared bulk copy; completion counted on `bar` (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}

// bulk prefetch of a global range into L2 (bytes % 16 == 0, 16-B aligned)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// shared -> global bulk copy (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Granule staging: the 16-byte granules covering [src, src + bytes) are copied
// to `dst` (16-B aligned) so that src lands at dst + (src & 15).  Returns the
// number of bytes the copy moves; *out receives the shared pointer of src.
struct Granules {
    const unsigned char* g0;
    unsigned bytes;
    unsigned off;
};
__device__ __forceinline__ Granules granules(const void* src, size_t bytes) {
    uintptr_t a = reinterpret_cast<uintptr_t>(src);
    uintptr_t a0 = a & ~uintptr_t(15);
    uintptr_t a1 = (a + bytes + 15) & ~uintptr_t(15);
    Granules g;
    g.g0 = reinterpret_cast<const unsigned char*>(a0);
    g.bytes = bytes ? (unsigned)(a1 - a0) : 0u;
    g.off = (unsigned)(a - a0);
    return g;
}

}  // namespace ekya
