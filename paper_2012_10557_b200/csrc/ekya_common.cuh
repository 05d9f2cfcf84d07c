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
    unsigned int err;       // OR of kErr* bits
    unsigned int pad[15];
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
