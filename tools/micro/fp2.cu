// Measured FP32 SIMT peak on sm_100a for the ALU-bound roofline (CLUSTER's rule-5 distances:
// FSUB / FMUL / FADD, no FMA contraction).  Scalar FADD / FMUL and packed FADD2 / FMUL2, 8
// independent chains per thread, 4 x 512-thread CTAs per SM, CUDA events; prints TFLOP/s
// (one flop per lane and op, two per packed op) and flop/clk/SM at the clock given as argv[1]
// (MHz, sampled by the caller with nvidia-smi during the run).
#include <cstdio>
#include <cstdlib>
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ u64 mul2(u64 a, u64 b) { u64 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
template <int OP>
__global__ void k_scalar(float* o, int n, float a) {
  float s[8]; for (int i = 0; i < 8; ++i) s[i] = threadIdx.x + i;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = OP == 0 ? __fadd_rn(s[j], a) : __fmul_rn(s[j], a);
  }
  float t = 0; for (int i = 0; i < 8; ++i) t += s[i]; o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int OP>
__global__ void k_packed(u64* o, int n, u64 a) {
  u64 s[8]; for (int i = 0; i < 8; ++i) s[i] = threadIdx.x + i;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = OP == 0 ? add2(s[j], a) : mul2(s[j], a);
  }
  u64 t = 0; for (int i = 0; i < 8; ++i) t ^= s[i]; o[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main(int argc, char** argv) {
  const double mhz = argc > 1 ? atof(argv[1]) : 1965.0;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, thr = 512, n = 20000;
  float* o; cudaMalloc(&o, (size_t)blocks * thr * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  double best = 0;
  for (int rep = 0; rep < 3; ++rep) {
    for (int v = 0; v < 4; ++v) {
      cudaEventRecord(e0);
      if (v == 0) k_scalar<0><<<blocks, thr>>>(o, n, 1.0f);
      if (v == 1) k_scalar<1><<<blocks, thr>>>(o, n, 1.0f);
      if (v == 2) k_packed<0><<<blocks, thr>>>((u64*)o, n, 0x3f8000003f800000ULL);
      if (v == 3) k_packed<1><<<blocks, thr>>>((u64*)o, n, 0x3f8000003f800000ULL);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * thr * n * 8 * (v >= 2 ? 2 : 1);
      const double tf = ops / ms / 1e9;
      if (rep > 0 && tf > best) best = tf;
      static const char* nm[4] = {"FADD", "FMUL", "FADD2 (packed)", "FMUL2 (packed)"};
      if (rep > 0) printf("%-15s %.3f ms  %.2f TFLOP/s  %.1f flop/clk/SM @%.0f MHz\n", nm[v], ms, tf, ops / (ms * 1e-3) / sms / (mhz * 1e6), mhz);
    }
  }
  printf("{\"fp32_simt_tflops\": %.3f, \"sm_mhz\": %.0f, \"sms\": %d}\n", best, mhz, sms);
  return 0;
}
