// Throughput of scalar FADD/FMUL vs packed FADD2/FMUL2/FFMA2 on sm_100a (microbenchmark for DESIGN.md).
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 add2(u64 a, u64 b){u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;}
__global__ void k_scalar(float* o, int n, float a) {
  float s[8]; for (int i=0;i<8;++i) s[i]=threadIdx.x+i;
  for (int i=0;i<n;++i) {
    #pragma unroll
    for (int j=0;j<8;++j) s[j] = __fadd_rn(s[j], a);
  }
  float t=0; for (int i=0;i<8;++i) t+=s[i]; o[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
__global__ void k_packed(u64* o, int n, u64 a) {
  u64 s[8]; for (int i=0;i<8;++i) s[i]=threadIdx.x+i;
  for (int i=0;i<n;++i) {
    #pragma unroll
    for (int j=0;j<8;++j) s[j] = add2(s[j], a);
  }
  u64 t=0; for (int i=0;i<8;++i) t^=s[i]; o[blockIdx.x*blockDim.x+threadIdx.x]=t;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms*4, thr = 512, n = 20000;
  float* o; cudaMalloc(&o, blocks*thr*8);
  cudaEvent_t e0,e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep=0; rep<2; ++rep) {
    cudaEventRecord(e0); k_scalar<<<blocks,thr>>>(o,n,1.0f); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms,e0,e1);
    double ops = (double)blocks*thr*n*8;
    printf("scalar FADD: %.3f ms  %.2f Tflop/s  %.1f flop/clk/SM @1965MHz\n", ms, ops/ms/1e9, ops/(ms*1e-3)/sms/1.965e9);
    cudaEventRecord(e0); k_packed<<<blocks,thr>>>((u64*)o,n,0x3f8000003f800000ULL); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms,e0,e1);
    ops = (double)blocks*thr*n*16;
    printf("packed FADD2: %.3f ms  %.2f Tflop/s  %.1f flop/clk/SM @1965MHz\n", ms, ops/ms/1e9, ops/(ms*1e-3)/sms/1.965e9);
  }
  return 0;
}
