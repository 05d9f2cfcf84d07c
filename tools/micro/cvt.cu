// Throughput of the Q32 conversion round(x 2^32) on sm_100a: 64-bit F2I vs a 32-bit split
// (two F2I.U32) vs pure integer bit manipulation (microbenchmark for DESIGN.md).
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ void q_f2i64(float x, unsigned& lo, unsigned& hi) {
  const u64 v = __float2ull_rn(__fmul_rn(x, 4294967296.0f)); lo = (unsigned)v & 0xFFFFu; hi = (unsigned)(v >> 16);
}
__device__ __forceinline__ void q_split(float x, unsigned& lo, unsigned& hi) {
  const float xs = __fmul_rn(x, 65536.0f); const float h = floorf(xs);
  const unsigned l = __float2uint_rn(__fmul_rn(__fsub_rn(xs, h), 65536.0f));
  hi = __float2uint_rz(h) + (l >> 16); lo = l & 0xFFFFu;
}
__device__ __forceinline__ void q_int(float x, unsigned& lo, unsigned& hi) {
  const unsigned b = __float_as_uint(x);
  const int e = (int)(b >> 23) - 127;                 // x in [0,1]: e <= 0
  const unsigned m = (b & 0x7FFFFFu) | 0x800000u;
  unsigned q;
  if (e >= -9) {                                       // exact: m 2^(e+9) < 2^33
    q = e >= 0 ? 0u : m << (e + 9);
  } else {
    const int s = min(-(e + 9), 31);
    const unsigned t = m >> s, r = m & ((1u << s) - 1u), half = 1u << (s - 1);
    q = t + ((r > half || (r == half && (t & 1u))) ? 1u : 0u);
    if ((b >> 23) == 0) q = 0;
  }
  hi = e >= 0 ? 65536u : q >> 16; lo = e >= 0 ? 0u : q & 0xFFFFu;
}
template <int MODE>
__global__ void k(const float* in, unsigned* o, int n) {
  unsigned a = 0, c = 0;
  float x[8];
  for (int j = 0; j < 8; ++j) x[j] = in[(threadIdx.x + j) & 1023];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned lo, hi;
      if (MODE == 0) q_f2i64(x[j], lo, hi); else if (MODE == 1) q_split(x[j], lo, hi); else q_int(x[j], lo, hi);
      a += lo; c += hi;
      x[j] = __uint_as_float(__float_as_uint(x[j]) ^ (i & 1));
    }
  }
  o[blockIdx.x * blockDim.x + threadIdx.x] = a ^ c;
}
__global__ void check(unsigned* bad) {
  for (unsigned b = blockIdx.x * blockDim.x + threadIdx.x; b <= 0x3F800000u; b += gridDim.x * blockDim.x) {
    const float x = __uint_as_float(b);
    unsigned l0, h0, l1, h1, l2, h2;
    q_f2i64(x, l0, h0); q_split(x, l1, h1); q_int(x, l2, h2);
    if (l0 != l1 || h0 != h1) atomicAdd(bad, 1u);
    if (l0 != l2 || h0 != h2) atomicAdd(bad + 1, 1u);
  }
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float h[1024]; for (int i = 0; i < 1024; ++i) h[i] = (i % 17 == 0) ? 1.0f : (float)(i * 2654435761u % 1000003) / 1000003.0f * ((i & 7) ? 1.0f : 1e-4f);
  float* in; cudaMalloc(&in, 4096); cudaMemcpy(in, h, 4096, cudaMemcpyHostToDevice);
  unsigned* o; int blocks = sms * 4, thr = 512, n = 4000; cudaMalloc(&o, blocks * thr * 4);
  // correctness of the two alternatives against the 64-bit conversion
  unsigned* d; cudaMalloc(&d, 8); cudaMemset(d, 0, 8);
  check<<<sms * 8, 256>>>(d);
  unsigned bad[2]; cudaMemcpy(bad, d, 8, cudaMemcpyDeviceToHost);
  printf("exhaustive [0,1]: split mismatches %u, integer mismatches %u\n", bad[0], bad[1]);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char* names[3] = {"F2I.U64", "split 2xF2I.U32", "integer bits"};
  for (int rep = 0; rep < 2; ++rep) for (int m = 0; m < 3; ++m) {
    cudaEventRecord(e0);
    if (m == 0) k<0><<<blocks, thr>>>(in, o, n); else if (m == 1) k<1><<<blocks, thr>>>(in, o, n); else k<2><<<blocks, thr>>>(in, o, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * n * 8;
    if (rep) printf("%-16s %.3f ms  %.1f conversions/clk/SM @1965MHz\n", names[m], ms, ops / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}
