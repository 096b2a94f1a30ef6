// Microbenchmark: throughput per SM of the f32x2 -> bf16x2 / f16x2 pack
// (F2FP), alone and interleaved with MUFU ex2, to see which pipe it uses.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>  // 0 = cvt bf16x2, 1 = cvt f16x2, 2 = ex2, 3 = ex2 + cvt bf16x2 (1:1), 4 = prmt
__global__ void k(unsigned* out, int iters, float seed) {
  float a[8];
  unsigned r[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = seed * (threadIdx.x + i) * 1e-6f - 1.0f; r[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 3)
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r[i]) : "f"(a[i]), "f"(__uint_as_float(r[(i + 1) & 7])));
      if (MODE == 1)
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r[i]) : "f"(a[i]), "f"(__uint_as_float(r[(i + 1) & 7])));
      if (MODE == 2 || MODE == 3) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 4) asm volatile("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(r[i]) : "r"(__float_as_uint(a[i])), "r"(r[(i + 1) & 7]));
    }
  }
  unsigned s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += r[i] + __float_as_uint(a[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE>
void run(const char* name, int sms, unsigned* out) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096, threads = 512;
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<MODE><<<sms, threads>>>(out, iters, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  double insts = double(threads) * iters * 8;  // per SM, per instruction kind
  printf("%-22s %.3f ms  %.1f thread-instr/clk/SM (each kind)\n", name, ms, insts / (ms * 1e6) / 1.965);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned* out; cudaMalloc(&out, sms * 1024 * 4);
  run<0>("cvt.rn.bf16x2.f32", sms, out);
  run<1>("cvt.rn.f16x2.f32", sms, out);
  run<2>("ex2.approx", sms, out);
  run<3>("ex2 + cvt bf16x2", sms, out);
  run<4>("prmt", sms, out);
  return 0;
}
