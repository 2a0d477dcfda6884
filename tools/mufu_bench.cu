// Throughput of the exp2 variants on one SM-full of warps (sm_100a):
// ex2.approx.ftz.f32, ex2.approx.f16x2, ex2.approx.ftz.bf16x2, and the FMA-pipe polynomial.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bench mufu_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_bf16.h>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t h[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = 0xBC00BC00u + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) { asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])); }
      if (MODE == 1) { asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i])); }
      if (MODE == 2) { asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i])); }
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + (float)h[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* d; cudaMalloc(&d, 4);
  int iters = 4096;
  const char* names[] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16, 32}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&]() {
        if (mode == 0) k<0><<<148, warps * 32>>>(d, iters);
        if (mode == 1) k<1><<<148, warps * 32>>>(d, iters);
        if (mode == 2) k<2><<<148, warps * 32>>>(d, iters);
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      double insts = (double)warps * 32 * iters * 8;   // lane-instructions per SM
      double cyc = ms * 1e-3 * clk * 1e3;
      printf("%-10s warps/SM %2d: %.2f lane-instr/clk/SM (%.3f ms, clk %d MHz)\n", names[mode], warps, insts / cyc, ms, clk / 1000);
    }
  }
  return 0;
}
