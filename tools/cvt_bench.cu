// Pipe throughput on sm_100a: ex2.approx.f32 (MUFU), cvt.rn.bf16x2.f32 (F2FP),
// and the two interleaved 2:1 as in the softmax (are they one pipe?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cvt_bench cvt_bench.cu
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void k(float* out, int iters) {
  float a[8];
  uint32_t h[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); h[i] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (MODE == 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(h[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
      if (MODE == 2) {
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
        if (i & 1) asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "+r"(h[i]) : "f"(a[i]), "f"(a[i - 1]));
      }
      if (MODE == 3) asm volatile("prmt.b32 %0, %0, %1, 0x7632;" : "+r"(h[i]) : "r"(h[(i + 3) & 7]));
    }
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i] + (float)h[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 4);
  const int iters = 4096;
  const char* names[] = {"ex2.f32 (MUFU)", "cvt.rn.bf16x2.f32", "ex2 + cvt (2:1)", "prmt"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int warps : {8, 16}) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&]() {
        if (mode == 0) k<0><<<148, warps * 32>>>(d, iters);
        if (mode == 1) k<1><<<148, warps * 32>>>(d, iters);
        if (mode == 2) k<2><<<148, warps * 32>>>(d, iters);
        if (mode == 3) k<3><<<148, warps * 32>>>(d, iters);
      };
      launch();
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      int clk;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      const double per_it = mode == 2 ? 12.0 : 8.0;   // instructions per thread per iteration
      const double insts = (double)warps * 32 * iters * per_it;
      const double cyc = ms * 1e-3 * clk * 1e3;
      printf("%-20s warps/SM %2d: %.1f lane-instr/clk/SM\n", names[mode], warps, insts / cyc);
    }
  }
  return 0;
}
