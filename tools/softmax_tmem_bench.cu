// The paired-tile softmax's per-block work without the MMAs: tcgen05.ld the
// scores of a 128-row tile from TMEM, 2^x of every element, pack to bf16 and
// tcgen05.st P back -- by ONE warp per TMEM lane quadrant (128 columns per
// thread, the shipped kernel) or TWO warps per quadrant (64 columns each, the
// split-row variants), with a named barrier per block between the two halves
// of a row in the second case.  Cycles per block (warp 4's clock64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2511_19835_b200/csrc -o softmax_tmem_bench softmax_tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

using namespace rsa;

template <int SPLIT>   // 1: one warp per quadrant, 2: two
__global__ void __launch_bounds__(384, 1) k(float* out, int iters) {
  __shared__ uint32_t tmem_slot;
  __shared__ float xch[2][128];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 1) ptx::tmem_alloc<512>(&tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int nw = 4 * SPLIT;
  if (warp >= 4 && warp < 4 + nw) {
    const int quad = warp & 3, h = (warp - 4) >> 2;
    const int cols = 128 / SPLIT;
    const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16) + (uint32_t)(h * cols);
    // initialise this thread's scores
    for (int c = 0; c < cols / 32; ++c) {
      uint32_t r[32];
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(0.01f * (i + lane) - 0.5f * c);
      ptx::tmem_st32(base + c * 32, r);
    }
    ptx::tmem_st_wait();
    const float2 sc2 = make_float2(0.12f, 0.12f), nb2 = make_float2(-1.f, -1.f);
    float acc = 0.f;
    long long t0 = 0;
    for (int it = 0; it < iters + 10; ++it) {
      if (it == 10) t0 = clock64();
      uint32_t sr[128 / SPLIT / 32][32];
#pragma unroll
      for (int c = 0; c < cols / 32; ++c) ptx::tmem_ld32(base + c * 32, sr[c]);
      ptx::tmem_ld_wait();
      float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < cols / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ptx::ffma2(make_float2(__uint_as_float(sr[c][2 * i]), __uint_as_float(sr[c][2 * i + 1])), sc2, nb2);
          const float2 p = make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
          sum2[i & 1] = ptx::fadd2(sum2[i & 1], p);
          pk[i] = ptx::pack_bf16(p.x, p.y);
        }
        ptx::tmem_st16(base + 64 + c * 16 - (SPLIT == 1 ? 0 : 0), pk);   // P into the upper half (keeps S intact)
      }
      ptx::tmem_st_wait();
      if (SPLIT == 2) {
        xch[h][quad * 32 + lane] = sum2[0].x;
        asm volatile("bar.sync %0, 64;" ::"r"(1 + quad) : "memory");
        acc += xch[1 - h][quad * 32 + lane];
      }
      acc += sum2[0].x + sum2[1].y;
    }
    long long t1 = clock64();
    if (warp == 4 && lane == 0 && blockIdx.x == 0)
      printf("  split %d: %.0f cycles per block\n", SPLIT, (double)(t1 - t0) / iters);
    out[blockIdx.x * 384 + threadIdx.x] = acc;
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 384 * 4);
  printf("one warp per quadrant (128 columns each):\n");
  k<1><<<148, 384>>>(out, 2000);
  cudaDeviceSynchronize();
  printf("two warps per quadrant (64 columns each):\n");
  k<2><<<148, 384>>>(out, 2000);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
