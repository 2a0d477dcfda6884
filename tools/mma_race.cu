// Is it safe for two warps of one CTA to issue tcgen05.mma / tcgen05.commit
// concurrently (into disjoint TMEM columns, from disjoint shared memory)?
// The two-tile ping-pong K3 gave wrong rows intermittently when both slot
// issuers ran at once.  Here each of two "slots" runs a
// lockstep pipeline like the attention kernel: an issuer warp issues an SS MMA
// (D1 += A.B^T) and a TS MMA (D2 += P[tmem].V) and commits to its barrier; four
// reader warps wait on the barrier, read both accumulators back (tcgen05.ld) and
// check them against the exact expected sums, then acknowledge.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_race tools/mma_race.cu
//   tools/mma_race [iters]   -> mismatches per mode: 0 both slots at once, 1 slot 0 only,
//                               2 both slots with the MMA issue serialised by a lock
#include <cstdio>
#include <cstdlib>
#include <cuda_bf16.h>

#include "../paper_2511_19835_b200/csrc/tc_ptx.cuh"

using namespace rsa;

constexpr int TILE = 128 * 128 * 2;    // 128 rows x 128 bf16 = 32 KB (two 64-column panels)
constexpr int PANEL = 128 * 128;
constexpr uint32_t IDESC = ptx::idesc_bf16(128, 64, false);   // M = 128, N = 64, K-major B

__global__ void __launch_bounds__(384, 1) race_kernel(int iters, int mode, unsigned* bad, float* sample) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  // per slot: A (32 KB), B (32 KB: 64 rows used), V (32 KB: 64 rows used)
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + 6 * TILE);
  uint64_t* full = bars;         // [2]
  uint64_t* ack = bars + 2;      // [2], 128 arrivals
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 4);
  int* lock = reinterpret_cast<int*>(bars + 5);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // fill: slot 0 A = 1, slot 1 A = 2, B = V = 1 (bf16); layout does not matter for constants
  for (int i = threadIdx.x; i < 6 * TILE / 2; i += blockDim.x) {
    const int slot = i / (3 * TILE / 2), which = (i % (3 * TILE / 2)) / (TILE / 2);
    reinterpret_cast<__nv_bfloat16*>(base)[i] = __float2bfloat16((which == 0 && slot == 1) ? 2.f : 1.f);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(full + s, 1);
      ptx::mbar_init(ack + s, 128);
    }
    *lock = 0;
    ptx::fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> MMA operand reads
  if (warp == 2) ptx::tmem_alloc<512>(tslot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tslot;
  // TMEM per slot s (256 columns): D1 [0,64), D2 [64,128), P [128,192) (bf16 pairs = 128 K)
  if (warp >= 4) {
    const int s = (warp - 4) >> 2, quad = warp & 3;
    const uint32_t lane_base = tmem + (uint32_t)(s * 256) + ((uint32_t)(quad * 32) << 16);
    uint32_t ones[32];
    const uint32_t one2 = 0x3F803F80u;   // bf16 (1, 1)
#pragma unroll
    for (int i = 0; i < 32; ++i) ones[i] = one2;
    ptx::tmem_st32(lane_base + 128, ones);
    ptx::tmem_st32(lane_base + 160, ones);
    ptx::tmem_st_wait();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();

  const bool slot_on[2] = {true, mode != 1};
  if (warp < 2) {
    const int s = warp;
    if (slot_on[s]) {
      const uint32_t a = ptx::smem_u32(base + (3 * s + 0) * TILE);
      const uint32_t b = ptx::smem_u32(base + (3 * s + 1) * TILE);
      const uint32_t v = ptx::smem_u32(base + (3 * s + 2) * TILE);
      const uint32_t tm = tmem + (uint32_t)(s * 256);
      for (int it = 0; it < iters; ++it) {
        if (it > 0) ptx::mbar_wait(ack + s, (uint32_t)((it - 1) & 1));
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          if (mode == 2)
            while (atomicCAS(lock, 0, 1) != 0) {
            }
#pragma unroll
          for (int k = 0; k < 8; ++k) {   // D1 += A . B^T, K = 128
            const uint64_t da = ptx::sw128_desc(a + (k / 4) * PANEL + (k % 4) * 32, 16, 1024);
            const uint64_t db = ptx::sw128_desc(b + (k / 4) * PANEL + (k % 4) * 32, 16, 1024);
            ptx::mma_ss(tm, da, db, IDESC, (it > 0 || k > 0) ? 1u : 0u);
          }
#pragma unroll
          for (int k = 0; k < 8; ++k) {   // D2 += P[tmem] . V^T, K = 128 (P: 8 columns per 16 K)
            const uint64_t dv = ptx::sw128_desc(v + (k / 4) * PANEL + (k % 4) * 32, 16, 1024);
            ptx::mma_ts(tm + 64, tm + 128 + k * 8, dv, IDESC, (it > 0 || k > 0) ? 1u : 0u);
          }
          ptx::tc_commit(full + s);
          if (mode == 2) atomicExch(lock, 0);
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    const int s = (warp - 4) >> 2, quad = warp & 3;
    if (slot_on[s]) {
      const uint32_t lane_base = tmem + (uint32_t)(s * 256) + ((uint32_t)(quad * 32) << 16);
      const float va = s == 1 ? 2.f : 1.f;
      unsigned nbad = 0;
      for (int it = 0; it < iters; ++it) {
        ptx::mbar_wait(full + s, (uint32_t)(it & 1));
        ptx::tc_fence_after();
        uint32_t d1[32], d2[32];
        ptx::tmem_ld32(lane_base + 0, d1);
        ptx::tmem_ld32(lane_base + 64, d2);
        ptx::tmem_ld_wait();
        const float e1 = (float)(it + 1) * 128.f * va, e2 = (float)(it + 1) * 128.f;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          nbad += __uint_as_float(d1[i]) != e1;
          nbad += __uint_as_float(d2[i]) != e2;
        }
        if (it == iters - 1 && quad == 0 && lane == 0) {
          sample[2 * s] = __uint_as_float(d1[0]);
          sample[2 * s + 1] = __uint_as_float(d2[0]);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(ack + s);
      }
      if (nbad) atomicAdd(bad + s, nbad);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 20000;   // (it + 1) * 256 stays exact in fp32
  const int smem = 6 * TILE + 1024 + 256;
  cudaFuncSetAttribute(race_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned* bad;
  float* sample;
  cudaMalloc(&bad, 8);
  cudaMalloc(&sample, 16);
  const char* names[] = {"both slots at once", "slot 0 only", "both, issue under a lock"};
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaMemset(bad, 0, 8);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      race_kernel<<<148, 384, smem>>>(iters, mode, bad, sample);   // one CTA per SM, all independent
      cudaEventRecord(e1);
      cudaError_t err = cudaDeviceSynchronize();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      unsigned h[2];
      float smp[4];
      cudaMemcpy(h, bad, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(smp, sample, 16, cudaMemcpyDeviceToHost);
      printf("rep %d mode %d (%s): %s, mismatches slot0 %u slot1 %u, last D1/D2 slot0 %.0f/%.0f slot1 %.0f/%.0f, "
             "%.3f ms (%.1f cycles/iter at 1.9 GHz)\n",
             rep, mode, names[mode], cudaGetErrorString(err), h[0], h[1], smp[0], smp[1], smp[2], smp[3], ms,
             ms * 1.9e6 / iters);
    }
  return 0;
}
