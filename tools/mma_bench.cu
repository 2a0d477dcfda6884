// Microbenchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) for SS / TS
// operand sources and N = 64 / 128 / 256, one CTA per SM.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_bench.cu -o tools/mma_bench
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2511_19835_b200/csrc/tc_ptx.cuh"

using namespace rsa::ptx;

template <int N, bool TS, int CHAINS, int COMMIT_EVERY = 0, int MN = 0>
__global__ void __launch_bounds__(128, 1) bench(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t dummy[4];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(dummy + i, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  long long t0 = 0, t1 = 0;
  if (threadIdx.x == 32) {
    const uint32_t a_addr = smem_u32(base);
    const uint32_t b_addr = smem_u32(base + 16384);
    constexpr uint32_t idesc = idesc_bf16(128, N, MN == 1);
    constexpr uint32_t idesc_k = idesc_bf16(128, N, false);
    // warm-up
    for (int i = 0; i < 64; ++i) {
      const uint64_t b = sw128_desc(b_addr + (i % 4) * 32, 16, 1024);
      if (TS) mma_ts(tmem, tmem + 384 + (i % 8) * 8, b, idesc, 1);
      else mma_ss(tmem, sw128_desc(a_addr + (i % 4) * 32, 16, 1024), b, idesc, 1);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      // MN == 1: B is MN-major (V-style: LBO = panel stride, K step = 16 rows = 2048 B);
      // MN == 2: alternate 8 K-major (S-style) and 8 MN-major (PV-style) MMAs
      // MN == 3: K-major only, alternating accumulators every 8; MN == 4: MN-major only, alternating;
      // MN == 5: alternating majorness, same accumulator and same A
      const bool mn = MN == 1 || MN == 4 || ((MN == 2 || MN == 5) && ((i / 8) & 1));
      if (MN == 6) {
        // the 64-key sub-step sequence: 8 x S_half (TS, N = 64, K-major B, acc at col 0)
        // then 4 x PV_half (TS, N = 128, MN-major B, K = 64 keys, acc at col 256), repeated
        const int ph = i % 12;
        if (ph < 8) {
          mma_ts(tmem, tmem + 384 + ph * 8, sw128_desc(b_addr + (ph % 4) * 32, 16, 1024), idesc_bf16(128, 64, false), 1);
        } else {
          mma_ts(tmem + 256u, tmem + 448 + (ph - 8) * 8, sw128_desc(b_addr + (ph - 8) * 2048, 16384, 1024),
                 idesc_bf16(128, 128, true), 1);
        }
        continue;
      }
      if (MN >= 3) {
        const uint64_t bb = mn ? sw128_desc(b_addr + (i % 8) * 2048, 16384, 1024) : sw128_desc(b_addr + (i % 4) * 32, 16, 1024);
        const uint32_t acc = (MN == 5) ? tmem : tmem + (((i / 8) & 1) ? 256u : 0u);
        mma_ts(acc, tmem + 384 + (i % 8) * 8, bb, mn ? idesc_bf16(128, N, true) : idesc_k, 1);
        continue;
      }
      const uint64_t b = mn ? sw128_desc(b_addr + (i % 8) * 2048, 16384, 1024)
                            : sw128_desc(b_addr + (i % 4) * 32, 16, 1024);
      const uint32_t d = tmem + (CHAINS > 1 ? (uint32_t)((i % CHAINS) * N) : 0u);
      if (MN == 2) { mma_ts(d, tmem + 384 + (i % 8) * 8, b, mn ? idesc_bf16(128, N, true) : idesc_k, 1); continue; }
      if (TS) mma_ts(d, tmem + 384 + (i % 8) * 8, b, idesc, 1);
      else mma_ss(d, sw128_desc(a_addr + (i % 4) * 32, 16, 1024), b, idesc, 1);
      if (COMMIT_EVERY && (i % COMMIT_EVERY) == COMMIT_EVERY - 1) tc_commit(dummy + ((i / COMMIT_EVERY) & 3));
    }
    tc_commit(&bar);
    mbar_wait(&bar, 1);
    t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS, int CHAINS, int COMMIT_EVERY = 0, int MN = 0>
void run(const char* name, int sms) {
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = bench<N, TS, CHAINS, COMMIT_EVERY, MN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  cudaMemset(d, 0, sms * sizeof(long long));
  const int iters = 4096;
  k<<<sms, 128, 100 * 1024>>>(d, iters);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<sms, 128, 100 * 1024>>>(d, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[200];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double flops = 2.0 * 128 * N * 16 * iters * sms;
  printf("%-28s cycles/MMA %7.1f  (ideal %5.1f)  %.0f TFLOP/s over %d SMs  err=%s\n", name, avg / iters,
         128.0 * N / 256.0, flops / (ms * 1e-3) / 1e12, sms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// The attention kernel's per-step MMA sequence: 8 x S = Q K^T (TS, A = Q in
// TMEM, B = K K-major, N = 128) into S buffer j%2 + 2 commits, then 8 x
// O += P V (TS, A = P in S buffer (j-1)%2, B = V MN-major or V^T K-major,
// N = D = 128) + 2 commits.  Cycles per step (ideal 16 x 64 = 1024).
template <bool VT, bool COMMITS>
__global__ void __launch_bounds__(128, 1) step_bench(long long* out, int steps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t dummy[4];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(dummy + i, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t IDS = idesc_bf16(128, 128, false);
  constexpr uint32_t IDO = idesc_bf16(128, 128, !VT);
  if (warp == 1) {
    const uint32_t kb = __shfl_sync(0xffffffffu, smem_u32(base), 0);
    const uint32_t vb = kb + 32768;
    long long t0 = clock64();
    for (int j = 0; j < steps; ++j) {
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          mma_ts(tmem + (j & 1) * 128, tmem + 384 + k * 8, sw128_desc(kb + (k / 4) * 16384 + (k % 4) * 32, 16, 1024), IDS, k > 0);
        if (COMMITS) { tc_commit(dummy + 0); tc_commit(dummy + 1); }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t b = VT ? sw128_desc(vb + (k / 4) * 16384 + (k % 4) * 32, 16, 1024)
                                : sw128_desc(vb + k * 2048, 16384, 1024);
          mma_ts(tmem + 256, tmem + ((j + 1) & 1) * 128 + k * 8, b, IDO, 1);
        }
        if (COMMITS) { tc_commit(dummy + 2); tc_commit(dummy + 3); }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    if (threadIdx.x == 32) out[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <bool VT, bool COMMITS>
void run_step(const char* name) {
  long long* d;
  const int sms = 148, steps = 2048;
  cudaMalloc(&d, sms * sizeof(long long));
  auto k = step_bench<VT, COMMITS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  k<<<sms, 128, 100 * 1024>>>(d, steps);
  k<<<sms, 128, 100 * 1024>>>(d, steps);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  printf("%-34s cycles/step %7.1f (ideal 1024)  err=%s\n", name, avg / sms / steps,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// The ping-pong kernel's per-block MMA sequence for one slot: two S halves as SS
// MMAs (A = Q in shared memory, 128 x 128; B = 64 keys, N = 64) + commits, then
// two PV halves (TS, A = P in TMEM, B = V MN-major, K = 64 keys each) + commits.
// `slots` = 2 runs two such streams from two warps into disjoint TMEM columns.
template <int SLOTS>
__global__ void __launch_bounds__(128, 1) pp_bench(long long* out, int steps) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ __align__(8) uint64_t dummy[8];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar + 1, 1); for (int i = 0; i < 8; ++i) mbar_init(dummy + i, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  constexpr uint32_t IDS = idesc_bf16(128, 64, false);
  constexpr uint32_t IDO = idesc_bf16(128, 128, true);
  if (warp >= 1 && warp <= SLOTS) {
    const int s = warp - 1;
    const uint32_t qa = __shfl_sync(0xffffffffu, smem_u32(base + s * 98304), 0);
    const uint32_t kb = qa + 32768, vb = qa + 65536;
    const uint32_t tm = tmem + (uint32_t)(s * 256);
    long long t0 = clock64();
    for (int j = 0; j < steps; ++j) {
      if (elect_one()) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            mma_ss(tm + h * 64, sw128_desc(qa + (k / 4) * 16384 + (k % 4) * 32, 16, 1024),
                   sw128_desc(kb + h * 8192 + (k / 4) * 16384 + (k % 4) * 32, 16, 1024), IDS, k > 0);
          tc_commit(dummy + 4 * s + h);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ts(tm + 128, tm + h * 64 + k * 8, sw128_desc(vb + h * 8192 + k * 2048, 16384, 1024), IDO, 1);
          tc_commit(dummy + 4 * s + 2 + h);
        }
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(bar + s);
    __syncwarp();
    mbar_wait(bar + s, 0);
    if ((threadIdx.x & 31) == 0) out[blockIdx.x * 2 + s] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int SLOTS>
void run_pp(const char* name) {
  long long* d;
  const int sms = 148, steps = 2048;
  cudaMalloc(&d, 2 * sms * sizeof(long long));
  auto k = pp_bench<SLOTS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k<<<sms, 128, 200 * 1024>>>(d, steps);
  k<<<sms, 128, 200 * 1024>>>(d, steps);
  long long h[296];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[2 * i];
  printf("%-34s cycles/block/slot %7.1f (ideal %d)  err=%s\n", name, avg / sms / steps, 1024 * SLOTS,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run_pp<1>("ping-pong block, 1 slot");
  run_pp<2>("ping-pong block, 2 slots");
  run_step<false, true>("kernel step: V MN-major + commits");
  run_step<true, true>("kernel step: V^T K-major + commits");
  run_step<false, false>("kernel step: V MN-major, no commits");
  run_step<true, false>("kernel step: V^T K-major, no commits");
  int sms = 148;
  run<128, false, 1>("SS N=128", sms);
  run<128, true, 1>("TS N=128", sms);
  run<256, false, 1>("SS N=256", sms);
  run<256, true, 1>("TS N=256", sms);
  run<64, false, 1>("SS N=64", sms);
  run<128, false, 2>("SS N=128 2 accumulators", sms);
  run<128, true, 2>("TS N=128 2 accumulators", sms);
  run<128, false, 1>("SS N=128 (1 SM)", 1);
  run<128, false, 1, 8>("SS N=128 commit/8", sms);
  run<128, true, 1, 8>("TS N=128 commit/8", sms);
  run<128, false, 1, 16>("SS N=128 commit/16", sms);
  run<128, false, 1, 4>("SS N=128 commit/4", sms);
  run<128, false, 1, 0, 1>("SS N=128 B MN-major", sms);
  run<128, true, 1, 0, 1>("TS N=128 B MN-major", sms);
  run<128, true, 1, 0, 2>("TS N=128 S/PV alternating", sms);
  run<64, true, 1, 0, 1>("TS N=64 B MN-major", sms);
  run<128, true, 1, 0, 3>("TS K-major, 2 accs alt/8", sms);
  run<128, true, 1, 0, 4>("TS MN-major, 2 accs alt/8", sms);
  run<128, true, 1, 0, 5>("TS K/MN alt/8 same acc", sms);
  run<64, true, 1>("TS N=64 K-major", sms);
  run<64, true, 1, 0, 6>("64-key sub-step: 8 S N=64 + 4 PV N=128 (ideal/MMA: 8x32+4x64 over 12)", sms);
  return 0;
}
