// Rate of the paired-tile softmax's exp loop on sm_100a, per SMSP, at 1 and 2
// warps per SMSP: per column pair FFMA2 (scale, -base), 2x ex2.approx.ftz.f32
// (MUFU), FADD2 (row sum) and cvt.rn.bf16x2 (F2FP pack), 64 pairs per row.
// MODE 1 adds the FMA-pipe polynomial for POLY of every 16 pairs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2511_19835_b200/csrc -o exp_loop_bench exp_loop_bench.cu
#include <cstdio>
#include <cstdint>
#include "tc_ptx.cuh"

using namespace rsa;

// VAR: 0 full loop, 1 pack by PRMT (no F2FP), 2 no row sum, 3 no pack and no sum,
//      4 phased: all FFMA2 of a chunk, then all ex2, then packs and sums
//      5 software-pipelined: pack/sum of pair i after the ex2 of pair i + LAG (asm volatile order)
template <int LAG>
__device__ __forceinline__ void exp_pipelined(float* v, float2 sc2, float2 nb2, float2* sum2, uint32_t* pk) {
  // v[32]: scores in, 2^x in place; pk[16] bf16 pairs; FFMA2 two pairs ahead, pack/sum LAG pairs behind
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float2 x = ptx::ffma2(make_float2(v[2 * i], v[2 * i + 1]), sc2, nb2);
    v[2 * i] = x.x; v[2 * i + 1] = x.y;
  }
#pragma unroll
  for (int i = 0; i < 16 + LAG; ++i) {
    if (i < 16) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[2 * i]));
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(v[2 * i + 1]));
    }
    if (i + 2 < 16) {
      const float2 x = ptx::ffma2(make_float2(v[2 * i + 4], v[2 * i + 5]), sc2, nb2);
      v[2 * i + 4] = x.x; v[2 * i + 5] = x.y;
    }
    if (i >= LAG) {
      const int q = i - LAG;
      uint32_t r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(v[2 * q + 1]), "f"(v[2 * q]));
      pk[q] = r;
      sum2[q & 1] = ptx::fadd2(sum2[q & 1], make_float2(v[2 * q], v[2 * q + 1]));
    }
  }
}

template <int POLY, int VAR = 0>
__global__ void k(const float* in, uint32_t* out, int iters) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = in[(threadIdx.x + i) & 1023];
  float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
  uint32_t acc = 0;
  const float2 sc2 = make_float2(0.088f, 0.088f), nb2 = make_float2(-3.f, -3.f);
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t pk[16];
      if (VAR >= 6) {
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = s[32 * c + i];
        if (VAR == 6) exp_pipelined<2>(v, sc2, nb2, sum2, pk);
        if (VAR == 7) exp_pipelined<3>(v, sc2, nb2, sum2, pk);
        if (VAR == 8) exp_pipelined<4>(v, sc2, nb2, sum2, pk);
      } else if (VAR == 5) {
        constexpr int LAG = 2;
        float2 xs[16], ps[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) xs[i] = ptx::ffma2(make_float2(s[32 * c + 2 * i], s[32 * c + 2 * i + 1]), sc2, nb2);
#pragma unroll
        for (int i = 0; i < 16 + LAG; ++i) {
          if (i < 16) {
            float a = xs[i].x, b = xs[i].y;
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
            asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(b));
            ps[i] = make_float2(a, b);
          }
          if (i >= LAG) {
            const int q = i - LAG;
            uint32_t r;
            asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(ps[q].y), "f"(ps[q].x));
            pk[q] = r;
            sum2[q & 1] = ptx::fadd2(sum2[q & 1], ps[q]);
          }
        }
      } else if (VAR == 4) {
        float xv[32];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ptx::ffma2(make_float2(s[32 * c + 2 * i], s[32 * c + 2 * i + 1]), sc2, nb2);
          xv[2 * i] = x.x; xv[2 * i + 1] = x.y;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(xv[i]));
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 p = make_float2(xv[2 * i], xv[2 * i + 1]);
          sum2[i & 1] = ptx::fadd2(sum2[i & 1], p);
          pk[i] = ptx::pack_bf16(p.x, p.y);
        }
      } else
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 x = ptx::ffma2(make_float2(s[32 * c + 2 * i], s[32 * c + 2 * i + 1]), sc2, nb2);
        const float2 p = (i < POLY) ? ptx::ex2_poly2(x) : make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
        if (VAR == 0 || VAR == 1) sum2[i & 1] = ptx::fadd2(sum2[i & 1], p);
        if (VAR == 0 || VAR == 2) pk[i] = ptx::pack_bf16(p.x, p.y);
        else if (VAR == 1) pk[i] = __byte_perm(__float_as_uint(p.x), __float_as_uint(p.y), 0x7632);
        else pk[i] = __float_as_uint(p.x) ^ __float_as_uint(p.y);
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) acc ^= pk[i];
    }
    s[it & 127] += 1e-7f;
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(sum2[0].x + sum2[1].y);
  if (threadIdx.x == 0 && blockIdx.x == 0) printf("  cycles per row-block (128 exps) per warp: %.0f\n", (double)(t1 - t0) / iters);
}

int main() {
  float* in; uint32_t* out;
  cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0, 4096 * 4);
  cudaMalloc(&out, 148 * 1024 * 4);
  for (int warps : {4, 8}) {
    printf("warps/SM %d (%d per SMSP), plain ex2:\n", warps, warps / 4);
    k<0><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, pack by PRMT:\n", warps);
    k<0, 1><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, no row sum:\n", warps);
    k<0, 2><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, no pack, no sum:\n", warps);
    k<0, 3><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, phased (FFMA2s, ex2s, packs):\n", warps);
    k<0, 4><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, software-pipelined lag 2:\n", warps);
    k<0, 5><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, in-place pipelined lag 2:\n", warps);
    k<0, 6><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, in-place pipelined lag 3:\n", warps);
    k<0, 7><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, in-place pipelined lag 4:\n", warps);
    k<0, 8><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, poly 2/16:\n", warps);
    k<2><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
    printf("warps/SM %d, poly 4/16:\n", warps);
    k<4><<<148, warps * 32>>>(in, out, 2000); cudaDeviceSynchronize();
  }
  return 0;
}
