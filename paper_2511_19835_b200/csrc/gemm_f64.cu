// fp64 batched GEMM on the DMMA tensor cores (mma.sync m8n8k4 .f64), for
// K2's two plain GEMMs and the validation diagnostics:
//   scores[n][c]  = q_pool[n][:] . k_cat[c][:]          NT  (ipar.py:41, masks.py:120-127)
//   comp[n][:]    = sum_m a_applied[n][m] v_pool[m][:]   NN  (rectify.py:84-87)
// Row-major operands with leading dimensions and batch strides:
//   C[b] (M x N) = A[b] (M x K) . op(B[b]),  op(B) = B^T (B is N x K) or B (K x N).
// Every product and sum is an IEEE fp64 operation (DMMA is an exact-product,
// fp64-accumulate FMA chain), so the result differs from numpy/OpenBLAS only
// by summation order -- the same freedom cuBLAS had; the downstream masks are
// bit-exact by margin (k-th gaps >= 1e-7 relative vs ~1e-16).
//
// Tiling: 64 x 64 CTA tile, 4 warps in 2 x 2, each a 32 x 32 warp tile of
// 4 x 4 DMMA 8x8 fragments; K in steps of 16, staged k-major in shared memory
// ([k][m], row pitch 72 doubles: the fragment loads of a warp hit every bank
// pair exactly twice = the 2-wavefront minimum for 256 bytes), double-buffered
// with the next k-tile prefetched into registers during the current MMAs.
#include "rsa_internal.cuh"

namespace rsa {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, PITCH = 72, GT = 128;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}

struct GemmArgs {
  int64_t M, N, K;
  const double* A; int64_t lda, sA;
  const double* B; int64_t ldb, sB;
  double* C; int64_t ldc, sC;
};

// one thread's share of a 64 x 16 tile stored k-contiguous in global memory
// (A, or B^T): row r = t / 2, eight consecutive k from (t % 2) * 8
__device__ __forceinline__ void load_kmajor(const double* __restrict__ p, int64_t ld, int64_t rows, int64_t K,
                                            int64_t r0, int64_t k0, double (&x)[8]) {
  const int t = threadIdx.x;
  const int64_t r = r0 + t / 2, k = k0 + (t % 2) * 8;
  if (r < rows && k + 8 <= K && ((reinterpret_cast<uintptr_t>(p + r * ld + k) & 15) == 0)) {
    const double2* src = reinterpret_cast<const double2*>(p + r * ld + k);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 v = __ldg(src + i);
      x[2 * i] = v.x;
      x[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (r < rows && k + i < K) ? __ldg(p + r * ld + k + i) : 0.0;
  }
}

__device__ __forceinline__ void store_kmajor(double* s, const double (&x)[8]) {
  const int t = threadIdx.x;
  const int m = t / 2, kb = (t % 2) * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) s[(kb + i) * PITCH + m] = x[i];
}

// one thread's share of a 16 x 64 tile stored n-contiguous (B of NN): row
// k = t / 8, eight consecutive n from (t % 8) * 8
__device__ __forceinline__ void load_nmajor(const double* __restrict__ p, int64_t ld, int64_t cols, int64_t K,
                                            int64_t c0, int64_t k0, double (&x)[8]) {
  const int t = threadIdx.x;
  const int64_t k = k0 + t / 8, c = c0 + (t % 8) * 8;
  if (k < K && c + 8 <= cols && ((reinterpret_cast<uintptr_t>(p + k * ld + c) & 15) == 0)) {
    const double2* src = reinterpret_cast<const double2*>(p + k * ld + c);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 v = __ldg(src + i);
      x[2 * i] = v.x;
      x[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (k < K && c + i < cols) ? __ldg(p + k * ld + c + i) : 0.0;
  }
}

__device__ __forceinline__ void store_nmajor(double* s, const double (&x)[8]) {
  const int t = threadIdx.x;
  double2* dst = reinterpret_cast<double2*>(s + (t / 8) * PITCH + (t % 8) * 8);
#pragma unroll
  for (int i = 0; i < 4; ++i) dst[i] = make_double2(x[2 * i], x[2 * i + 1]);
}

template <bool NT>
__global__ void __launch_bounds__(GT) dgemm_kernel(GemmArgs a) {
  __shared__ __align__(16) double As[2][BK * PITCH];
  __shared__ __align__(16) double Bs[2][BK * PITCH];
  const int64_t b = blockIdx.z;
  const double* A = a.A + b * a.sA;
  const double* B = a.B + b * a.sB;
  double* C = a.C + b * a.sC;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int g = lane >> 2, tg = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double xa[8], xb[8];
  auto fetch = [&](int64_t k0) {
    load_kmajor(A, a.lda, a.M, a.K, m0, k0, xa);
    if (NT) load_kmajor(B, a.ldb, a.N, a.K, n0, k0, xb);
    else load_nmajor(B, a.ldb, a.N, a.K, n0, k0, xb);
  };
  auto stash = [&](int buf) {
    store_kmajor(As[buf], xa);
    if (NT) store_kmajor(Bs[buf], xb);
    else store_nmajor(Bs[buf], xb);
  };
  const int64_t k_tiles = (a.K + BK - 1) / BK;
  fetch(0);
  stash(0);
  __syncthreads();
  for (int64_t kt = 0; kt < k_tiles; ++kt) {
    const int buf = (int)(kt & 1);
    if (kt + 1 < k_tiles) fetch((kt + 1) * BK);
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = as[(kk + tg) * PITCH + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = bs[(kk + tg) * PITCH + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
    if (kt + 1 < k_tiles) stash(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm + i * 8 + g;
    if (r >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + wn + j * 8 + tg * 2;
      if (c < a.N) C[r * a.ldc + c] = acc[i][j][0];
      if (c + 1 < a.N) C[r * a.ldc + c + 1] = acc[i][j][1];
    }
  }
}

}  // namespace

cudaError_t launch_dgemm(int64_t batch, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         int64_t strideA, const double* B, int64_t ldb, int64_t strideB, bool b_transposed,
                         double* C, int64_t ldc, int64_t strideC, cudaStream_t st) {
  if (batch <= 0 || M <= 0 || N <= 0) return cudaSuccess;
  if (batch > 65535 || (M + BM - 1) / BM > 65535) return cudaErrorInvalidValue;
  GemmArgs a{M, N, K, A, lda, strideA, B, ldb, strideB, C, ldc, strideC};
  const dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)batch);
  if (b_transposed) dgemm_kernel<true><<<grid, GT, 0, st>>>(a);
  else dgemm_kernel<false><<<grid, GT, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace rsa
