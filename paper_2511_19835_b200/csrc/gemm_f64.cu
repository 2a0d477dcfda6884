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
// Tiling: BM x BN CTA tile of 32 x 32 warp tiles (4 x 4 DMMA 8x8 fragments
// each); K in steps of 16, staged k-major in shared memory ([k][m], row pitch
// BM + 8 doubles: the fragment loads of a warp hit every bank pair exactly
// twice = the 2-wavefront minimum for 256 bytes), double-buffered with the
// next k-tile prefetched into registers during the current MMAs.  Short-K
// problems (the scores GEMM, K = d) use 128-row tiles so each CTA's prologue
// is amortised over twice the MMAs.
#include "rsa_internal.cuh"

namespace rsa {
namespace {

constexpr int BK = 16;

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

// chunk c (8 consecutive k) of a ROWS x 16 tile stored k-contiguous in global
// memory (A, or B^T): row c / 2, k offset (c % 2) * 8
__device__ __forceinline__ void load_kmajor(const double* __restrict__ p, int64_t ld, int64_t rows, int64_t K,
                                            int64_t r0, int64_t k0, int c, double (&x)[8]) {
  const int64_t r = r0 + c / 2, k = k0 + (c % 2) * 8;
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

template <int PITCH>
__device__ __forceinline__ void store_kmajor(double* s, int c, const double (&x)[8]) {
  const int m = c / 2, kb = (c % 2) * 8;
#pragma unroll
  for (int i = 0; i < 8; ++i) s[(kb + i) * PITCH + m] = x[i];
}

// chunk c (8 consecutive n) of a 16 x COLS tile stored n-contiguous (B of NN):
// row k = c / (COLS / 8), n offset (c % (COLS / 8)) * 8
template <int COLS>
__device__ __forceinline__ void load_nmajor(const double* __restrict__ p, int64_t ld, int64_t cols, int64_t K,
                                            int64_t c0, int64_t k0, int c, double (&x)[8]) {
  const int64_t k = k0 + c / (COLS / 8), n = c0 + (c % (COLS / 8)) * 8;
  if (k < K && n + 8 <= cols && ((reinterpret_cast<uintptr_t>(p + k * ld + n) & 15) == 0)) {
    const double2* src = reinterpret_cast<const double2*>(p + k * ld + n);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 v = __ldg(src + i);
      x[2 * i] = v.x;
      x[2 * i + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = (k < K && n + i < cols) ? __ldg(p + k * ld + n + i) : 0.0;
  }
}

template <int PITCH, int COLS>
__device__ __forceinline__ void store_nmajor(double* s, int c, const double (&x)[8]) {
  double2* dst = reinterpret_cast<double2*>(s + (c / (COLS / 8)) * PITCH + (c % (COLS / 8)) * 8);
#pragma unroll
  for (int i = 0; i < 4; ++i) dst[i] = make_double2(x[2 * i], x[2 * i + 1]);
}

template <int BM, int BN, bool NT>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32) dgemm_kernel(GemmArgs a) {
  constexpr int WN = BN / 32;                   // warps along N
  constexpr int T = (BM / 32) * WN * 32;
  constexpr int PA = BM + 8, PB = BN + 8;       // shared-memory pitches (doubles)
  constexpr int CA = BM * BK / 8, CB = BN * BK / 8;   // 8-double chunks per tile
  constexpr int RA = (CA + T - 1) / T, RB = (CB + T - 1) / T;
  extern __shared__ __align__(16) double smem_d[];
  double* As[2] = {smem_d, smem_d + BK * PA};
  double* Bs[2] = {smem_d + 2 * BK * PA, smem_d + 2 * BK * PA + BK * PB};
  const int64_t b = blockIdx.z;
  const double* A = a.A + b * a.sA;
  const double* B = a.B + b * a.sB;
  double* C = a.C + b * a.sC;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;
  const int g = lane >> 2, tg = lane & 3;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double xa[RA][8], xb[RB][8];
  auto fetch = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < RA; ++r)
      if (t + r * T < CA) load_kmajor(A, a.lda, a.M, a.K, m0, k0, t + r * T, xa[r]);
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (t + r * T < CB) {
        if (NT) load_kmajor(B, a.ldb, a.N, a.K, n0, k0, t + r * T, xb[r]);
        else load_nmajor<BN>(B, a.ldb, a.N, a.K, n0, k0, t + r * T, xb[r]);
      }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int r = 0; r < RA; ++r)
      if (t + r * T < CA) store_kmajor<PA>(As[buf], t + r * T, xa[r]);
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (t + r * T < CB) {
        if (NT) store_kmajor<PB>(Bs[buf], t + r * T, xb[r]);
        else store_nmajor<PB, BN>(Bs[buf], t + r * T, xb[r]);
      }
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
      for (int i = 0; i < 4; ++i) fa[i] = as[(kk + tg) * PA + wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) fb[j] = bs[(kk + tg) * PB + wn + j * 8 + g];
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
      double* dst = C + r * a.ldc + c;
      if (c + 1 < a.N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < a.N) dst[0] = acc[i][j][0];
        if (c + 1 < a.N) dst[1] = acc[i][j][1];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Multistage variant (the default): cp.async 16-byte copies straight into
// shared memory, STAGES k-tiles in flight, no register staging.  A (and B^T)
// tiles stay m-major [m][k] (pitch BK + 2 doubles: a warp's fragment loads
// a[g][tg] hit each bank pair exactly twice), B of NN stays k-major [k][n]
// (pitch BN + 8).  Needs even leading dimensions (16-byte aligned rows of
// pairs); otherwise the register-staged kernel above runs.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes)
               : "memory");
}

template <int BM, int BN, bool NT, int STAGES>
__global__ void __launch_bounds__((BM / 32) * (BN / 32) * 32) dgemm_ms_kernel(GemmArgs a) {
  constexpr int WN = BN / 32;
  constexpr int T = (BM / 32) * WN * 32;
  constexpr int PK = BK + 2;                     // [m][k] pitch
  constexpr int PN = BN + 8;                     // [k][n] pitch
  constexpr int A_EL = BM * PK;
  constexpr int B_EL = NT ? BN * PK : BK * PN;
  extern __shared__ __align__(16) double smem_d[];
  const int64_t b = blockIdx.z;
  const double* A = a.A + b * a.sA;
  const double* B = a.B + b * a.sB;
  double* C = a.C + b * a.sC;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int t = threadIdx.x, warp = t / 32, lane = t % 32;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;
  const int g = lane >> 2, tg = lane & 3;

  auto stage_a = [&](int st) { return smem_d + st * (A_EL + B_EL); };
  auto stage_b = [&](int st) { return smem_d + st * (A_EL + B_EL) + A_EL; };
  // one k-tile: 16-byte pieces (2 doubles); out-of-range pieces zero-filled
  auto load = [&](int st, int64_t k0) {
    double* sa = stage_a(st);
    for (int c = t; c < BM * BK / 2; c += T) {
      const int m = c / (BK / 2), kp = (c % (BK / 2)) * 2;
      const int64_t r = m0 + m, k = k0 + kp;
      const int bytes = (r < a.M) ? (int)(max((int64_t)0, min((int64_t)2, a.K - k)) * 8) : 0;
      cp_async16(sa + m * PK + kp, bytes ? A + r * a.lda + k : A, bytes);
    }
    double* sb = stage_b(st);
    if (NT) {
      for (int c = t; c < BN * BK / 2; c += T) {
        const int n = c / (BK / 2), kp = (c % (BK / 2)) * 2;
        const int64_t r = n0 + n, k = k0 + kp;
        const int bytes = (r < a.N) ? (int)(max((int64_t)0, min((int64_t)2, a.K - k)) * 8) : 0;
        cp_async16(sb + n * PK + kp, bytes ? B + r * a.ldb + k : B, bytes);
      }
    } else {
      for (int c = t; c < BK * BN / 2; c += T) {
        const int kk = c / (BN / 2), np = (c % (BN / 2)) * 2;
        const int64_t k = k0 + kk, n = n0 + np;
        const int bytes = (k < a.K) ? (int)(max((int64_t)0, min((int64_t)2, a.N - n)) * 8) : 0;
        cp_async16(sb + kk * PN + np, bytes ? B + k * a.ldb + n : B, bytes);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t k_tiles = (a.K + BK - 1) / BK;
#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < k_tiles) load(st, st * BK);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int64_t kt = 0; kt < k_tiles; ++kt) {
    asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 2) : "memory");
    __syncthreads();   // k-tile kt landed for every thread; k-tile kt - 1's stage is free
    {
      const int64_t nx = kt + STAGES - 1;
      if (nx < k_tiles) load((int)(nx % STAGES), nx * BK);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    const double* as = stage_a((int)(kt % STAGES));
    const double* bs = stage_b((int)(kt % STAGES));
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double fa[4], fb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) fa[i] = as[(wm + i * 8 + g) * PK + kk + tg];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        fb[j] = NT ? bs[(wn + j * 8 + g) * PK + kk + tg] : bs[(kk + tg) * PN + wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], fa[i], fb[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + wm + i * 8 + g;
    if (r >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t c = n0 + wn + j * 8 + tg * 2;
      double* dst = C + r * a.ldc + c;
      if (c + 1 < a.N && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
        *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
      } else {
        if (c < a.N) dst[0] = acc[i][j][0];
        if (c + 1 < a.N) dst[1] = acc[i][j][1];
      }
    }
  }
}

template <int BM, int BN, int STAGES>
cudaError_t launch_ms(const GemmArgs& a, int64_t batch, bool nt, cudaStream_t st) {
  if (batch > 65535 || (a.M + BM - 1) / BM > 65535) return cudaErrorInvalidValue;
  constexpr int T = (BM / 32) * (BN / 32) * 32;
  const int smem = STAGES * (BM * (BK + 2) + (nt ? BN * (BK + 2) : BK * (BN + 8))) * 8;
  const dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + BM - 1) / BM), (unsigned)batch);
  auto kern = nt ? dgemm_ms_kernel<BM, BN, true, STAGES> : dgemm_ms_kernel<BM, BN, false, STAGES>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, T, smem, st>>>(a);
  return cudaGetLastError();
}

template <int BM, int BN>
cudaError_t launch_tiles(const GemmArgs& a, int64_t batch, bool nt, cudaStream_t st) {
  if (batch > 65535 || (a.M + BM - 1) / BM > 65535) return cudaErrorInvalidValue;
  constexpr int T = (BM / 32) * (BN / 32) * 32;
  constexpr int SMEM = 2 * BK * ((BM + 8) + (BN + 8)) * 8;
  const dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + BM - 1) / BM), (unsigned)batch);
  auto kern = nt ? dgemm_kernel<BM, BN, true> : dgemm_kernel<BM, BN, false>;
  if (SMEM > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, T, SMEM, st>>>(a);
  return cudaGetLastError();
}

// cfg: register-staged 1 = 64 x 64, 2 = 128 x 64, 3 = 64 x 128, 4 = 128 x 128;
// multistage 5 = 64 x 64 x 4 stages, 6 = 64 x 64 x 6, 7 = 128 x 64 x 4,
// 8 = 64 x 128 x 4; 0 = by shape
cudaError_t launch_dgemm_cfg(const GemmArgs& a, int64_t batch, bool nt, cudaStream_t st, int cfg) {
  const bool even = a.lda % 2 == 0 && a.ldb % 2 == 0 && a.sA % 2 == 0 && a.sB % 2 == 0 &&
                    (reinterpret_cast<uintptr_t>(a.A) & 15) == 0 && (reinterpret_cast<uintptr_t>(a.B) & 15) == 0;
  if (cfg == 0) cfg = even ? 5 : 1;
  if (cfg >= 5 && !even) cfg = 1;
  switch (cfg) {
    case 5: return launch_ms<64, 64, 4>(a, batch, nt, st);
    case 6: return launch_ms<64, 64, 6>(a, batch, nt, st);
    case 7: return launch_ms<128, 64, 4>(a, batch, nt, st);
    case 8: return launch_ms<64, 128, 4>(a, batch, nt, st);
    case 1: return launch_tiles<64, 64>(a, batch, nt, st);
    case 2: return launch_tiles<128, 64>(a, batch, nt, st);
    case 3: return launch_tiles<64, 128>(a, batch, nt, st);
    default: return launch_tiles<128, 128>(a, batch, nt, st);
  }
}

}  // namespace

cudaError_t launch_dgemm(int64_t batch, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         int64_t strideA, const double* B, int64_t ldb, int64_t strideB, bool b_transposed,
                         double* C, int64_t ldc, int64_t strideC, cudaStream_t st) {
  if (batch <= 0 || M <= 0 || N <= 0) return cudaSuccess;
  GemmArgs a{M, N, K, A, lda, strideA, B, ldb, strideB, C, ldc, strideC};
  return launch_dgemm_cfg(a, batch, b_transposed, st, 0);
}

}  // namespace rsa
