// K1: exactly rounded fp64 block pooling (HBM-bound streaming reduction).
//
// Reference: block_pool / block_sums (pkg/src/rectattn/core.py:154-189) use
// math.fsum per column, pool_problem (core.py:192-201) pools Q video blocks,
// K video blocks and all V blocks; _pool_rows (masks.py:130-135) pools the
// text keys per (possibly ragged) text block; pooling_error (masks.py:165-171)
// needs the deficits sum - len * mean.
//
// Layout: one CTA per (block, segment, head); 256 threads stream the block's
// rows with 128-bit non-allocating loads (8 bf16 / 4 f32 / 2 f64 per load),
// each thread owning a column chunk and a row phase.  For bf16/f32 data the
// sums are plain fp64 adds, proven exact per block from its magnitude range
// (see pass 1 below); otherwise (f64 data, or a block spanning too many
// binades) partial sums are (hi, lo) TwoSum pairs.  Either way the merged
// result is the exactly rounded sum, i.e. bit-identical to math.fsum, and
// independent of launch geometry.
#include "rsa_internal.cuh"

namespace rsa {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}

template <typename T, int VEC>
__device__ __forceinline__ void load_vec_f32(const T* p, float (&out)[VEC]) {
  if constexpr (VEC * sizeof(T) == 16) {
    uint4 raw;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w) : "l"(p));
    const T* v = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < VEC; ++i) out[i] = to_f32(v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) out[i] = to_f32(p[i]);
  }
}

template <typename T, int VEC>
__device__ __forceinline__ void load_vec(const T* p, double (&out)[VEC]) {
  if constexpr (VEC * sizeof(T) == 16) {
    uint4 raw;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(raw.x), "=r"(raw.y), "=r"(raw.z), "=r"(raw.w) : "l"(p));
    const T* v = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int i = 0; i < VEC; ++i) out[i] = to_f64(v[i]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) out[i] = to_f64(p[i]);
  }
}

// segment 0: Q video blocks, 1: K blocks (video + text), 2: V blocks
template <typename T, int VEC>
__global__ void __launch_bounds__(kThreads)
pool_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
            Workspace ws, Geometry g) {
  const int seg = blockIdx.y;
  const int64_t blk = blockIdx.x;
  const int64_t h = blockIdx.z;
  const int64_t nblocks = seg == 0 ? g.N : g.M;
  if (blk >= nblocks) return;
  const int64_t d = g.d;
  const int64_t row0 = blk * g.B;  // text blocks follow the video blocks contiguously
  const int64_t len = (blk < g.N) ? g.B : (blk == g.M - 1 ? g.last_len : g.B);
  const T* src = (seg == 0 ? q : seg == 1 ? k : v) + (h * g.T + row0) * d;

  __shared__ double s_hi[2048];
  __shared__ double s_lo[2048];

  const int tpr = (int)(d / VEC);          // threads per row
  const int rg_count = kThreads / tpr;     // row phases
  const int t = threadIdx.x;
  const int c = t % tpr;
  const int rg = t / tpr;
  const bool text_k = (seg == 1) && (blk >= g.N);
  double* raw_out = text_k ? ws.k_cat + (h * g.n_cols + g.N + (row0 - g.Tv)) * d : nullptr;

  // Pass 1 (bf16 / f32 data): plain fp64 sums plus the block's magnitude
  // range.  Every value is a multiple of 2^(e_min - p + 1) (p significant
  // bits), so all partial sums are exact in fp64 while
  //   e_max - e_min + p + ceil(log2(len)) < 53;
  // then the plain sums ARE the exactly rounded sums.  Otherwise (or for f64
  // data) pass 2 recomputes the block with TwoSum (hi, lo) pairs.
  constexpr bool kTryPlain = sizeof(T) < 8;
  constexpr int kMant = sizeof(T) == 2 ? 8 : 24;
  __shared__ float s_amax[kThreads / 32], s_amin[kThreads / 32];
  __shared__ int s_exact;
  bool exact = false;
  if constexpr (kTryPlain) {
    double acc[VEC];
    float amax = 0.f, amin = INFINITY;
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = 0.0;
    if (rg < rg_count) {
      int64_t r = rg;
      for (; r + 7 * rg_count < len; r += 8 * rg_count) {
        float x[8][VEC];
#pragma unroll
        for (int u = 0; u < 8; ++u) load_vec_f32<T, VEC>(src + (r + u * rg_count) * d + c * VEC, x[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
          for (int i = 0; i < VEC; ++i) {
            acc[i] += (double)x[u][i];
            const float ax = fabsf(x[u][i]);
            amax = fmaxf(amax, ax);
            amin = fminf(amin, ax > 0.f ? ax : INFINITY);
          }
          if (raw_out) {
#pragma unroll
            for (int i = 0; i < VEC; ++i) raw_out[(r + u * rg_count) * d + c * VEC + i] = (double)x[u][i];
          }
        }
      }
      for (; r < len; r += rg_count) {
        float x[VEC];
        load_vec_f32<T, VEC>(src + r * d + c * VEC, x);
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          acc[i] += (double)x[i];
          const float ax = fabsf(x[i]);
          amax = fmaxf(amax, ax);
          amin = fminf(amin, ax > 0.f ? ax : INFINITY);
        }
        if (raw_out) {
#pragma unroll
          for (int i = 0; i < VEC; ++i) raw_out[r * d + c * VEC + i] = (double)x[i];
        }
      }
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        s_hi[rg * d + i * tpr + c] = acc[i];   // column-interleaved: conflict-free
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      amin = fminf(amin, __shfl_xor_sync(0xffffffffu, amin, o));
    }
    if (t % 32 == 0) { s_amax[t / 32] = amax; s_amin[t / 32] = amin; }
    __syncthreads();
    if (t == 0) {
      float mx = 0.f, mn = INFINITY;
      for (int w = 0; w < kThreads / 32; ++w) { mx = fmaxf(mx, s_amax[w]); mn = fminf(mn, s_amin[w]); }
      int lg = 0;
      while ((int64_t(1) << lg) < len) ++lg;
      s_exact = (mn == INFINITY) || (ilogbf(mx) - ilogbf(mn) + kMant + lg < 53);
    }
    __syncthreads();
    exact = s_exact != 0;
  }
  if (!exact) {
    double hi[VEC], lo[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) { hi[i] = 0.0; lo[i] = 0.0; }
    if (rg < rg_count) {
      for (int64_t r = rg; r < len; r += rg_count) {
        double x[VEC];
        load_vec<T, VEC>(src + r * d + c * VEC, x);
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          double sm, e;
          two_sum(hi[i], x[i], sm, e);
          hi[i] = sm;
          lo[i] += e;
        }
        if (raw_out && !kTryPlain) {
#pragma unroll
          for (int i = 0; i < VEC; ++i) raw_out[r * d + c * VEC + i] = x[i];
        }
      }
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        s_hi[rg * d + i * tpr + c] = hi[i];
        s_lo[rg * d + i * tpr + c] = lo[i];
      }
    }
  }
  __syncthreads();

  for (int64_t col = t; col < d; col += kThreads) {
    const int64_t slot = (col % VEC) * tpr + col / VEC;
    double sum;
    if (exact) {
      sum = 0.0;   // exact partial sums: plain adds stay exact (same bound)
      for (int p = 0; p < rg_count; ++p) sum += s_hi[p * d + slot];
    } else {
      double S = 0.0, E = 0.0;
      for (int p = 0; p < rg_count; ++p) {
        double s, e;
        two_sum(S, s_hi[p * d + slot], s, e);
        S = s;
        E += e + s_lo[p * d + slot];
      }
      sum = S + E;                            // exactly rounded block sum
    }
    const double flen = (double)len;
    const double mean = sum / flen;           // core.py:172 fsum(...) / length
    const double deficit = sum - flen * mean; // masks.py:166 / masks.py:171
    if (seg == 0) {
      ws.q_pool[(h * g.N + blk) * d + col] = mean;
      ws.q_def[(h * g.N + blk) * d + col] = deficit;
    } else if (seg == 1) {
      const int64_t kc_row = blk < g.N ? blk : g.N + g.Tt + (blk - g.N);
      ws.k_cat[(h * g.n_cols + kc_row) * d + col] = mean;
      ws.k_def[(h * g.M + blk) * d + col] = deficit;
    } else {
      ws.v_pool[(h * g.M + blk) * d + col] = mean;
    }
    if (seg < 2 && deficit != 0.0) atomicOr(ws.status + ST_DEFICIT, 1);
  }
}

template <typename T>
cudaError_t launch_typed(const Geometry& g, const void* q, const void* k, const void* v,
                         const Workspace& ws, cudaStream_t st) {
  dim3 grid((unsigned)g.M, 3, (unsigned)g.H);
  constexpr int V16 = 16 / sizeof(T);
  const bool aligned = (g.d % V16 == 0) && ((uintptr_t)q % 16 == 0) &&
                       ((uintptr_t)k % 16 == 0) && ((uintptr_t)v % 16 == 0);
  if (aligned && g.d / V16 <= kThreads && (kThreads / (g.d / V16)) * g.d <= 2048) {
    pool_kernel<T, V16><<<grid, kThreads, 0, st>>>((const T*)q, (const T*)k, (const T*)v, ws, g);
  } else {
    pool_kernel<T, 1><<<grid, kThreads, 0, st>>>((const T*)q, (const T*)k, (const T*)v, ws, g);
  }
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_pool(const Geometry& g, const void* q, const void* k, const void* v,
                        const Workspace& ws, cudaStream_t st, int* launches) {
  ++*launches;
  switch (g.dtype) {
    case RSA_BF16: return launch_typed<__nv_bfloat16>(g, q, k, v, ws, st);
    case RSA_F32: return launch_typed<float>(g, q, k, v, ws, st);
    default: return launch_typed<double>(g, q, k, v, ws, st);
  }
}

}  // namespace rsa
