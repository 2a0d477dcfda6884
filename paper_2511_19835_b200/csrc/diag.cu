// Validation diagnostics on the GPU (quadratic in sequence length; fp64 like
// the reference):
//   gain_error(..., with_exact=True)   masks.py:189-219   relaxed + exact GAPR forms
//   gapr_condition_agreement           metrics.py:116-124 (from the four arrays)
//   denominator_equivalence_report     metrics.py:90-113  s_sum, s_sum_pool
// Per head: Q/K converted to fp64, S = Q K^T for a chunk of query blocks by a
// cuBLAS DGEMM (a plain library GEMM), then our kernels: per-row max and
// sum of exp((S/sqrt d) - max) (the full-attention softmax of core.py:211-225),
// the denominators, and per (query block, kv block) sum |w_ij - a_tok[n,m]|.
// Needs rsa_pool + rsa_select on the workspace (pooled scores, deficits).
#include "rsa_internal.cuh"


#include <algorithm>
#include <cfloat>

namespace rsa {
namespace {

constexpr int DT = 256;

__device__ double block_reduce_sum(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  double y = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < DT / 32; ++i) y += red[i];   // fixed order
  if (threadIdx.x == 0) red[0] = y;
  __syncthreads();
  return red[0];
}
__device__ double block_reduce_max(double x, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double y = -DBL_MAX;
    for (int i = 0; i < DT / 32; ++i) y = fmax(y, red[i]);
    red[0] = y;
  }
  __syncthreads();
  return red[0];
}

// (the diagnostics reject a ragged final video block, capi.cu)
__device__ __forceinline__ double kv_lenf(const Geometry& g, int64_t m) { return (double)kv_len(g, m); }
// pooled score s_pool[n][m] (masks.py:120-127): video columns, then pooled text
__device__ __forceinline__ double s_pool(const Geometry& g, const double* srow, int64_t m) {
  return m < g.N ? srow[m] : srow[g.N + g.Tt + (m - g.N)];
}

template <typename T>
__global__ void to_f64_kernel(const T* __restrict__ src, double* __restrict__ dst, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = to_f64(src[i]);
}

// one CTA per query block n of head h: token-level pooled map a_tok, exact
// gain B len a_tok, relaxed gain |B len s_pool| and error (masks.py:138-176)
__global__ void __launch_bounds__(DT) diag_pooled_kernel(Workspace ws, Geometry g, int64_t h, double* a_tok,
                                                         double* exact_gain, double* gain, double* error,
                                                         double* pmax_out, double inv_sqrt_d) {
  __shared__ double red[DT / 32];
  const int64_t n = blockIdx.x, M = g.M;
  const double* srow = ws.scores + (h * g.N + n) * g.n_cols;
  double mx = -DBL_MAX;
  for (int64_t m = threadIdx.x; m < M; m += DT) mx = fmax(mx, s_pool(g, srow, m));
  mx = block_reduce_max(mx, red);
  double part = 0.0;
  for (int64_t m = threadIdx.x; m < M; m += DT) part += exp(s_pool(g, srow, m) - mx) * kv_len(g, m);
  const double denom = block_reduce_sum(part, red);
  const bool deficit = ws.status[ST_DEFICIT] != 0;
  const int64_t d = g.d;
  for (int64_t m = threadIdx.x; m < M; m += DT) {
    const double len = kv_lenf(g, m), s = s_pool(g, srow, m);
    const double at = exp(s - mx) / denom;
    a_tok[n * M + m] = at;
    exact_gain[(h * g.N + n) * M + m] = (double)g.B * len * at;
    gain[(h * g.N + n) * M + m] = fabs(((double)g.B * len) * s);
    double err = 0.0;
    if (deficit) {
      const int64_t krow = (m < g.N) ? m : g.N + g.Tt + (m - g.N);
      const double* kp = ws.k_cat + (h * g.n_cols + krow) * d;
      const double* kd = ws.k_def + (h * M + m) * d;
      const double* qp = ws.q_pool + (h * g.N + n) * d;
      const double* qd = ws.q_def + (h * g.N + n) * d;
      double d1 = 0.0, d2 = 0.0;
      for (int64_t c = 0; c < d; ++c) { d1 = fma(qd[c], kp[c], d1); d2 = fma(qp[c], kd[c], d2); }
      err = fabs((d1 * len) * inv_sqrt_d + ((double)g.B * d2) * inv_sqrt_d);
    }
    error[(h * g.N + n) * M + m] = err;
  }
  if (threadIdx.x == 0) pmax_out[n] = mx;
}

// one CTA per token row of the chunk: row max and sum of exp of S/sqrt(d)
// (core.py:204-208), then the denominators of metrics.py:103-108
__global__ void __launch_bounds__(DT) diag_row_kernel(const double* __restrict__ S, Workspace ws, Geometry g,
                                                      int64_t h, int64_t row0, const double* pmax,
                                                      double* rmax, double* rsum, double* s_sum,
                                                      double* s_sum_pool, double sqrt_d) {
  __shared__ double red[DT / 32];
  const int64_t r = blockIdx.x;               // row within the chunk
  const int64_t i = row0 + r;                 // video token
  const int64_t n = i / g.B;
  const double* srow = S + r * g.T;
  double mx = -DBL_MAX;
  for (int64_t j = threadIdx.x; j < g.T; j += DT) mx = fmax(mx, srow[j] / sqrt_d);
  mx = block_reduce_max(mx, red);
  double part = 0.0;
  for (int64_t j = threadIdx.x; j < g.T; j += DT) part += exp(srow[j] / sqrt_d - mx);
  const double sum = block_reduce_sum(part, red);
  const double shift = fmax(mx, pmax[n]);
  const double* prow = ws.scores + (h * g.N + n) * g.n_cols;
  double pp = 0.0;
  for (int64_t m = threadIdx.x; m < g.M; m += DT) pp += kv_lenf(g, m) * exp(s_pool(g, prow, m) - shift);
  const double pooled = block_reduce_sum(pp, red);
  if (threadIdx.x == 0) {
    rmax[r] = mx;
    rsum[r] = sum;
    s_sum[h * g.Tv + i] = sum * exp(mx - shift);
    s_sum_pool[h * g.Tv + i] = pooled;
  }
}

// one CTA per (kv block m, query block n of the chunk): sum over the block's
// token pairs of |w_ij - a_tok[n][m]|, w = softmax row (masks.py:214-218)
__global__ void __launch_bounds__(DT) diag_err_kernel(const double* __restrict__ S, Geometry g, int64_t h,
                                                      int64_t n0, const double* rmax, const double* rsum,
                                                      const double* a_tok, double* exact_error, double sqrt_d) {
  __shared__ double red[DT / 32];
  const int64_t m = blockIdx.x, nl = blockIdx.y, n = n0 + nl;
  const int64_t len = kv_len(g, m), start = kv_row0(g, m);
  const double a = a_tok[n * g.M + m];
  double part = 0.0;
  for (int64_t idx = threadIdx.x; idx < g.B * len; idx += DT) {
    const int64_t rr = nl * g.B + idx / len, j = start + idx % len;
    const double w = exp(S[rr * g.T + j] / sqrt_d - rmax[rr]) / rsum[rr];
    part += fabs(w - a);
  }
  const double tot = block_reduce_sum(part, red);
  if (threadIdx.x == 0) exact_error[(h * g.N + n) * g.M + m] = tot;
}

// softmax rows in place: W = exp(S/sqrt d - max) / sum  (core.py:204-208, 223-224)
__global__ void __launch_bounds__(DT) softmax_rows_kernel(double* __restrict__ S, int64_t T, double sqrt_d) {
  __shared__ double red[DT / 32];
  double* row = S + (int64_t)blockIdx.x * T;
  double mx = -DBL_MAX;
  for (int64_t j = threadIdx.x; j < T; j += DT) {
    const double s = row[j] / sqrt_d;
    row[j] = s;
    mx = fmax(mx, s);
  }
  mx = block_reduce_max(mx, red);
  double part = 0.0;
  for (int64_t j = threadIdx.x; j < T; j += DT) {
    const double e = exp(row[j] - mx);
    row[j] = e;
    part += e;
  }
  const double sum = block_reduce_sum(part, red);
  for (int64_t j = threadIdx.x; j < T; j += DT) row[j] = row[j] / sum;
}

}  // namespace

int64_t diag_chunk_blocks(const Geometry& g) {
  const int64_t per_block = g.B * g.T * 8;
  return std::max<int64_t>(1, std::min<int64_t>(g.N, ((int64_t)1 << 30) / per_block));
}

size_t diag_scratch_size(const Geometry& g) {
  const int64_t nc = diag_chunk_blocks(g);
  return (size_t)(g.T * g.d + g.Tv * g.d + nc * g.B * g.T + 2 * nc * g.B + g.N * g.M + g.N) * 8 + 1024;
}

cudaError_t launch_diagnostics(const Geometry& g, const void* q, const void* k, const Workspace& ws,
                               double* gain, double* error, double* exact_gain, double* exact_error,
                               double* s_sum, double* s_sum_pool, void* scratch, cudaStream_t st) {
  const int64_t nc = diag_chunk_blocks(g);
  double* k64 = static_cast<double*>(scratch);
  double* q64 = k64 + g.T * g.d;
  double* S = q64 + g.Tv * g.d;
  double* rmax = S + nc * g.B * g.T;
  double* rsum = rmax + nc * g.B;
  double* a_tok = rsum + nc * g.B;
  double* pmax = a_tok + g.N * g.M;
  const double sqrt_d = sqrt((double)g.d);
  const size_t esz = g.dtype == RSA_BF16 ? 2 : g.dtype == RSA_F32 ? 4 : 8;
  auto convert = [&](const void* src, double* dst, int64_t n) {
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (g.dtype == RSA_BF16) to_f64_kernel<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), dst, n);
    else if (g.dtype == RSA_F32) to_f64_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(src), dst, n);
    else to_f64_kernel<<<blocks, 256, 0, st>>>(static_cast<const double*>(src), dst, n);
  };
  for (int64_t h = 0; h < g.H; ++h) {
    convert(static_cast<const char*>(k) + (size_t)h * g.T * g.d * esz, k64, g.T * g.d);
    convert(static_cast<const char*>(q) + (size_t)h * g.T * g.d * esz, q64, g.Tv * g.d);
    diag_pooled_kernel<<<(unsigned)g.N, DT, 0, st>>>(ws, g, h, a_tok, exact_gain, gain, error, pmax, 1.0 / sqrt_d);
    for (int64_t n0 = 0; n0 < g.N; n0 += nc) {
      const int64_t cn = std::min(nc, g.N - n0), rows = cn * g.B;
      // S (row-major rows x T) = q64[rows] . k64^T
      cudaError_t e = launch_dgemm(1, rows, g.T, g.d, q64 + n0 * g.B * g.d, g.d, 0, k64, g.d, 0, true, S, g.T, 0, st);
      if (e != cudaSuccess) return e;
      diag_row_kernel<<<(unsigned)rows, DT, 0, st>>>(S, ws, g, h, n0 * g.B, pmax, rmax, rsum, s_sum, s_sum_pool,
                                                      sqrt_d);
      diag_err_kernel<<<dim3((unsigned)g.M, (unsigned)cn), DT, 0, st>>>(S, g, h, n0, rmax, rsum, a_tok,
                                                                       exact_error, sqrt_d);
    }
  }
  return cudaGetLastError();
}

size_t dense_scratch_size(const Geometry& g) {
  const int64_t nc = diag_chunk_blocks(g);
  return (size_t)(3 * g.T * g.d + nc * g.B * g.T) * 8 + 1024;
}

// Dense fp64 attention of every query row (video and text) over all keys:
// the reference's ground truth full_attention_oracle (core.py:211-225).
cudaError_t launch_dense_reference(const Geometry& g, const void* q, const void* k, const void* v, double* out,
                                   void* scratch, cudaStream_t st) {
  const int64_t rows_per = diag_chunk_blocks(g) * g.B;
  double* k64 = static_cast<double*>(scratch);
  double* v64 = k64 + g.T * g.d;
  double* q64 = v64 + g.T * g.d;
  double* W = q64 + g.T * g.d;
  const double sqrt_d = sqrt((double)g.d);
  const size_t esz = g.dtype == RSA_BF16 ? 2 : g.dtype == RSA_F32 ? 4 : 8;
  auto convert = [&](const void* src, double* dst, int64_t n) {
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (g.dtype == RSA_BF16) to_f64_kernel<<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(src), dst, n);
    else if (g.dtype == RSA_F32) to_f64_kernel<<<blocks, 256, 0, st>>>(static_cast<const float*>(src), dst, n);
    else to_f64_kernel<<<blocks, 256, 0, st>>>(static_cast<const double*>(src), dst, n);
  };
  for (int64_t h = 0; h < g.H; ++h) {
    const size_t off = (size_t)h * g.T * g.d * esz;
    convert(static_cast<const char*>(k) + off, k64, g.T * g.d);
    convert(static_cast<const char*>(v) + off, v64, g.T * g.d);
    convert(static_cast<const char*>(q) + off, q64, g.T * g.d);
    for (int64_t r0 = 0; r0 < g.T; r0 += rows_per) {
      const int64_t rows = std::min(rows_per, g.T - r0);
      // W (row-major rows x T) = q64[rows] . k64^T
      cudaError_t e = launch_dgemm(1, rows, g.T, g.d, q64 + r0 * g.d, g.d, 0, k64, g.d, 0, true, W, g.T, 0, st);
      if (e != cudaSuccess) return e;
      softmax_rows_kernel<<<(unsigned)rows, DT, 0, st>>>(W, g.T, sqrt_d);
      // out rows (row-major rows x d) = W (rows x T) . V (T x d)
      e = launch_dgemm(1, rows, g.d, g.T, W, g.T, 0, v64, g.d, 0, false, out + (h * g.T + r0) * g.d, g.d, 0, st);
      if (e != cudaSuccess) return e;
    }
  }
  return cudaGetLastError();
}

}  // namespace rsa
