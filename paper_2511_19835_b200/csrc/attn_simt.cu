// K3 (CUDA-core variant): block-sparse online-softmax attention for shapes
// the tcgen05 kernel does not cover (any block size, head_dim <= 256, and the
// reference's fp32 / fp64 precisions), with the rectification epilogue.
//
// Reference: _query_block_pass / block_sparse_attention / text_full_attention
// (pkg/src/rectattn/kernel.py:43-145): per query block, running max,
// denominator and accumulator over the retained kv blocks in ascending order,
// scores (q k^T) * dtype(1/sqrt d), out = acc / denom, lse = ln(denom) + max;
// apply_rectification (rectify.py:66-89): out' = R_n out + comp_n in fp64, cast
// back to the input dtype.
//
// Layout: CTA = 32 query rows of one head (4 warps x 8 rows); kv blocks are
// streamed through shared memory in 32-key chunks; lane j owns key j of a
// chunk for the scores and dims {lane + 32 i} of the accumulator.
#include "rsa_internal.cuh"

#include <cfloat>

namespace rsa {
namespace {

constexpr int QT = 32, KC = 32, WARPS = 4, RPW = QT / WARPS;

template <typename A> __device__ __forceinline__ A ex(A x);
template <> __device__ __forceinline__ float ex<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double ex<double>(double x) { return exp(x); }

template <typename A> __device__ __forceinline__ A warp_max_t(A x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
template <typename A> __device__ __forceinline__ A warp_sum_t(A x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <typename T> __device__ __forceinline__ typename Acc<T>::type ld_acc(const T* p) {
  return (typename Acc<T>::type)to_f64(*p);
}
template <> __device__ __forceinline__ float ld_acc<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <> __device__ __forceinline__ float ld_acc<float>(const float* p) { return *p; }

template <typename T> __device__ __forceinline__ T cast_out(double x);
template <> __device__ __forceinline__ __nv_bfloat16 cast_out<__nv_bfloat16>(double x) {
  return __float2bfloat16_rn((float)x);
}
template <> __device__ __forceinline__ float cast_out<float>(double x) { return (float)x; }
template <> __device__ __forceinline__ double cast_out<double>(double x) { return x; }

// text == false: tiles walk ws.kv_list of their query block; text == true:
// tiles of text queries walk every kv block (text_full_attention).
template <typename T, int DPL>
__global__ void __launch_bounds__(QT * WARPS)
attn_simt_kernel(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                 T* __restrict__ out, float* __restrict__ lse, Workspace ws, Geometry g,
                 bool rectify, bool text, typename Acc<T>::type scale) {
  using A = typename Acc<T>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int64_t d = g.d, ld = d + 1;
  A* qs = reinterpret_cast<A*>(smem_raw);
  A* ks = qs + QT * ld;
  A* vs = ks + KC * ld;

  // ---- tile -> (head, row range, kv list) ----
  int64_t h, row0, nrows, n = -1;
  if (!text) {
    const int64_t subs = (g.B + QT - 1) / QT;
    const int64_t per_head = g.N * subs;
    h = blockIdx.x / per_head;
    const int64_t rem = blockIdx.x % per_head;
    n = rem / subs;
    const int64_t sub = rem % subs;
    row0 = n * g.B + sub * QT;
    nrows = min((int64_t)QT, q_len(g, n) - sub * QT);
    if (nrows <= 0) return;   // past the end of a ragged final video block (CTA-uniform)
  } else {
    const int64_t per_head = (g.qt_rows + QT - 1) / QT;
    h = blockIdx.x / per_head;
    const int64_t t = blockIdx.x % per_head;
    row0 = g.qt_row0 + t * QT;
    nrows = min((int64_t)QT, g.qt_row0 + g.qt_rows - row0);
  }
  const int64_t count = text ? g.M : ws.kv_count[h * g.N + n];
  const int32_t* list = text ? nullptr : ws.kv_list + (h * g.N + n) * g.M;
  const T* qh = q + h * g.q_rows * d;   // q / out rows: [H][q_rows][d]
  const T* kh = k + h * g.T * d;
  const T* vh = v + h * g.T * d;

  for (int64_t e = threadIdx.x; e < QT * d; e += blockDim.x) {
    const int64_t r = e / d, c = e % d;
    qs[r * ld + c] = r < nrows ? ld_acc<T>(qh + (row0 + r) * d + c) : A(0);
  }

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  A m_run[RPW], l_run[RPW], acc[RPW][DPL];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    m_run[r] = -INFINITY;
    l_run[r] = A(0);
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[r][i] = A(0);
  }

  for (int64_t it = 0; it < count; ++it) {
    const int64_t m = text ? it : list[it];
    const int64_t kv0 = kv_row0(g, m);
    const int64_t len = kv_len(g, m);
    for (int64_t c0 = 0; c0 < len; c0 += KC) {
      const int64_t clen = min((int64_t)KC, len - c0);
      __syncthreads();
      for (int64_t e = threadIdx.x; e < KC * d; e += blockDim.x) {
        const int64_t r = e / d, c = e % d;
        const bool ok = r < clen;
        ks[r * ld + c] = ok ? ld_acc<T>(kh + (kv0 + c0 + r) * d + c) : A(0);
        vs[r * ld + c] = ok ? ld_acc<T>(vh + (kv0 + c0 + r) * d + c) : A(0);
      }
      __syncthreads();
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int row = warp * RPW + r;
        if (row >= nrows) continue;  // warp-uniform
        A s = -INFINITY;
        if (lane < clen) {
          A dot = A(0);
          const A* qr = qs + row * ld;
          const A* kr = ks + lane * ld;
          for (int64_t c = 0; c < d; ++c) dot = fma(qr[c], kr[c], dot);
          s = dot * scale;
        }
        const A cmax = warp_max_t(s);
        const A m_new = max(m_run[r], cmax);
        const A corr = ex<A>(m_run[r] - m_new);
        const A p = lane < clen ? ex<A>(s - m_new) : A(0);
        l_run[r] = l_run[r] * corr + warp_sum_t(p);
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[r][i] *= corr;
        for (int j = 0; j < clen; ++j) {
          const A pj = __shfl_sync(0xffffffffu, p, j);
#pragma unroll
          for (int i = 0; i < DPL; ++i) {
            const int64_t c = lane + 32 * i;
            if (c < d) acc[r][i] = fma(pj, vs[j * ld + c], acc[r][i]);
          }
        }
        m_run[r] = m_new;
      }
    }
  }

  // ---- epilogue: normalise, rectify (rectify.py:66-89), store ----
  double rfac = 1.0;
  const double* comp = nullptr;
  if (!text && rectify) {
    rfac = ws.r[h * g.N + n];
    comp = ws.comp + (h * g.N + n) * d;
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    const int row = warp * RPW + r;
    if (row >= nrows) continue;
    const int64_t grow = row0 + row;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int64_t c = lane + 32 * i;
      if (c < d) {
        const A o = acc[r][i] / l_run[r];
        double y = (double)o;
        if (comp) y = y * rfac + comp[c];
        out[(h * g.q_rows + grow) * d + c] = cast_out<T>(y);
      }
    }
    if (lse && lane == 0) lse[h * g.q_rows + grow] = (float)(log((double)l_run[r]) + (double)m_run[r]);
  }
}

template <typename T, int DPL>
cudaError_t launch_dpl(const Geometry& g, const void* q, const void* k, const void* v, void* out,
                       float* lse, const Workspace& ws, bool rectify, bool text, cudaStream_t st) {
  using A = typename Acc<T>::type;
  const size_t smem = (size_t)(QT + 2 * KC) * (g.d + 1) * sizeof(A);
  auto kern = attn_simt_kernel<T, DPL>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t tiles = text ? g.H * ((g.qt_rows + QT - 1) / QT) : g.H * g.N * ((g.B + QT - 1) / QT);
  if (tiles == 0) return cudaSuccess;
  const A scale = (A)(1.0 / sqrt((double)g.d));  // kernel.py:90 dtype(1/sqrt(d))
  kern<<<(unsigned)tiles, QT * WARPS, smem, st>>>((const T*)q, (const T*)k, (const T*)v, (T*)out,
                                                  lse, ws, g, rectify, text, scale);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_typed(const Geometry& g, const void* q, const void* k, const void* v, void* out,
                         float* lse, const Workspace& ws, bool rectify, bool text, cudaStream_t st) {
  const int64_t dpl = (g.d + 31) / 32;
  if (dpl <= 1) return launch_dpl<T, 1>(g, q, k, v, out, lse, ws, rectify, text, st);
  if (dpl <= 2) return launch_dpl<T, 2>(g, q, k, v, out, lse, ws, rectify, text, st);
  if (dpl <= 4) return launch_dpl<T, 4>(g, q, k, v, out, lse, ws, rectify, text, st);
  return launch_dpl<T, 8>(g, q, k, v, out, lse, ws, rectify, text, st);
}

}  // namespace

cudaError_t launch_attn_simt(const Geometry& g, const void* q, const void* k, const void* v,
                             void* out, float* lse, const Workspace& ws, bool rectify, bool text,
                             cudaStream_t st, int* launches) {
  ++*launches;
  switch (g.dtype) {
    case RSA_BF16: return launch_typed<__nv_bfloat16>(g, q, k, v, out, lse, ws, rectify, text, st);
    case RSA_F32: return launch_typed<float>(g, q, k, v, out, lse, ws, rectify, text, st);
    default: return launch_typed<double>(g, q, k, v, out, lse, ws, rectify, text, st);
  }
}

}  // namespace rsa
