// Internal declarations shared by the sm_100a kernels of librsa_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/rsa_b200.h"

namespace rsa {

// Device pointers into the caller's workspace (see rsa_workspace_layout).
struct Workspace {
  double* q_pool;
  double* q_def;
  double* k_cat;
  double* k_def;
  double* v_pool;
  double* scores;
  double* a_pool;
  uint8_t* mask_bits;
  double* r;
  float* r_eff;
  double* comp;
  int32_t* kv_count;
  int32_t* kv_list;
  int32_t* tile_count;
  int32_t* tile_list;
  __nv_bfloat16* v_t;   // [H][d][T] transposed V (tcgen05 path)
  float* text_part;     // [H][text tiles][chunks][128][d] split-K text partial O (tcgen05 path)
  float* text_ml;       // [H][text tiles][chunks][128][2] partial row max (log2) and sum
  double* a_applied;    // [H][N][M] a_pool where compensation is applied, else 0 (GEMM operand)
  int32_t* status;
};

// Problem geometry resolved on the host (rsa_plan).
struct Geometry {
  int64_t H, Tv, Tt, T, d, B;
  int64_t N, M, n_text, last_len, n_cols;
  int dtype;
  // text-query layout (text_full_attention may have any query count):
  // text query i of head h is row qt_row0 + i of a [H][q_rows][d] buffer
  int64_t qt_rows, qt_row0, q_rows;
  // token count of the last video block: B, or T_v - (N-1)B for a ragged final
  // video block (opt-in extension; the reference
  // raises BlockSizeError, core.py:71-72)
  int64_t q_last;
  // element strides of the rows of Q, K, V and O (d contiguous): head h is
  // batch entry h / hb, head h % hb of it.  Contiguous [H][T][d]: hb = H,
  // s_tok = d, s_head = T d, s_batch = H T d (rsa_shape without a layout).
  int64_t hb, s_tok, s_head, s_batch;
  // the same for the output O (a strided call may write a layout of its own)
  int64_t o_hb, o_tok, o_head, o_batch;
};

// element offset of row `row` of head h
__host__ __device__ __forceinline__ int64_t row_off(const Geometry& g, int64_t h, int64_t row) {
  return (h / g.hb) * g.s_batch + (h % g.hb) * g.s_head + row * g.s_tok;
}

// element offset of output row `row` of head h
__host__ __device__ __forceinline__ int64_t out_off(const Geometry& g, int64_t h, int64_t row) {
  return (h / g.o_hb) * g.o_batch + (h % g.o_hb) * g.o_head + row * g.o_tok;
}

// tokens in video (query) block n
__host__ __device__ __forceinline__ int64_t q_len(const Geometry& g, int64_t n) {
  return n == g.N - 1 ? g.q_last : g.B;
}
// tokens in kv block m: video blocks, then text blocks (only the last ragged)
__host__ __device__ __forceinline__ int64_t kv_len(const Geometry& g, int64_t m) {
  return m < g.N ? q_len(g, m) : (m == g.M - 1 ? g.last_len : g.B);
}
// first row of kv block m in [T] (text rows start at T_v)
__host__ __device__ __forceinline__ int64_t kv_row0(const Geometry& g, int64_t m) {
  return m < g.N ? m * g.B : g.Tv + (m - g.N) * g.B;
}

enum MaskBit : uint8_t {
  BIT_MASK = 1, BIT_IMPORTANCE = 2, BIT_COMP = 4, BIT_ADJ = 8, BIT_APPLIED = 16
};

// ST_NONFINITE: K1 saw an inf / NaN in Q, K or V (the reference's
// check_matrix ShapeError, core.py:23-31, folded into the pooling pass)
enum StatusFlag { ST_DEGENERATE = 0, ST_EMPTY_ROW = 1, ST_DEFICIT = 2, ST_NONFINITE = 3 };

constexpr int kTcTileRows = 128;   // query rows per tcgen05 tile (UMMA M)

// kv-block chunks per 128-row text query tile of the tcgen05 kernel (split-K:
// a text tile walks every kv block, ~10x a video tile's retained list)
inline int64_t text_chunks(const Geometry& g) { return g.M > 128 ? (g.M + 127) / 128 : 1; }

// ---- dtype helpers ---------------------------------------------------------
template <typename T> struct Acc { using type = float; };
template <> struct Acc<double> { using type = double; };

__device__ __forceinline__ float to_f32(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ float to_f32(float x) { return x; }
__device__ __forceinline__ double to_f64(__nv_bfloat16 x) { return (double)__bfloat162float(x); }
__device__ __forceinline__ double to_f64(float x) { return (double)x; }
__device__ __forceinline__ double to_f64(double x) { return x; }

template <typename T> __device__ __forceinline__ T from_acc(float x);
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <typename T> __device__ __forceinline__ T from_acc(double x) { return (T)x; }

// ---- launchers (one per .cu file) -----------------------------------------
// perm (device int32 [T_v], may be null): pool the video tokens in the order
// perm (row r of the permuted problem = original row perm[r]) and write the
// permuted K and V ([H][T][d], text rows copied) to kp / vp for K3, and the
// permuted video Q rows to qp (if given; its text rows are the caller's copy)
cudaError_t launch_pool(const Geometry& g, const void* q, const void* k, const void* v,
                        const Workspace& ws, cudaStream_t st, int* launches,
                        const int32_t* perm = nullptr, void* kp = nullptr, void* vp = nullptr,
                        void* qp = nullptr);
// fp64 DMMA GEMM (gemm_f64.cu): C[b] = A[b] . op(B[b]), row-major,
// op(B) = B^T (B is N x K) when b_transposed, else B (K x N)
cudaError_t launch_dgemm(int64_t batch, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         int64_t strideA, const double* B, int64_t ldb, int64_t strideB, bool b_transposed,
                         double* C, int64_t ldc, int64_t strideC, cudaStream_t st);
cudaError_t launch_select(const Geometry& g, const rsa_config& cfg, int64_t k_floor,
                          const Workspace& ws, cudaStream_t st, int* launches);
cudaError_t launch_lists_from_mask(const Geometry& g, const uint8_t* mask,
                                   const Workspace& ws, cudaStream_t st, int* launches);
cudaError_t launch_tile_lists(const Geometry& g, const Workspace& ws, cudaStream_t st,
                              int* launches);
cudaError_t launch_attn_simt(const Geometry& g, const void* q, const void* k, const void* v,
                             void* out, float* lse, const Workspace& ws, bool rectify,
                             bool text, cudaStream_t st, int* launches);
bool tc_supported(const Geometry& g);
void morton_permutation_host(int64_t t, int64_t h, int64_t w, int32_t* perm);
size_t diag_scratch_size(const Geometry& g);
size_t dense_scratch_size(const Geometry& g);
cudaError_t launch_dense_reference(const Geometry& g, const void* q, const void* k, const void* v, double* out,
                                   void* scratch, cudaStream_t st);
cudaError_t launch_diagnostics(const Geometry& g, const void* q, const void* k, const Workspace& ws,
                               double* gain, double* error, double* exact_gain, double* exact_error,
                               double* s_sum, double* s_sum_pool, void* scratch, cudaStream_t st);
cudaError_t launch_permute_rows(const Geometry& g, const int32_t* perm, const void* src, void* dst,
                                bool inverse, cudaStream_t st);
cudaError_t launch_attn_tc(const Geometry& g, const void* q, const void* k, const void* v,
                           void* out, float* lse, const Workspace& ws, bool rectify,
                           bool text, cudaStream_t st, int* launches, const int32_t* perm = nullptr,
                           const void* q_perm = nullptr, int kernel = RSA_KERNEL_AUTO);

}  // namespace rsa
