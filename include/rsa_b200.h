/*
 * rsa_b200.h -- C ABI of the B200-native Rectified SpaAttn hot path.
 *
 * One call = the reference's `rectified_attention_pipeline(problem, config,
 * variant)` (reference: pkg/src/rectattn/rectify.py:107-176) for H independent
 * single-head problems at once.  Plain pointers and sizes only: no torch types.
 *
 * Memory: every pointer is a DEVICE pointer owned by the caller.  Q, K, V and
 * O are [heads][T][d] with T = t_video + t_text; rows [0, t_video) are video
 * tokens and rows [t_video, T) text tokens (reference core.py:6-8).
 * The library never allocates device memory: callers size the workspace with
 * rsa_workspace_size() and pass it in.  All work is enqueued on `stream`; no
 * call synchronises except rsa_check_device_status().
 *
 * Errors: every entry point returns an rsa_status whose values map 1:1 onto
 * the reference's exception classes (pkg/src/rectattn/errors.py:4-45); the
 * thread-local rsa_last_error() holds the message.
 */
#ifndef RSA_B200_H
#define RSA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RSA_OK = 0,
  RSA_ERR_SHAPE = 1,            /* ShapeError          errors.py:8-9   */
  RSA_ERR_BLOCK_SIZE = 2,       /* BlockSizeError      errors.py:12-13 */
  RSA_ERR_EMPTY_ROW = 3,        /* EmptyRowError       errors.py:16-17 */
  RSA_ERR_CONFIG = 4,           /* ConfigError         errors.py:28-29 */
  RSA_ERR_DEGENERATE_ROW = 5,   /* DegenerateRowError  errors.py:24-25 */
  RSA_ERR_CUDA = 6,             /* CUDA runtime / launch failure       */
  RSA_ERR_UNSUPPORTED = 7       /* shape outside the compiled kernels  */
} rsa_status;

typedef enum { RSA_BF16 = 0, RSA_F32 = 1, RSA_F64 = 2 } rsa_dtype;

/* Reference VARIANTS, rectify.py:23-24, in the same order. */
typedef enum {
  RSA_VARIANT_FULL = 0,
  RSA_VARIANT_SPARSE_UNRECTIFIED = 1,
  RSA_VARIANT_SPARSE_RECTIFIED = 2,
  RSA_VARIANT_SPARSE_RECTIFIED_NO_GAPR = 3,
  RSA_VARIANT_COMPENSATE_ALL = 4
} rsa_variant;

/* Attention kernel selection (K3).  AUTO / TCGEN05: bf16 -> the tcgen05 kernel
 * of the shape class (d = B = 128: the paired-tile kernel; block or head_dim 64:
 * the one-tile persistent kernel), f32/f64 -> the CUDA-core kernel.
 * TCGEN05_PERSISTENT / TCGEN05_PINGPONG force the one-tile persistent or the
 * two-slot ping-pong tcgen05 kernel at d = B = 128, and SIMT the CUDA-core
 * kernel for bf16 (cross-checks; never chosen silently). */
typedef enum {
  RSA_KERNEL_AUTO = 0,
  RSA_KERNEL_TCGEN05 = 1,
  RSA_KERNEL_SIMT = 2,
  RSA_KERNEL_TCGEN05_PERSISTENT = 3,
  RSA_KERNEL_TCGEN05_PINGPONG = 4
} rsa_kernel;

/* rsa_shape.flags */
#define RSA_SHAPE_RAGGED_VIDEO 1  /* allow T_v % block != 0: the final video block holds
                                     T_v - (N-1)*block tokens (extension, SURVEY.md 8f
                                     row 4; the reference raises BlockSizeError,
                                     core.py:71-72).  Not accepted by the diagnostics. */

typedef struct {
  int64_t heads;        /* independent (batch, head) problems                */
  int64_t t_video;      /* T_v, a multiple of block (core.py:71-72) unless
                           flags has RSA_SHAPE_RAGGED_VIDEO                    */
  int64_t t_text;       /* T_t >= 0                                          */
  int64_t head_dim;     /* d                                                 */
  int64_t block;        /* B: query and key block size                       */
  int32_t dtype;        /* rsa_dtype of Q/K/V/O                              */
  int32_t kernel;       /* rsa_kernel                                        */
  int32_t flags;        /* RSA_SHAPE_* bits, 0 = the reference's rules        */
  int32_t reserved;     /* 0                                                  */
} rsa_shape;

/* SparsityConfig (masks.py:21-41) + variant (rectify.py:23-24). */
typedef struct {
  double top_k_fraction;     /* f in (0, 1]                 */
  double weight_threshold;   /* p in [0, 1]                 */
  int32_t adjacency_radius;  /* r >= 0                      */
  int32_t force_text_blocks; /* bool                        */
  int32_t variant;           /* rsa_variant                 */
  int32_t reserved;
} rsa_config;

/* Block grid (core.py:94-123 BlockGrid): N query blocks, M kv blocks. */
typedef struct {
  int64_t n_q;
  int64_t n_kv;
  int64_t n_text_blocks;
  int64_t last_text_block_len;
  int64_t n_cols;            /* N + T_t + n_text: columns of the score matrix */
  int64_t last_video_block_len;  /* block, or T_v - (N-1)*block when ragged */
} rsa_grid;

/* Byte offsets of the intermediate results inside the workspace.  Every array
 * is [heads][...] row-major.  fp64 unless noted. */
typedef struct {
  size_t q_pool;      /* [N][d]        pooled video queries   (core.py:192-201)   */
  size_t q_def;       /* [N][d]        q_sums - B*q_pool      (masks.py:165-166)   */
  size_t k_cat;       /* [n_cols][d]   k_v_pool ; raw text keys ; pooled text keys  */
  size_t k_def;       /* [M][d]        k_sums - len*k_pool    (masks.py:170-171)   */
  size_t v_pool;      /* [M][d]        pooled values          (core.py:198)        */
  size_t scores;      /* [N][n_cols]   q_pool.k_cat / sqrt(d) (ipar.py:41, masks.py:127) */
  size_t a_pool;      /* [N][M]        implicit full attention (ipar.py:69-86)     */
  size_t mask_bits;   /* u8 [N][M]: bit0 mask, bit1 importance, bit2 gain>error,
                         bit3 adjacency, bit4 applied compensation                 */
  size_t r;           /* [N]           rectification factors  (rectify.py:56-63) */
  size_t r_eff;       /* f32 [N]       factor the epilogue applies (1 if unrectified) */
  size_t comp;        /* [N][d]        sum_applied a_pool v_pool (rectify.py:84-87) */
  size_t kv_count;    /* i32 [N]       retained kv blocks per query block           */
  size_t kv_list;     /* i32 [N][M]    ascending retained kv block ids               */
  size_t tile_count;  /* i32 [tiles]   kv entries per 128-row tcgen05 tile (B = 64;
                         at B = 128 a tile is one query block: kv_count / kv_list) */
  size_t tile_list;   /* i32 [tiles][M] (kv id | member bits << 24)                  */
  size_t v_t;         /* bf16 [d][T]   V transposed (tcgen05 path: K-major PV operand) */
  size_t text_part;   /* f32 [text tiles][chunks][128][d] split-K partial O of text queries */
  size_t text_ml;     /* f32 [text tiles][chunks][128][2] partial row max (log2) and row sum */
  size_t a_applied;   /* [N][M]        a_pool where compensation is applied, else 0        */
  size_t status;      /* i32 [4]       device status flags (degenerate row, ...)     */
  size_t total;
} rsa_workspace_layout;

/* Validation + block grid; RSA_ERR_* mirrors AttentionProblem.__post_init__
 * (core.py:59-80) and SparsityConfig.__post_init__ (masks.py:35-41). */
rsa_status rsa_plan(const rsa_shape* shape, const rsa_config* cfg, rsa_grid* grid);
rsa_status rsa_workspace_layout_query(const rsa_shape* shape, rsa_workspace_layout* layout);
size_t rsa_workspace_size(const rsa_shape* shape);

/* K1: exactly rounded fp64 block pooling of Q_video, K (video / text blocks
 * isolated) and V.  Replaces pool_problem + block_sums (core.py:154-201,
 * masks.py:130-135, masks.py:165-171). */
rsa_status rsa_pool(const rsa_shape* shape, const void* q, const void* k, const void* v,
                    void* workspace, void* stream);

/* K2: fp64 pooled scoring, IPAR reallocation, deterministic top-k/threshold
 * selection, gain/error gate, rectification factors and compensation rows.
 * Replaces implicit_full_attention (ipar.py:69-86), build_sparse_mask
 * (masks.py:83-117), gain_error/compensation_mask (masks.py:120-219) and
 * rectification_factors (rectify.py:56-63).  Needs rsa_pool first. */
rsa_status rsa_select(const rsa_shape* shape, const rsa_config* cfg, void* workspace,
                      void* stream);

/* K3+K4: block-sparse flash attention over the retained kv blocks with the
 * IPAR rescale and GAPR compensation fused into the epilogue, plus full
 * attention for the text queries.  Replaces block_sparse_attention
 * (kernel.py:65-117), text_full_attention (kernel.py:120-145) and
 * apply_rectification (rectify.py:66-89).  `lse` (f32 [heads][T], natural
 * log, may be NULL) is the reference's row_log_denominators. Needs rsa_select. */
rsa_status rsa_attention(const rsa_shape* shape, const rsa_config* cfg, const void* q,
                         const void* k, const void* v, void* out, float* lse,
                         void* workspace, void* stream);

/* K1 -> K2 -> K3+K4: the whole pipeline (rectify.py:107-176). */
rsa_status rsa_forward(const rsa_shape* shape, const rsa_config* cfg, const void* q,
                       const void* k, const void* v, void* out, float* lse,
                       void* workspace, void* stream);

/* Element strides of Q, K, V and O for rsa_forward_strided (head_dim is
 * contiguous): head h of the call is head (h % heads_per_batch) of batch entry
 * (h / heads_per_batch), and its token row t starts at element
 *   (h / heads_per_batch) * batch_stride + (h % heads_per_batch) * head_stride
 *   + t * token_stride.
 * Contiguous [B, H, T, d]: {H, d, T d, H T d}.  A model's [B, T, H, d]
 * projection output, without a transpose: {H, H d, d, T H d}. */
typedef struct {
  int64_t heads_per_batch;
  int64_t token_stride;
  int64_t head_stride;
  int64_t batch_stride;
} rsa_layout;

/* rsa_forward on strided views: `layout` for Q, K and V, `out_layout` for O
 * (NULL: the same as `layout`); `lse` and the workspace keep their [heads][T] /
 * rsa_workspace_layout shapes.  bf16 with
 * the tcgen05 kernels (block and head_dim in {64, 128}); strides multiples of
 * 8 elements and 16-byte aligned pointers, else RSA_ERR_UNSUPPORTED.  K1 and
 * K3 read the rows through 4-D TMA maps and K3 stores through the same
 * strides: no transpose or contiguous copy is made.  The reference's arrays
 * are 2-D [T, d] (core.py:51-57); this is the batched model-facing form of
 * the same call. */
rsa_status rsa_forward_strided(const rsa_shape* shape, const rsa_config* cfg, const rsa_layout* layout,
                               const rsa_layout* out_layout, const void* q, const void* k, const void* v,
                               void* out, float* lse, void* workspace, void* stream);

/* rsa_forward from HOST memory (end-to-end call): host_q/k/v/out are host
 * pointers (page-locked for the copies to overlap), dq/dk/dv/dout device
 * buffers of the same [heads][T][d] size.  Heads are processed in chunks of
 * `heads_per_chunk`: chunk c+1's host->device copy and chunk c-1's
 * device->host copy run on two internal streams while chunk c computes on
 * `stream`.  Work is enqueued on `stream`; the output is in host memory once
 * `stream` reaches the end of the call. */
rsa_status rsa_forward_host(const rsa_shape* shape, const rsa_config* cfg, const void* host_q,
                            const void* host_k, const void* host_v, void* host_out, void* dq,
                            void* dk, void* dv, void* dout, float* lse, void* workspace,
                            int64_t heads_per_chunk, void* stream);

/* Kernel-only seam (kernel.py:65-117): video queries over an explicit block
 * mask (u8 [heads][N][M], nonzero = retained); no rectification.  Text rows
 * of `out` are left untouched. */
rsa_status rsa_block_sparse_attention(const rsa_shape* shape, const void* q, const void* k,
                                      const void* v, const uint8_t* block_mask, void* out,
                                      float* lse, void* workspace, void* stream);

/* Kernel-only seam (kernel.py:120-145): `n_queries` text queries attend over
 * all `n_keys` keys, tiled by `block` (last tile ragged).  q/out are
 * [heads][n_queries][d], k/v [heads][n_keys][d]; `workspace` is unused. */
rsa_status rsa_text_full_attention(int64_t heads, int64_t n_queries, int64_t n_keys,
                                   int64_t head_dim, int64_t block, int32_t dtype, const void* q,
                                   const void* k, const void* v, void* out, float* lse,
                                   void* workspace, void* stream);

/* Morton (Z-order) token permutation of a (t, h, w) grid, w fastest
 * (core.py:263-291 morton_code_3d / morton_permutation): perm[i] = original
 * video row placed at position i (numpy's stable argsort of the codes).
 * `perm` is HOST memory of t*h*w entries; no device work. */
rsa_status rsa_morton_permutation(int64_t t, int64_t h, int64_t w, int32_t* perm);

/* Row permutation of one [heads][T][d] tensor of `shape`'s dtype (the data
 * movement of reorder_morton, core.py:294-318): video rows dst[r] =
 * src[perm[r]], or dst[perm[r]] = src[r] with `inverse` (undo); text rows are
 * copied.  `perm` is a DEVICE int32 array of t_video entries. */
rsa_status rsa_permute_rows(const rsa_shape* shape, const int32_t* perm, const void* src, void* dst,
                            int32_t inverse, void* stream);

/* Bytes of the `perm_buf` rsa_forward_permuted needs (permuted Q, K and V). */
size_t rsa_permuted_buffer_size(const rsa_shape* shape);

/* rsa_forward on the problem whose video tokens are reordered by `perm`
 * (DEVICE int32 [t_video]) -- the reference harness's morton_reorder option,
 * reorder_morton + rectified_attention_pipeline (harness.py:172-173) -- with
 * Q/K/V and O/LSE in the ORIGINAL token order: K1 gathers the rows and writes
 * the permuted K/V into `perm_buf`, K3 gathers the query rows and scatters the
 * output rows; the workspace results (masks, a_pool, ...) are those of the
 * reordered problem.  bf16 with the tcgen05 kernel only (RSA_ERR_UNSUPPORTED
 * otherwise: use rsa_permute_rows + rsa_forward). */
rsa_status rsa_forward_permuted(const rsa_shape* shape, const rsa_config* cfg, const void* q,
                                const void* k, const void* v, const int32_t* perm, void* perm_buf,
                                void* out, float* lse, void* workspace, void* stream);

/* Validation diagnostics (quadratic; fp64 like the reference), after
 * rsa_pool + rsa_select on `workspace`.  Outputs (device, fp64):
 *   gain, error, exact_gain, exact_error  [heads][N][M]  -- gain_error(...,
 *       with_exact=True), masks.py:189-219 (the relaxed pair is what K2 gates on)
 *   s_sum, s_sum_pool                      [heads][t_video] -- the true and
 *       pooled softmax denominators of denominator_equivalence_report,
 *       metrics.py:90-113
 * gapr_condition_agreement (metrics.py:116-124) and the satisfied fraction
 * follow from them.  `scratch`: rsa_diagnostics_scratch_size() bytes. */
size_t rsa_diagnostics_scratch_size(const rsa_shape* shape);
rsa_status rsa_diagnostics(const rsa_shape* shape, const void* q, const void* k, void* workspace,
                           double* gain, double* error, double* exact_gain, double* exact_error,
                           double* s_sum, double* s_sum_pool, void* scratch, void* stream);

/* The reference's ground truth, full_attention_oracle (core.py:211-225):
 * dense fp64 softmax(Q K^T / sqrt d) V for every query row (video and text)
 * of every head; `out` is fp64 [heads][T][d] (device).  Used by the harness
 * core (run_variants) to score the variants as the reference does. */
size_t rsa_dense_reference_scratch_size(const rsa_shape* shape);
rsa_status rsa_dense_reference(const rsa_shape* shape, const void* q, const void* k, const void* v,
                               double* out, void* scratch, void* stream);

/* Synchronises `stream` and converts device-side status flags (e.g. a
 * reallocation denominator <= 0, ipar.py:62-64) into an rsa_status. */
rsa_status rsa_check_device_status(void* workspace, void* stream);

/* Stream-ordered, non-synchronising status: ORs the call's device status
 * flags (int32[4]: degenerate row, empty row, deficit, non-finite input)
 * into the caller's device buffer `status_accum`, which the caller zeroes
 * once and may read back whenever it synchronises anyway (a model loop).
 * rsa_status_from_flags() turns a host copy of those flags into the status
 * rsa_check_device_status() would have returned. */
rsa_status rsa_accumulate_status(const void* workspace, int32_t* status_accum, void* stream);
rsa_status rsa_status_from_flags(const int32_t* host_flags);

/* Number of kernel launches the last rsa_forward/rsa_attention enqueued. */
int32_t rsa_last_launch_count(void);
const char* rsa_last_error(void);
const char* rsa_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RSA_B200_H */
