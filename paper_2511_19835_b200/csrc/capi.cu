// extern "C" entry points of librsa_b200.so (include/rsa_b200.h).
//
// Host-side validation mirrors the reference's eager checks:
//   AttentionProblem.__post_init__  core.py:59-80   (ShapeError, BlockSizeError)
//   partition                       core.py:140-151 (N, M, ragged last text block)
//   SparsityConfig.__post_init__    masks.py:35-41  (ConfigError)
//   rectified_attention_pipeline    rectify.py:118-119 (unknown variant -> ConfigError)
// and orchestrates K1 -> K2 -> K3 on the caller's stream with the caller's
// workspace (no allocation, no synchronisation).
#include "rsa_internal.cuh"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

namespace {

thread_local std::string g_last_error;
thread_local int g_launches = 0;

rsa_status fail(rsa_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

rsa_status cuda_fail(cudaError_t e, const char* where) {
  return fail(RSA_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

rsa_status make_geometry(const rsa_shape* s, rsa::Geometry* g) {
  if (!s) return fail(RSA_ERR_SHAPE, "null shape");
  if (s->dtype < RSA_BF16 || s->dtype > RSA_F64)
    return fail(RSA_ERR_SHAPE, "q/k/v must be bfloat16, float32 or float64");
  if (s->heads < 1) return fail(RSA_ERR_SHAPE, "heads must be >= 1");
  if (s->head_dim < 1) return fail(RSA_ERR_SHAPE, "head_dim must be >= 1");
  if (s->t_video < 0 || s->t_text < 0) return fail(RSA_ERR_SHAPE, "token counts must be >= 0");
  if (s->block <= 0)
    return fail(RSA_ERR_BLOCK_SIZE, "block size must be positive, got " + std::to_string(s->block));
  if (s->t_video % s->block != 0 && !(s->flags & RSA_SHAPE_RAGGED_VIDEO))
    return fail(RSA_ERR_BLOCK_SIZE, "T_v=" + std::to_string(s->t_video) +
                                        " is not divisible by block size " + std::to_string(s->block));
  if (s->t_video == 0) return fail(RSA_ERR_SHAPE, "T_v must be >= 1 block");
  g->H = s->heads;
  g->Tv = s->t_video;
  g->Tt = s->t_text;
  g->T = s->t_video + s->t_text;
  g->d = s->head_dim;
  g->B = s->block;
  g->N = (s->t_video + s->block - 1) / s->block;
  g->q_last = s->t_video - (g->N - 1) * s->block;   // == B unless the final video block is ragged
  g->n_text = (s->t_text + s->block - 1) / s->block;
  g->M = g->N + g->n_text;
  g->last_len = g->n_text ? s->t_text - (g->n_text - 1) * s->block : 0;
  g->n_cols = g->N + g->Tt + g->n_text;
  g->dtype = s->dtype;
  g->qt_rows = g->Tt;
  g->qt_row0 = g->Tv;
  g->q_rows = g->T;
  g->hb = g->H;   // contiguous [H][T][d] (rsa_shape_set_layout may override)
  g->s_tok = g->d;
  g->s_head = g->T * g->d;
  g->s_batch = g->H * g->T * g->d;
  g->o_hb = g->hb; g->o_tok = g->s_tok; g->o_head = g->s_head; g->o_batch = g->s_batch;
  const int64_t dmax = s->dtype == RSA_F64 ? 128 : 256;
  if (g->d > dmax)
    return fail(RSA_ERR_UNSUPPORTED, "head_dim " + std::to_string(g->d) + " > " + std::to_string(dmax));
  if (g->M > 8192) return fail(RSA_ERR_UNSUPPORTED, "more than 8192 kv blocks");
  return RSA_OK;
}

bool contiguous(const rsa::Geometry& g) {
  return g.hb == g.H && g.s_tok == g.d && g.s_head == g.T * g.d && g.s_batch == g.H * g.T * g.d &&
         g.o_hb == g.H && g.o_tok == g.d && g.o_head == g.T * g.d && g.o_batch == g.H * g.T * g.d;
}

// A strided call's element strides (rsa_layout) replace the contiguous
// [H][T][d] default.  The strided path is the model-facing one: bf16 on the
// tcgen05 kernels, whose TMA maps need 16-byte row / head / batch strides.
rsa_status check_layout(const rsa_layout* l, const rsa::Geometry& g) {
  if (l->heads_per_batch < 1 || g.H % l->heads_per_batch != 0)
    return fail(RSA_ERR_SHAPE, "heads must be a multiple of layout.heads_per_batch");
  if (l->token_stride < g.d || l->head_stride < 0 || l->batch_stride < 0)
    return fail(RSA_ERR_SHAPE, "layout strides must be non-negative and token_stride >= head_dim");
  if (l->token_stride % 8 || l->head_stride % 8 || l->batch_stride % 8)
    return fail(RSA_ERR_UNSUPPORTED, "layout strides must be multiples of 8 elements (16-byte TMA rows)");
  // (an expanded / broadcast dimension -- stride 0 -- is not a TMA-mappable view)
  if ((l->heads_per_batch > 1 && l->head_stride == 0) || (g.H / l->heads_per_batch > 1 && l->batch_stride == 0))
    return fail(RSA_ERR_UNSUPPORTED, "layout strides of dimensions longer than 1 must be non-zero");
  return RSA_OK;
}

// A strided call's element strides (rsa_layout) replace the contiguous
// [H][T][d] default.  The strided path is the model-facing one: bf16 on the
// tcgen05 kernels, whose TMA maps need 16-byte row / head / batch strides.
rsa_status apply_layout(const rsa_layout* l, const rsa_layout* lo, const void* const* ptrs, int n_ptrs,
                        rsa::Geometry* g) {
  if (!l) return fail(RSA_ERR_SHAPE, "null layout");
  if (!lo) lo = l;
  if (g->dtype != RSA_BF16) return fail(RSA_ERR_UNSUPPORTED, "strided q/k/v/out are supported for bfloat16 only");
  rsa_status s = check_layout(l, *g);
  if (s != RSA_OK) return s;
  s = check_layout(lo, *g);
  if (s != RSA_OK) return s;
  for (int i = 0; i < n_ptrs; ++i)
    if (reinterpret_cast<uintptr_t>(ptrs[i]) % 16)
      return fail(RSA_ERR_UNSUPPORTED, "strided q/k/v/out must be 16-byte aligned");
  g->hb = l->heads_per_batch;
  g->s_tok = l->token_stride;
  g->s_head = l->head_stride;
  g->s_batch = l->batch_stride;
  g->o_hb = lo->heads_per_batch;
  g->o_tok = lo->token_stride;
  g->o_head = lo->head_stride;
  g->o_batch = lo->batch_stride;
  return RSA_OK;
}

rsa_status check_config(const rsa_config* c) {
  if (!c) return fail(RSA_ERR_CONFIG, "null config");
  if (!(c->top_k_fraction > 0.0 && c->top_k_fraction <= 1.0))
    return fail(RSA_ERR_CONFIG, "top_k_fraction must be in (0, 1], got " + std::to_string(c->top_k_fraction));
  if (!(c->weight_threshold >= 0.0 && c->weight_threshold <= 1.0))
    return fail(RSA_ERR_CONFIG, "weight_threshold must be in [0, 1], got " + std::to_string(c->weight_threshold));
  if (c->adjacency_radius < 0)
    return fail(RSA_ERR_CONFIG, "adjacency_radius must be >= 0, got " + std::to_string(c->adjacency_radius));
  if (c->variant < RSA_VARIANT_FULL || c->variant > RSA_VARIANT_COMPENSATE_ALL)
    return fail(RSA_ERR_CONFIG, "unknown variant " + std::to_string(c->variant));
  return RSA_OK;
}

int64_t tiles_per_head(const rsa::Geometry& g) {
  const int64_t G = (g.B <= rsa::kTcTileRows && rsa::kTcTileRows % g.B == 0) ? rsa::kTcTileRows / g.B : 1;
  return (g.N + G - 1) / G;
}

void layout_of(const rsa::Geometry& g, rsa_workspace_layout* L) {
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = align_up(off + bytes); return o; };
  const size_t H = g.H, N = g.N, M = g.M, d = g.d, C = g.n_cols, TT = tiles_per_head(g);
  L->status = take(64);
  L->q_pool = take(H * N * d * 8);
  L->q_def = take(H * N * d * 8);
  L->k_cat = take(H * C * d * 8);
  L->k_def = take(H * M * d * 8);
  L->v_pool = take(H * M * d * 8);
  L->scores = take(H * N * C * 8);
  L->a_pool = take(H * N * M * 8);
  L->mask_bits = take(H * N * M);
  L->r = take(H * N * 8);
  L->r_eff = take(H * N * 4);
  L->comp = take(H * N * d * 8);
  L->kv_count = take(H * N * 4);
  L->kv_list = take(H * N * M * 4);
  L->tile_count = take(H * TT * 4);
  L->tile_list = take(H * TT * M * 4);
  L->v_t = take(0);   // (unused since round 2; kept for the layout ABI)
  const size_t text_parts = g.dtype == RSA_BF16 ? H * (size_t)((g.Tt + 127) / 128) * rsa::text_chunks(g) * 128 : 0;
  L->text_part = take(text_parts * d * 4);
  L->text_ml = take(text_parts * 8);
  L->a_applied = take(H * N * M * 8);
  L->total = off;
}

rsa::Workspace bind(const rsa::Geometry& g, void* base) {
  rsa_workspace_layout L;
  layout_of(g, &L);
  char* b = static_cast<char*>(base);
  rsa::Workspace w;
  w.status = reinterpret_cast<int32_t*>(b + L.status);
  w.q_pool = reinterpret_cast<double*>(b + L.q_pool);
  w.q_def = reinterpret_cast<double*>(b + L.q_def);
  w.k_cat = reinterpret_cast<double*>(b + L.k_cat);
  w.k_def = reinterpret_cast<double*>(b + L.k_def);
  w.v_pool = reinterpret_cast<double*>(b + L.v_pool);
  w.scores = reinterpret_cast<double*>(b + L.scores);
  w.a_pool = reinterpret_cast<double*>(b + L.a_pool);
  w.mask_bits = reinterpret_cast<uint8_t*>(b + L.mask_bits);
  w.r = reinterpret_cast<double*>(b + L.r);
  w.r_eff = reinterpret_cast<float*>(b + L.r_eff);
  w.comp = reinterpret_cast<double*>(b + L.comp);
  w.kv_count = reinterpret_cast<int32_t*>(b + L.kv_count);
  w.kv_list = reinterpret_cast<int32_t*>(b + L.kv_list);
  w.tile_count = reinterpret_cast<int32_t*>(b + L.tile_count);
  w.tile_list = reinterpret_cast<int32_t*>(b + L.tile_list);
  w.v_t = reinterpret_cast<__nv_bfloat16*>(b + L.v_t);
  w.text_part = reinterpret_cast<float*>(b + L.text_part);
  w.text_ml = reinterpret_cast<float*>(b + L.text_ml);
  w.a_applied = reinterpret_cast<double*>(b + L.a_applied);
  return w;
}

bool use_tc(const rsa_shape* s, const rsa::Geometry& g) {
  if (s->kernel == RSA_KERNEL_SIMT) return false;
  return rsa::tc_supported(g);
}

rsa_status run_attention(const rsa_shape* s, const rsa::Geometry& g, const rsa::Workspace& ws,
                         const void* q, const void* k, const void* v, void* out, float* lse,
                         bool rectify, bool text, cudaStream_t st, const int32_t* perm = nullptr,
                         const void* q_perm = nullptr) {
  cudaError_t e;
  const bool tc = use_tc(s, g);
  // bf16 runs on the tensor-core kernel; the CUDA-core kernel serves the
  // reference's fp32/fp64 precisions, and bf16 only when asked for by name
  // (a cross-check) -- never as a silent second backend
  if ((s->kernel == RSA_KERNEL_TCGEN05 || s->kernel == RSA_KERNEL_TCGEN05_PERSISTENT ||
       s->kernel == RSA_KERNEL_TCGEN05_PINGPONG || (s->kernel == RSA_KERNEL_AUTO && g.dtype == RSA_BF16)) && !tc)
    return fail(RSA_ERR_UNSUPPORTED, "bf16 attention runs on the tcgen05 kernel, which needs block and "
                                     "head_dim in {64, 128} (kernel='simt' selects the CUDA-core kernel "
                                     "explicitly)");
  if (tc) {
    e = rsa::launch_tile_lists(g, ws, st, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "tile_lists");
    e = rsa::launch_attn_tc(g, q, k, v, out, lse, ws, rectify, text, st, &g_launches, perm, q_perm, s->kernel);
    if (e != cudaSuccess) return cuda_fail(e, "attn_tc");
  } else {
    if (perm) return fail(RSA_ERR_UNSUPPORTED, "the permuted problem needs the tcgen05 kernel (bf16)");
    if (!contiguous(g)) return fail(RSA_ERR_UNSUPPORTED, "strided q/k/v/out need the tcgen05 kernel");
    e = rsa::launch_attn_simt(g, q, k, v, out, lse, ws, rectify, false, st, &g_launches);
    if (e != cudaSuccess) return cuda_fail(e, "attn_simt(video)");
    if (text && g.Tt > 0) {
      e = rsa::launch_attn_simt(g, q, k, v, out, lse, ws, false, true, st, &g_launches);
      if (e != cudaSuccess) return cuda_fail(e, "attn_simt(text)");
    }
  }
  return RSA_OK;
}

__global__ void accumulate_status_kernel(const int32_t* __restrict__ flags, int32_t* __restrict__ accum) {
  if (threadIdx.x < 4 && flags[threadIdx.x]) atomicOr(accum + threadIdx.x, flags[threadIdx.x]);
}

bool rectifies(int variant) {
  return variant == RSA_VARIANT_SPARSE_RECTIFIED || variant == RSA_VARIANT_SPARSE_RECTIFIED_NO_GAPR ||
         variant == RSA_VARIANT_COMPENSATE_ALL;
}

}  // namespace

extern "C" {

rsa_status rsa_plan(const rsa_shape* shape, const rsa_config* cfg, rsa_grid* grid) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  if (cfg) {
    s = check_config(cfg);
    if (s != RSA_OK) return s;
  }
  if (grid) {
    grid->n_q = g.N;
    grid->n_kv = g.M;
    grid->n_text_blocks = g.n_text;
    grid->last_text_block_len = g.last_len;
    grid->n_cols = g.n_cols;
    grid->last_video_block_len = g.q_last;
  }
  return RSA_OK;
}

rsa_status rsa_workspace_layout_query(const rsa_shape* shape, rsa_workspace_layout* layout) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  layout_of(g, layout);
  return RSA_OK;
}

size_t rsa_workspace_size(const rsa_shape* shape) {
  rsa_workspace_layout L;
  if (rsa_workspace_layout_query(shape, &L) != RSA_OK) return 0;
  return L.total;
}

}  // extern "C"

namespace {
// K1; `reset_status` clears the device status flags first (a new call).  The
// host-memory call keeps them across its head chunks, so an error raised by
// any chunk survives to the final check.
rsa_status pool_geom(const rsa::Geometry& g, const void* q, const void* k, const void* v, void* workspace,
                     void* stream, bool reset_status) {
  if (!q || !k || !v || !workspace) return fail(RSA_ERR_SHAPE, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rsa::Workspace ws = bind(g, workspace);
  cudaError_t e = reset_status ? cudaMemsetAsync(ws.status, 0, 64, st) : cudaSuccess;
  if (e != cudaSuccess) return cuda_fail(e, "memset status");
  e = rsa::launch_pool(g, q, k, v, ws, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "pool");
  return RSA_OK;
}

rsa_status pool_impl(const rsa_shape* shape, const void* q, const void* k, const void* v, void* workspace,
                     void* stream, bool reset_status) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  return pool_geom(g, q, k, v, workspace, stream, reset_status);
}

rsa_status select_geom(const rsa::Geometry& g, const rsa_config* cfg, void* workspace, void* stream) {
  rsa_status s = check_config(cfg);
  if (s != RSA_OK) return s;
  if (!workspace) return fail(RSA_ERR_SHAPE, "null workspace");
  // k_floor = math.ceil(top_k_fraction * M) (masks.py:100), IEEE double on the host
  const int64_t k_floor = (int64_t)std::ceil(cfg->top_k_fraction * (double)g.M);
  rsa::Workspace ws = bind(g, workspace);
  cudaError_t e = rsa::launch_select(g, *cfg, k_floor, ws, static_cast<cudaStream_t>(stream), &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "select");
  return RSA_OK;
}

rsa_status attention_geom(const rsa_shape* shape, const rsa::Geometry& g, const rsa_config* cfg, const void* q,
                          const void* k, const void* v, void* out, float* lse, void* workspace, void* stream) {
  rsa_status s = check_config(cfg);
  if (s != RSA_OK) return s;
  if (!q || !k || !v || !out || !workspace) return fail(RSA_ERR_SHAPE, "null pointer");
  rsa::Workspace ws = bind(g, workspace);
  return run_attention(shape, g, ws, q, k, v, out, lse, rectifies(cfg->variant), true,
                       static_cast<cudaStream_t>(stream));
}

rsa_status forward_impl(const rsa_shape* shape, const rsa_config* cfg, const void* q, const void* k,
                        const void* v, void* out, float* lse, void* workspace, void* stream, bool reset_status);
rsa_status forward_geom(const rsa_shape* shape, const rsa::Geometry& g, const rsa_config* cfg, const void* q,
                        const void* k, const void* v, void* out, float* lse, void* workspace, void* stream,
                        bool reset_status);
}  // namespace

extern "C" {

rsa_status rsa_pool(const rsa_shape* shape, const void* q, const void* k, const void* v,
                    void* workspace, void* stream) {
  return pool_impl(shape, q, k, v, workspace, stream, true);
}

rsa_status rsa_select(const rsa_shape* shape, const rsa_config* cfg, void* workspace, void* stream) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  return select_geom(g, cfg, workspace, stream);
}

rsa_status rsa_attention(const rsa_shape* shape, const rsa_config* cfg, const void* q,
                         const void* k, const void* v, void* out, float* lse, void* workspace,
                         void* stream) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  return attention_geom(shape, g, cfg, q, k, v, out, lse, workspace, stream);
}

rsa_status rsa_forward(const rsa_shape* shape, const rsa_config* cfg, const void* q, const void* k,
                       const void* v, void* out, float* lse, void* workspace, void* stream) {
  g_launches = 0;
  return forward_impl(shape, cfg, q, k, v, out, lse, workspace, stream, true);
}

rsa_status rsa_forward_strided(const rsa_shape* shape, const rsa_config* cfg, const rsa_layout* layout,
                               const rsa_layout* out_layout, const void* q, const void* k, const void* v,
                               void* out, float* lse, void* workspace, void* stream) {
  g_launches = 0;
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  const void* ptrs[4] = {q, k, v, out};
  s = apply_layout(layout, out_layout, ptrs, 4, &g);
  if (s != RSA_OK) return s;
  if (!rsa::tc_supported(g) || shape->kernel == RSA_KERNEL_SIMT)
    return fail(RSA_ERR_UNSUPPORTED, "strided q/k/v/out need the tcgen05 kernel (bf16, block and head_dim "
                                     "in {64, 128})");
  return forward_geom(shape, g, cfg, q, k, v, out, lse, workspace, stream, true);
}

}  // extern "C"

namespace {
rsa_status forward_geom(const rsa_shape* shape, const rsa::Geometry& g, const rsa_config* cfg, const void* q,
                        const void* k, const void* v, void* out, float* lse, void* workspace, void* stream,
                        bool reset_status) {
  rsa_status s = check_config(cfg);
  if (s != RSA_OK) return s;
  s = pool_geom(g, q, k, v, workspace, stream, reset_status);
  if (s != RSA_OK) return s;
  s = select_geom(g, cfg, workspace, stream);
  if (s != RSA_OK) return s;
  return attention_geom(shape, g, cfg, q, k, v, out, lse, workspace, stream);
}

rsa_status forward_impl(const rsa_shape* shape, const rsa_config* cfg, const void* q, const void* k,
                        const void* v, void* out, float* lse, void* workspace, void* stream, bool reset_status) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  return forward_geom(shape, g, cfg, q, k, v, out, lse, workspace, stream, reset_status);
}

// per-thread pool of timing-free events for the host-memory call (no
// create/destroy per call)
cudaError_t host_events(size_t n, std::vector<cudaEvent_t>** out) {
  static thread_local std::vector<cudaEvent_t> pool;
  static thread_local int pool_dev = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (pool_dev != dev) {   // events belong to a device: start a fresh pool (old ones are leaked, not reused)
    pool.clear();
    pool_dev = dev;
  }
  while (pool.size() < n) {
    cudaEvent_t x;
    if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) return e;
    pool.push_back(x);
  }
  *out = &pool;
  return cudaSuccess;
}
}  // namespace

extern "C" {

// End-to-end call from host memory: heads are processed in chunks so chunk
// c+1's host->device copy (copy-in stream) overlaps chunk c's K1->K2->K3
// (caller's stream) and chunk c-1's device->host copy (copy-out stream).
rsa_status rsa_forward_host(const rsa_shape* shape, const rsa_config* cfg, const void* host_q,
                            const void* host_k, const void* host_v, void* host_out, void* dq, void* dk,
                            void* dv, void* dout, float* lse, void* workspace, int64_t heads_per_chunk,
                            void* stream) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  s = check_config(cfg);
  if (s != RSA_OK) return s;
  if (!host_q || !host_k || !host_v || !host_out || !dq || !dk || !dv || !dout || !workspace)
    return fail(RSA_ERR_SHAPE, "null pointer");
  if (heads_per_chunk < 1 || heads_per_chunk > g.H) heads_per_chunk = g.H;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  static thread_local cudaStream_t s_in = nullptr, s_out = nullptr;
  static thread_local int dev_of_streams = -1;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  if (dev_of_streams != dev) {
    if ((e = cudaStreamCreateWithFlags(&s_in, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&s_out, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_fail(e, "stream create");
    dev_of_streams = dev;
  }
  const size_t esz = g.dtype == RSA_BF16 ? 2 : g.dtype == RSA_F32 ? 4 : 8;
  const size_t head_bytes = (size_t)g.T * g.d * esz;
  const int64_t n_chunks = (g.H + heads_per_chunk - 1) / heads_per_chunk;
  std::vector<cudaEvent_t>* evp = nullptr;
  if ((e = host_events((size_t)(3 * n_chunks + 1), &evp)) != cudaSuccess) return cuda_fail(e, "event");
  std::vector<cudaEvent_t>& ev = *evp;
  // the copy-in stream starts after whatever the caller queued on `stream`
  cudaEventRecord(ev[3 * n_chunks], st);
  cudaStreamWaitEvent(s_in, ev[3 * n_chunks], 0);
  int launches = 0;
  for (int64_t c = 0; c < n_chunks && s == RSA_OK; ++c) {
    const int64_t h0 = c * heads_per_chunk, hc = std::min(heads_per_chunk, g.H - h0);
    const size_t off = (size_t)h0 * head_bytes, bytes = (size_t)hc * head_bytes;
    auto H = [&](const void* p) { return static_cast<const char*>(p) + off; };
    auto D = [&](void* p) { return static_cast<char*>(p) + off; };
    if ((e = cudaMemcpyAsync(D(dq), H(host_q), bytes, cudaMemcpyHostToDevice, s_in)) != cudaSuccess ||
        (e = cudaMemcpyAsync(D(dk), H(host_k), bytes, cudaMemcpyHostToDevice, s_in)) != cudaSuccess ||
        (e = cudaMemcpyAsync(D(dv), H(host_v), bytes, cudaMemcpyHostToDevice, s_in)) != cudaSuccess)
      return cuda_fail(e, "H2D");
    cudaEventRecord(ev[3 * c], s_in);
    cudaStreamWaitEvent(st, ev[3 * c], 0);
    rsa_shape sub = *shape;
    sub.heads = hc;
    // the status flags are cleared by the first chunk only: a non-finite input,
    // degenerate or empty row in any chunk survives to rsa_check_device_status
    g_launches = 0;
    s = forward_impl(&sub, cfg, D(dq), D(dk), D(dv), D(dout), lse ? lse + h0 * g.T : nullptr, workspace, stream,
                     c == 0);
    launches += g_launches;
    cudaEventRecord(ev[3 * c + 1], st);
    cudaStreamWaitEvent(s_out, ev[3 * c + 1], 0);
    if ((e = cudaMemcpyAsync(static_cast<char*>(host_out) + off, D(dout), bytes, cudaMemcpyDeviceToHost,
                             s_out)) != cudaSuccess)
      return cuda_fail(e, "D2H");
    cudaEventRecord(ev[3 * c + 2], s_out);
  }
  // the caller's stream resumes once every output chunk is in host memory
  for (int64_t c = 0; c < n_chunks; ++c) cudaStreamWaitEvent(st, ev[3 * c + 2], 0);
  g_launches = launches;
  if (s != RSA_OK) return s;
  e = cudaGetLastError();
  return e == cudaSuccess ? RSA_OK : cuda_fail(e, "forward_host");
}

rsa_status rsa_block_sparse_attention(const rsa_shape* shape, const void* q, const void* k,
                                      const void* v, const uint8_t* block_mask, void* out,
                                      float* lse, void* workspace, void* stream) {
  g_launches = 0;
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  if (!q || !k || !v || !block_mask || !out || !workspace) return fail(RSA_ERR_SHAPE, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rsa::Workspace ws = bind(g, workspace);
  cudaError_t e = cudaMemsetAsync(ws.status, 0, 64, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset status");
  e = rsa::launch_lists_from_mask(g, block_mask, ws, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "lists_from_mask");
  return run_attention(shape, g, ws, q, k, v, out, lse, false, false, st);
}

rsa_status rsa_text_full_attention(int64_t heads, int64_t n_queries, int64_t n_keys,
                                   int64_t head_dim, int64_t block, int32_t dtype, const void* q,
                                   const void* k, const void* v, void* out, float* lse,
                                   void* workspace, void* stream) {
  g_launches = 0;
  if (block <= 0) return fail(RSA_ERR_BLOCK_SIZE, "block size must be positive");
  if (n_keys < 1) return fail(RSA_ERR_SHAPE, "need at least one key row");
  // keys tiled by `block` from row 0 (kernel.py:138): full tiles as "video"
  // blocks, the remainder as one ragged trailing block
  rsa_shape s{heads, (n_keys / block) * block, n_keys % block, head_dim, block, dtype, RSA_KERNEL_SIMT, 0, 0};
  rsa::Geometry g;
  g.H = heads; g.Tv = s.t_video; g.Tt = s.t_text; g.T = n_keys; g.d = head_dim; g.B = block;
  g.N = g.Tv / block; g.n_text = g.Tt > 0 ? 1 : 0; g.M = g.N + g.n_text;
  g.last_len = g.Tt; g.n_cols = 0; g.dtype = dtype; g.q_last = block;
  g.hb = heads; g.s_tok = head_dim; g.s_head = n_keys * head_dim; g.s_batch = heads * n_keys * head_dim;
  g.o_hb = g.hb; g.o_tok = g.s_tok; g.o_head = g.s_head; g.o_batch = g.s_batch;
  g.qt_rows = n_queries; g.qt_row0 = 0; g.q_rows = n_queries;
  if (dtype < RSA_BF16 || dtype > RSA_F64) return fail(RSA_ERR_SHAPE, "bad dtype");
  if (head_dim < 1 || head_dim > (dtype == RSA_F64 ? 128 : 256))
    return fail(RSA_ERR_UNSUPPORTED, "head_dim out of range");
  if (n_queries == 0) return RSA_OK;
  rsa::Workspace ws;
  memset(&ws, 0, sizeof(ws));
  (void)workspace;
  cudaError_t e = rsa::launch_attn_simt(g, q, k, v, out, lse, ws, false, true,
                                        static_cast<cudaStream_t>(stream), &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "attn_simt(text)");
  return RSA_OK;
}

rsa_status rsa_morton_permutation(int64_t t, int64_t h, int64_t w, int32_t* perm) {
  if (t < 1 || h < 1 || w < 1 || t >= (1 << 21) || h >= (1 << 21) || w >= (1 << 21))
    return fail(RSA_ERR_SHAPE, "grid_dims must be positive and < 2^21 each");
  if (t * h * w >= ((int64_t)1 << 31)) return fail(RSA_ERR_UNSUPPORTED, "more than 2^31 tokens");
  if (!perm) return fail(RSA_ERR_SHAPE, "null pointer");
  rsa::morton_permutation_host(t, h, w, perm);
  return RSA_OK;
}

rsa_status rsa_permute_rows(const rsa_shape* shape, const int32_t* perm, const void* src, void* dst,
                            int32_t inverse, void* stream) {
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  if (!perm || !src || !dst) return fail(RSA_ERR_SHAPE, "null pointer");
  if (src == dst) return fail(RSA_ERR_SHAPE, "rsa_permute_rows cannot run in place");
  cudaError_t e = rsa::launch_permute_rows(g, perm, src, dst, inverse != 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "permute_rows");
  return RSA_OK;
}

size_t rsa_permuted_buffer_size(const rsa_shape* shape) {
  rsa::Geometry g;
  if (make_geometry(shape, &g) != RSA_OK) return 0;
  const size_t esz = g.dtype == RSA_BF16 ? 2 : g.dtype == RSA_F32 ? 4 : 8;
  return 3 * (size_t)g.H * g.T * g.d * esz;   // permuted K, V and Q
}

rsa_status rsa_forward_permuted(const rsa_shape* shape, const rsa_config* cfg, const void* q, const void* k,
                                const void* v, const int32_t* perm, void* perm_buf, void* out, float* lse,
                                void* workspace, void* stream) {
  g_launches = 0;
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  s = check_config(cfg);
  if (s != RSA_OK) return s;
  if (!q || !k || !v || !perm || !perm_buf || !out || !workspace) return fail(RSA_ERR_SHAPE, "null pointer");
  if (!use_tc(shape, g)) return fail(RSA_ERR_UNSUPPORTED, "the fused permuted path needs bf16 and the tcgen05 kernel");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  rsa::Workspace ws = bind(g, workspace);
  char* kp = static_cast<char*>(perm_buf);
  char* vp = kp + (size_t)g.H * g.T * g.d * 2;
  char* qp = vp + (size_t)g.H * g.T * g.d * 2;
  cudaError_t e = cudaMemsetAsync(ws.status, 0, 64, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset status");
  // K1: gathers the video rows in permuted order, writes permuted Q, K and V
  e = rsa::launch_pool(g, q, k, v, ws, st, &g_launches, perm, kp, vp, qp);
  if (e == cudaErrorNotSupported)
    return fail(RSA_ERR_UNSUPPORTED, "the fused permuted path needs 16-byte aligned bf16 rows, d in {64, 128}");
  if (e != cudaSuccess) return cuda_fail(e, "pool(permuted)");
  const int64_t k_floor = (int64_t)std::ceil(cfg->top_k_fraction * (double)g.M);
  e = rsa::launch_select(g, *cfg, k_floor, ws, st, &g_launches);
  if (e != cudaSuccess) return cuda_fail(e, "select");
  // the text query rows of the permuted Q copy are the original ones
  if (g.Tt > 0) {
    const size_t pitch = (size_t)g.T * g.d * 2;
    e = cudaMemcpy2DAsync(qp + (size_t)g.Tv * g.d * 2, pitch, static_cast<const char*>(q) + (size_t)g.Tv * g.d * 2,
                          pitch, (size_t)g.Tt * g.d * 2, (size_t)g.H, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return cuda_fail(e, "text Q copy");
  }
  // K3 on the permuted Q/K/V (the persistent kernel gathers Q rows through perm
  // instead); O / LSE rows scattered back via perm
  return run_attention(shape, g, ws, q, kp, vp, out, lse, rectifies(cfg->variant), true, st, perm, qp);
}

size_t rsa_diagnostics_scratch_size(const rsa_shape* shape) {
  rsa::Geometry g;
  if (make_geometry(shape, &g) != RSA_OK) return 0;
  return rsa::diag_scratch_size(g);
}

rsa_status rsa_diagnostics(const rsa_shape* shape, const void* q, const void* k, void* workspace, double* gain,
                           double* error, double* exact_gain, double* exact_error, double* s_sum,
                           double* s_sum_pool, void* scratch, void* stream) {
  g_launches = 0;
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  if (g.q_last != g.B) return fail(RSA_ERR_UNSUPPORTED, "diagnostics need full video blocks");
  if (!q || !k || !workspace || !gain || !error || !exact_gain || !exact_error || !s_sum || !s_sum_pool || !scratch)
    return fail(RSA_ERR_SHAPE, "null pointer");
  rsa::Workspace ws = bind(g, workspace);
  cudaError_t e = rsa::launch_diagnostics(g, q, k, ws, gain, error, exact_gain, exact_error, s_sum, s_sum_pool,
                                          scratch, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "diagnostics");
  return RSA_OK;
}

size_t rsa_dense_reference_scratch_size(const rsa_shape* shape) {
  rsa::Geometry g;
  if (make_geometry(shape, &g) != RSA_OK) return 0;
  return rsa::dense_scratch_size(g);
}

rsa_status rsa_dense_reference(const rsa_shape* shape, const void* q, const void* k, const void* v, double* out,
                               void* scratch, void* stream) {
  g_launches = 0;
  rsa::Geometry g;
  rsa_status s = make_geometry(shape, &g);
  if (s != RSA_OK) return s;
  if (g.q_last != g.B) return fail(RSA_ERR_UNSUPPORTED, "diagnostics need full video blocks");
  if (!q || !k || !v || !out || !scratch) return fail(RSA_ERR_SHAPE, "null pointer");
  cudaError_t e = rsa::launch_dense_reference(g, q, k, v, out, scratch, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "dense_reference");
  return RSA_OK;
}

rsa_status rsa_check_device_status(void* workspace, void* stream) {
  if (!workspace) return fail(RSA_ERR_SHAPE, "null workspace");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t flags[4] = {0, 0, 0, 0};
  cudaError_t e = cudaMemcpyAsync(flags, workspace, sizeof(flags), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "status readback");
  return rsa_status_from_flags(flags);
}

rsa_status rsa_accumulate_status(const void* workspace, int32_t* status_accum, void* stream) {
  if (!workspace || !status_accum) return fail(RSA_ERR_SHAPE, "null pointer");
  accumulate_status_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const int32_t*>(workspace), status_accum);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? RSA_OK : cuda_fail(e, "accumulate_status");
}

rsa_status rsa_status_from_flags(const int32_t* flags) {
  if (!flags) return fail(RSA_ERR_SHAPE, "null pointer");
  if (flags[rsa::ST_NONFINITE]) return fail(RSA_ERR_SHAPE, "q/k/v contain non-finite entries");
  if (flags[rsa::ST_DEGENERATE])
    return fail(RSA_ERR_DEGENERATE_ROW, "reallocation denominator is zero on some rows");
  if (flags[rsa::ST_EMPTY_ROW]) return fail(RSA_ERR_EMPTY_ROW, "a mask row retains no key block");
  return RSA_OK;
}

int32_t rsa_last_launch_count(void) { return g_launches; }
const char* rsa_last_error(void) { return g_last_error.c_str(); }
const char* rsa_version(void) { return "rsa_b200 0.1.0 (sm_100a)"; }

}  // extern "C"
