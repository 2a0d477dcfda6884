// torch_ops.cpp -- TORCH_LIBRARY registration of the hot path as
// torch.ops.rsa_b200.* (SURVEY.md 8b "Registered as torch.ops.rsa.* via
// TORCH_LIBRARY, with fake/meta kernels so torch.compile can trace").
//
// A thin host layer over the C ABI (include/rsa_b200.h): it validates the
// tensors, allocates the output and the workspace from the caching allocator,
// and calls rsa_forward / rsa_forward_strided on the current stream.  No
// compute happens here and there is no CPU kernel: the ops are registered for
// the CUDA dispatch key only (plus Meta for tracing), so a CPU tensor raises.
//
// The op is the batched model-facing form of the reference's
// rectified_attention_pipeline(problem, config, variant)
// (pkg/src/rectattn/rectify.py:107-176): q/k/v are [..., T, d] with the last
// num_text_tokens rows text (core.py:6-8), the config fields are
// SparsityConfig's (masks.py:30-33) and `variant` one of VARIANTS
// (rectify.py:23-24).  Errors carry the reference exception's class name as
// the message prefix ("ShapeError: ..."); paper_2511_19835_b200.ops re-raises
// them as those classes (errors.py:4-45).

#include <ATen/ATen.h>
#include <ATen/cuda/CUDAContext.h>
#include <c10/cuda/CUDAGuard.h>
#include <torch/library.h>

#include <string>
#include <vector>

#include "rsa_b200.h"

namespace {

const char* status_class(int st) {
  switch (st) {
    case RSA_ERR_SHAPE: return "ShapeError";
    case RSA_ERR_BLOCK_SIZE: return "BlockSizeError";
    case RSA_ERR_EMPTY_ROW: return "EmptyRowError";
    case RSA_ERR_CONFIG: return "ConfigError";
    case RSA_ERR_DEGENERATE_ROW: return "DegenerateRowError";
    default: return "NativeError";
  }
}

[[noreturn]] void raise_status(int st) {
  TORCH_CHECK(false, status_class(st), ": ", rsa_last_error());
}

void check(rsa_status st) {
  if (st != RSA_OK) raise_status(st);
}

int32_t dtype_code(at::ScalarType t) {
  switch (t) {
    case at::kBFloat16: return RSA_BF16;
    case at::kFloat: return RSA_F32;
    case at::kDouble: return RSA_F64;
    default:
      TORCH_CHECK(false, "ShapeError: q/k/v must be bfloat16, float32 or float64, got ", t);
  }
}

int32_t variant_code(const std::string& v) {
  static const char* names[] = {"full", "sparse-unrectified", "sparse-rectified", "sparse-rectified-no-gapr",
                                "compensate-all"};
  for (int i = 0; i < 5; ++i)
    if (v == names[i]) return i;
  TORCH_CHECK(false, "ConfigError: unknown variant '", v, "'");  // rectify.py:118-119
}

// Concrete metadata of a (possibly symbolic, under torch.compile dynamic
// shapes) tensor: every size / stride the host logic reads is guarded, so a
// traced graph is specialised on exactly the facts the CUDA kernel branches
// on.  Outputs are still built from the symbolic sizes.
struct Meta {
  std::vector<int64_t> sizes, strides;
  int64_t offset = 0, itemsize = 0;
  bool contiguous = false;
  int64_t dim() const { return static_cast<int64_t>(sizes.size()); }
  int64_t size(int64_t i) const { return sizes[i < 0 ? i + dim() : i]; }
  int64_t stride(int64_t i) const { return strides[i < 0 ? i + dim() : i]; }
};

Meta meta_of(const at::Tensor& x) {
  Meta m;
  for (const auto& s : x.sym_sizes()) m.sizes.push_back(s.guard_int(__FILE__, __LINE__));
  for (const auto& s : x.sym_strides()) m.strides.push_back(s.guard_int(__FILE__, __LINE__));
  m.offset = x.sym_storage_offset().guard_int(__FILE__, __LINE__);
  m.itemsize = static_cast<int64_t>(x.element_size());
  m.contiguous = x.sym_is_contiguous().guard_bool(__FILE__, __LINE__);
  return m;
}

// rsa_layout of a [..., T, d] view of up to 4 dimensions whose rows are
// contiguous and whose token / head / batch strides are multiples of 8
// elements (16-byte TMA rows, 16-byte aligned start); false otherwise.  Reads
// metadata only (sizes, strides, storage offset), so the Meta kernel makes the
// same choice as the CUDA kernel.
bool layout_of(const Meta& x, rsa_layout* out) {
  if (x.dim() > 4 || x.stride(-1) != 1) return false;
  if ((x.offset * x.itemsize) % 16) return false;
  std::vector<int64_t> shp = x.sizes, st = x.strides;
  while (shp.size() < 4) {
    shp.insert(shp.begin(), 1);
    st.insert(st.begin(), 0);
  }
  const int64_t B = shp[0], H = shp[1], T = shp[2];
  const int64_t tok = st[2];
  const int64_t head = H > 1 ? st[1] : tok * T;   // a size-1 dimension's stride is never used
  const int64_t bat = B > 1 ? st[0] : head * H;
  if (tok % 8 || head % 8 || bat % 8 || head == 0 || bat == 0) return false;   // broadcast dims: copy
  *out = rsa_layout{H, tok, head, bat};
  return true;
}

// The no-copy strided path: non-contiguous bf16 q/k/v sharing one stride
// pattern at a tcgen05 shape (rsa_forward_strided, rsa_b200.h).  Anything
// else is made contiguous first.
bool use_strided(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v, int64_t block, rsa_layout* lay) {
  const Meta mq = meta_of(q), mk = meta_of(k), mv = meta_of(v);
  if (mq.contiguous && mk.contiguous && mv.contiguous) return false;
  if (q.scalar_type() != at::kBFloat16 || mq.strides != mk.strides || mq.strides != mv.strides) return false;
  const int64_t d = mq.size(-1);
  if ((d != 64 && d != 128) || (block != 64 && block != 128)) return false;
  rsa_layout lk, lv;
  return layout_of(mq, lay) && layout_of(mk, &lk) && layout_of(mv, &lv);
}

// A dense tensor of x's shape whose dimensions are laid out in x's stride
// order: the output of a [B, T, 3, H, d] fused-qkv slice viewed [B, H, T, d] is
// a dense [B, T, H, d] buffer (what the caller's next projection reads).
at::Tensor dense_like(const at::Tensor& x) {
  const Meta m = meta_of(x);
  const int64_t n = m.dim();
  std::vector<int64_t> order(n), inv(n);
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return m.stride(a) > m.stride(b); });
  std::vector<c10::SymInt> sizes;
  for (int64_t i = 0; i < n; ++i) sizes.push_back(x.sym_size(order[i]));
  for (int64_t i = 0; i < n; ++i) inv[order[i]] = i;
  return at::empty_symint(sizes, x.options()).permute(inv);
}

struct Call {
  rsa_shape shape{};
  rsa_config cfg{};
};

Call plan(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v, int64_t num_text_tokens, int64_t block,
          double top_k_fraction, double weight_threshold, int64_t adjacency_radius, bool force_text_blocks,
          const std::string& variant) {
  const Meta mq = meta_of(q), mk = meta_of(k), mv = meta_of(v);
  TORCH_CHECK(mq.dim() >= 3 && mq.sizes == mk.sizes && mk.sizes == mv.sizes,
              "ShapeError: q/k/v must share a [..., T, d] shape, got ", q.sym_sizes(), ", ", k.sym_sizes(), ", ",
              v.sym_sizes());
  TORCH_CHECK(q.scalar_type() == k.scalar_type() && k.scalar_type() == v.scalar_type(),
              "ShapeError: q/k/v dtypes differ (core.py:73-75)");
  Call c;
  const int64_t T = mq.size(-2), d = mq.size(-1);
  c.shape.heads = 1;
  for (int64_t i = 0; i + 2 < mq.dim(); ++i) c.shape.heads *= mq.size(i);
  c.shape.t_video = T - num_text_tokens;
  c.shape.t_text = num_text_tokens;
  c.shape.head_dim = d;
  c.shape.block = block;
  c.shape.dtype = dtype_code(q.scalar_type());
  c.shape.kernel = RSA_KERNEL_AUTO;
  c.cfg.top_k_fraction = top_k_fraction;
  c.cfg.weight_threshold = weight_threshold;
  c.cfg.adjacency_radius = static_cast<int32_t>(adjacency_radius);
  c.cfg.force_text_blocks = force_text_blocks ? 1 : 0;
  c.cfg.variant = variant_code(variant);
  rsa_grid grid;
  check(rsa_plan(&c.shape, &c.cfg, &grid));
  return c;
}

// Runs K1 -> K2 -> K3+K4 on the current stream; returns (out, workspace).
std::pair<at::Tensor, at::Tensor> forward(const at::Tensor& q_in, const at::Tensor& k_in, const at::Tensor& v_in,
                                          const Call& c) {
  TORCH_CHECK(q_in.is_cuda() && k_in.device() == q_in.device() && v_in.device() == q_in.device(),
              "ShapeError: q, k and v must be CUDA tensors on one device");
  c10::cuda::CUDAGuard guard(q_in.device());
  cudaStream_t stream = at::cuda::getCurrentCUDAStream(q_in.device().index()).stream();
  auto ws = at::empty({static_cast<int64_t>(rsa_workspace_size(&c.shape))},
                      q_in.options().dtype(at::kByte));
  rsa_layout lay;
  if (use_strided(q_in, k_in, v_in, c.shape.block, &lay)) {
    at::Tensor out = dense_like(q_in);
    rsa_layout olay;
    TORCH_CHECK(layout_of(meta_of(out), &olay), "NativeError: output layout");
    check(rsa_forward_strided(&c.shape, &c.cfg, &lay, &olay, q_in.data_ptr(), k_in.data_ptr(), v_in.data_ptr(),
                              out.data_ptr(), nullptr, ws.data_ptr(), stream));
    return {out, ws};
  }
  const at::Tensor q = q_in.contiguous(), k = k_in.contiguous(), v = v_in.contiguous();
  at::Tensor out = at::empty(q.sizes(), q.options());
  check(rsa_forward(&c.shape, &c.cfg, q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), nullptr,
                    ws.data_ptr(), stream));
  return {out, ws};
}

// Eager form: the device flags (non-finite input -> ShapeError, degenerate
// reallocation row, empty mask row; core.py:23-31, ipar.py:62-64,
// kernel.py:85-87) are checked after one stream synchronisation, like the
// reference's eager checks.
at::Tensor rsa_cuda(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v, int64_t num_text_tokens,
                    int64_t block, double top_k_fraction, double weight_threshold, int64_t adjacency_radius,
                    bool force_text_blocks, c10::string_view variant) {
  const Call c = plan(q, k, v, num_text_tokens, block, top_k_fraction, weight_threshold, adjacency_radius,
                      force_text_blocks, std::string(variant));
  auto [out, ws] = forward(q, k, v, c);
  c10::cuda::CUDAGuard guard(q.device());
  check(rsa_check_device_status(ws.data_ptr(), at::cuda::getCurrentCUDAStream(q.device().index()).stream()));
  return out;
}

// Non-synchronising form: (out, status int32[4]) where status holds this
// call's device flags (rsa_accumulate_status); raise_for_status() raises the
// reference exception once the caller synchronises anyway.
std::tuple<at::Tensor, at::Tensor> rsa_status_cuda(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v,
                                                   int64_t num_text_tokens, int64_t block, double top_k_fraction,
                                                   double weight_threshold, int64_t adjacency_radius,
                                                   bool force_text_blocks, c10::string_view variant) {
  const Call c = plan(q, k, v, num_text_tokens, block, top_k_fraction, weight_threshold, adjacency_radius,
                      force_text_blocks, std::string(variant));
  auto [out, ws] = forward(q, k, v, c);
  c10::cuda::CUDAGuard guard(q.device());
  at::Tensor status = at::zeros({4}, q.options().dtype(at::kInt));
  check(rsa_accumulate_status(ws.data_ptr(), status.data_ptr<int32_t>(),
                              at::cuda::getCurrentCUDAStream(q.device().index()).stream()));
  return {out, status};
}

// Meta (fake) kernels: the CUDA kernels' output metadata, for tracing and
// torch.compile.  Host-side validation runs here too, so a traced graph
// rejects the same shapes and configurations.
at::Tensor out_meta(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v, int64_t block) {
  rsa_layout lay;
  return use_strided(q, k, v, block, &lay) ? dense_like(q) : at::empty_symint(q.sym_sizes(), q.options());
}

at::Tensor rsa_meta(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v, int64_t num_text_tokens,
                    int64_t block, double top_k_fraction, double weight_threshold, int64_t adjacency_radius,
                    bool force_text_blocks, c10::string_view variant) {
  plan(q, k, v, num_text_tokens, block, top_k_fraction, weight_threshold, adjacency_radius, force_text_blocks,
       std::string(variant));
  return out_meta(q, k, v, block);
}

std::tuple<at::Tensor, at::Tensor> rsa_status_meta(const at::Tensor& q, const at::Tensor& k, const at::Tensor& v,
                                                   int64_t num_text_tokens, int64_t block, double top_k_fraction,
                                                   double weight_threshold, int64_t adjacency_radius,
                                                   bool force_text_blocks, c10::string_view variant) {
  plan(q, k, v, num_text_tokens, block, top_k_fraction, weight_threshold, adjacency_radius, force_text_blocks,
       std::string(variant));
  return {out_meta(q, k, v, block), at::empty({4}, q.options().dtype(at::kInt))};
}

}  // namespace

TORCH_LIBRARY(rsa_b200, m) {
  m.def("rectified_sparse_attention(Tensor q, Tensor k, Tensor v, int num_text_tokens, int block=128, "
        "float top_k_fraction=0.1, float weight_threshold=0.0, int adjacency_radius=0, "
        "bool force_text_blocks=False, str variant=\"sparse-rectified\") -> Tensor");
  m.def("rectified_sparse_attention_status(Tensor q, Tensor k, Tensor v, int num_text_tokens, int block=128, "
        "float top_k_fraction=0.1, float weight_threshold=0.0, int adjacency_radius=0, "
        "bool force_text_blocks=False, str variant=\"sparse-rectified\") -> (Tensor, Tensor)");
}

TORCH_LIBRARY_IMPL(rsa_b200, CUDA, m) {
  m.impl("rectified_sparse_attention", &rsa_cuda);
  m.impl("rectified_sparse_attention_status", &rsa_status_cuda);
}

TORCH_LIBRARY_IMPL(rsa_b200, Meta, m) {
  m.impl("rectified_sparse_attention", &rsa_meta);
  m.impl("rectified_sparse_attention_status", &rsa_status_meta);
}
