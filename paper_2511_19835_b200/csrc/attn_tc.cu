// K3 + K4 (tensor-core variant): block-sparse flash attention on tcgen05 with
// the IPAR rescale and GAPR compensation fused into the epilogue.
//
// Reference semantics: _query_block_pass / block_sparse_attention /
// text_full_attention (pkg/src/rectattn/kernel.py:43-145) -- per query block
// an online softmax over the retained kv blocks in ascending order -- and
// apply_rectification (rectify.py:66-89): O' = R_n O + sum_applied a_pool v_pool.
//
// One CTA = one 128-row query tile (UMMA M = 128): one video query block for
// B = 128, two for B = 64 (walking the union of their kv lists with per-row
// membership), or 128 text queries (every kv block).  Warp roles:
//   warp 0      TMA producer: Q once, then K_j / V_j tiles (box 64 x B, 128B
//               swizzle) into an NST-stage ring in exactly the order the MMA
//               warp consumes them (K0 K1 V0 K2 V1 ... V_{c-1})
//   warp 1      single-thread tcgen05.mma issuer:
//                 S_j = Q K_j^T  (SS, into TMEM S buffer j%2)   -- issued one
//                 step ahead, so it runs while softmax works on S_{j-1}
//                 O  += P_j V_j  (TS: P_j read straight from TMEM)
//   warp 2      TMEM allocation / release
//   warps 4-7   softmax: one query row per thread (TMEM lane), fp32 online
//               softmax in the log2 domain with lazy (threshold 2^8) O
//               rescaling, P packed to bf16 back into the S columns; then the
//               epilogue O / l * R_n + comp_n -> bf16 store, LSE.
// TMEM columns: S0 [0,B), S1 [B,2B), O [2B, 2B+D).
#include "rsa_internal.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

namespace rsa {
namespace {

constexpr int kThreads = 256;
constexpr int kNst = 4;                 // K/V ring stages
constexpr float kRescaleThreshold = 8.0f;  // log2 units: rescale O only if max grows by > 2^8

template <int D, int BKV>
struct Cfg {
  static constexpr int PANELS = D / 64;
  static constexpr int Q_PANEL = 128 * 128;     // bytes: 128 rows x 128 B
  static constexpr int KV_PANEL = BKV * 128;    // bytes: B rows x 128 B
  static constexpr int Q_BYTES = 128 * D * 2;
  static constexpr int STAGE = BKV * D * 2;
  static constexpr int O_COL = 2 * BKV;
  static constexpr int TMEM_COLS = (2 * BKV + D) <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + Q_BYTES + kNst * STAGE + 256;
  static constexpr uint32_t IDESC_S = ptx::idesc_bf16(128, BKV, false);
  static constexpr uint32_t IDESC_O = ptx::idesc_bf16(128, D, true);
};

struct TcParams {
  Geometry g;
  Workspace ws;
  __nv_bfloat16* out;
  float* lse;
  int rectify;
  int64_t n_text_tiles;
  int64_t text_tiles_per_head;
  int64_t video_tiles_per_head;
  float scale_log2;  // log2(e) / sqrt(d)
};

template <int D, int BKV>
__global__ void __launch_bounds__(kThreads, 1)
attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
               const __grid_constant__ CUtensorMap tm_v, const TcParams P) {
  using C = Cfg<D, BKV>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* q_s = base;
  uint8_t* kv_s = base + C::Q_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(kv_s + kNst * C::STAGE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + kNst;
  uint64_t* s_full = kv_empty + kNst;      // [2]
  uint64_t* p_full = s_full + 2;           // [2]
  uint64_t* pv_done = p_full + 2;          // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 1);

  const Geometry& g = P.g;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // ---- tile decode (LPT order: text tiles first) ----
  const int64_t bid = blockIdx.x;
  const bool text = bid < P.n_text_tiles;
  int64_t h, q_row0, rows_valid, count;
  const int32_t* list = nullptr;
  if (text) {
    h = bid / P.text_tiles_per_head;
    const int64_t t = bid % P.text_tiles_per_head;
    q_row0 = g.Tv + t * 128;
    rows_valid = min((int64_t)128, g.Tt - t * 128);
    count = g.M;
  } else {
    const int64_t b = bid - P.n_text_tiles;
    h = b / P.video_tiles_per_head;
    const int64_t t = b % P.video_tiles_per_head;
    q_row0 = t * 128;
    rows_valid = min((int64_t)128, g.Tv - q_row0);
    count = P.ws.tile_count[h * P.video_tiles_per_head + t];
    list = P.ws.tile_list + (h * P.video_tiles_per_head + t) * g.M;
  }

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < kNst; ++i) {
      ptx::mbar_init(kv_full + i, 1);
      ptx::mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(s_full + i, 1);
      ptx::mbar_init(p_full + i, 128);
    }
    ptx::mbar_init(pv_done, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0 && count > 0) {
      ptx::prefetch_tmap(&tm_q);
      ptx::prefetch_tmap(&tm_k);
      ptx::prefetch_tmap(&tm_v);
      ptx::mbar_expect_tx(q_full, C::Q_BYTES);
#pragma unroll
      for (int p = 0; p < C::PANELS; ++p)
        ptx::tma_load_3d(q_s + p * C::Q_PANEL, &tm_q, q_full, 64 * p, (int)q_row0, (int)h);
      int it = 0;
      auto load = [&](int64_t j, bool is_v) {
        const int s = it % kNst;
        const uint32_t ph = (it / kNst) & 1;
        const int64_t m = list ? (list[j] & 0xFFFFFF) : j;
        ptx::mbar_wait(kv_empty + s, ph ^ 1);
        ptx::mbar_expect_tx(kv_full + s, C::STAGE);
        uint8_t* dst = kv_s + s * C::STAGE;
#pragma unroll
        for (int p = 0; p < C::PANELS; ++p)
          ptx::tma_load_3d(dst + p * C::KV_PANEL, is_v ? &tm_v : &tm_k, kv_full + s, 64 * p,
                           (int)(m * g.B), (int)h);
        ++it;
      };
      for (int64_t j = 0; j <= count; ++j) {
        if (j < count) load(j, false);
        if (j >= 1) load(j - 1, true);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0 && count > 0) {
      ptx::mbar_wait(q_full, 0);
      ptx::tc_fence_after();
      const uint32_t q_addr = ptx::smem_u32(q_s);
      const uint32_t kv_addr = ptx::smem_u32(kv_s);
      int it = 0;
      for (int64_t j = 0; j <= count; ++j) {
        if (j < count) {
          const int s = it % kNst;
          ptx::mbar_wait(kv_full + s, (it / kNst) & 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)((j & 1) * BKV);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (uint32_t)((k % 4) * 32);   // 16 bf16 = 32 B inside the 128 B row
            const uint64_t a = ptx::sw128_desc(q_addr + (k / 4) * C::Q_PANEL + off, 16, 1024);
            const uint64_t b = ptx::sw128_desc(kv_addr + s * C::STAGE + (k / 4) * C::KV_PANEL + off, 16, 1024);
            ptx::mma_ss(d_tmem, a, b, C::IDESC_S, k > 0);
          }
          ptx::tc_commit(kv_empty + s);
          ptx::tc_commit(s_full + (j & 1));
          ++it;
        }
        if (j >= 1) {
          const int64_t jj = j - 1;
          ptx::mbar_wait(p_full + (jj & 1), (uint32_t)((jj >> 1) & 1));
          const int s = it % kNst;
          ptx::mbar_wait(kv_full + s, (it / kNst) & 1);
          ptx::tc_fence_after();
          const uint32_t a_tmem = tmem + (uint32_t)((jj & 1) * BKV);
#pragma unroll
          for (int k = 0; k < BKV / 16; ++k) {
            const uint64_t b = ptx::sw128_desc(kv_addr + s * C::STAGE + k * 2048, C::KV_PANEL, 1024);
            ptx::mma_ts(tmem + C::O_COL, a_tmem + k * 8, b, C::IDESC_O, (jj > 0 || k > 0) ? 1u : 0u);
          }
          ptx::tc_commit(kv_empty + s);
          ptx::tc_commit(pv_done);
          ++it;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax + epilogue =====================
    const int quad = warp - 4;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const int sub = row / (int)g.B;          // which member query block of the tile
    float m_run = -INFINITY, l_run = 0.f;
    const float sl2 = P.scale_log2;
    for (int64_t j = 0; j < count; ++j) {
      int64_t m;
      bool member;
      if (list) {
        const int32_t e = list[j];
        m = e & 0xFFFFFF;
        member = (e >> (24 + sub)) & 1;
      } else {
        m = j;
        member = true;
      }
      const int len = (m == g.M - 1 && g.n_text > 0) ? (int)g.last_len : (int)g.B;
      ptx::mbar_wait(s_full + (j & 1), (uint32_t)((j >> 1) & 1));
      ptx::tc_fence_after();
      const uint32_t s_addr = lane_base + (uint32_t)((j & 1) * BKV);
      uint32_t sr[BKV / 32][32];
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) ptx::tmem_ld32(s_addr + c * 32, sr[c]);
      ptx::tmem_ld_wait();
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float s = __uint_as_float(sr[c][i]);
          if (!member || c * 32 + i >= len) s = -INFINITY;
          sr[c][i] = __float_as_uint(s);
          mx = fmaxf(mx, s);
        }
      const float m_blk = mx * sl2;              // -inf if the row retains nothing here
      const float m_old = m_run;
      float alpha = 1.f;
      bool rescale_o = false;
      if (m_blk > m_run + kRescaleThreshold || (m_run == -INFINITY && m_blk > -INFINITY)) {
        alpha = (m_old == -INFINITY) ? 0.f : ptx::ex2(m_old - m_blk);
        rescale_o = (m_old != -INFINITY) && j > 0;
        m_run = m_blk;
      }
      const float base_m = (m_run == -INFINITY) ? 0.f : m_run;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < BKV / 32; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = ptx::ex2(fmaf(__uint_as_float(sr[c][2 * i]), sl2, -base_m));
          const float p1 = ptx::ex2(fmaf(__uint_as_float(sr[c][2 * i + 1]), sl2, -base_m));
          sum += p0 + p1;
          pk[i] = ptx::pack_bf16(p0, p1);
        }
        ptx::tmem_st16(s_addr + c * 16, pk);
      }
      l_run = l_run * alpha + sum;
      // tcgen05.ld/st are warp-collective (.sync.aligned): the correction runs
      // for the whole warp whenever any of its rows needs it
      if (__any_sync(0xffffffffu, rescale_o)) {
        // O must hold exactly PV_0..PV_{j-1} before it is rescaled
        ptx::mbar_wait(pv_done, (uint32_t)((j - 1) & 1));
        ptx::tc_fence_after();
        const float a = rescale_o ? alpha : 1.f;
#pragma unroll
        for (int c = 0; c < D / 32; ++c) {
          uint32_t o[32];
          ptx::tmem_ld32(lane_base + C::O_COL + c * 32, o);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
          ptx::tmem_st32(lane_base + C::O_COL + c * 32, o);
        }
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full + (j & 1));
    }

    // ---- epilogue: O / l, rectification (rectify.py:66-89), bf16 store, LSE ----
    if (count > 0) {
      ptx::mbar_wait(pv_done, (uint32_t)((count - 1) & 1));
      ptx::tc_fence_after();
    }
    const bool valid = row < rows_valid;
    const int64_t grow = q_row0 + row;
    float rfac = 1.f;
    const double* comp = nullptr;
    if (!text && P.rectify && valid) {
      const int64_t n_blk = grow / g.B;
      rfac = P.ws.r_eff[h * g.N + n_blk];
      comp = P.ws.comp + (h * g.N + n_blk) * D;
    }
    const float inv_l = (count > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
    __nv_bfloat16* orow = P.out + (h * g.T + grow) * D;
#pragma unroll
    for (int c = 0; c < D / 32; ++c) {
      uint32_t o[32];
      ptx::tmem_ld32(lane_base + C::O_COL + c * 32, o);
      ptx::tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int v8 = 0; v8 < 4; ++v8) {
          uint32_t w[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int col = c * 32 + v8 * 8 + 2 * i;
            float y0 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * i]) * inv_l * rfac;
            float y1 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * i + 1]) * inv_l * rfac;
            if (comp) {
              y0 += (float)comp[col];
              y1 += (float)comp[col + 1];
            }
            w[i] = ptx::pack_bf16(y0, y1);
          }
          *reinterpret_cast<uint4*>(orow + c * 32 + v8 * 8) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
    if (valid && P.lse)
      P.lse[h * g.T + grow] = l_run > 0.f ? (log2f(l_run) + m_run) * 0.69314718055994531f : -INFINITY;
  }

  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_tmap(CUtensorMap* tm, const void* ptr, const Geometry& g, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {(cuuint64_t)g.d, (cuuint64_t)g.T, (cuuint64_t)g.H};
  cuuint64_t strides[2] = {(cuuint64_t)g.d * 2, (cuuint64_t)g.T * g.d * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int D, int BKV>
cudaError_t launch_cfg(const Geometry& g, const void* q, const void* k, const void* v, void* out, float* lse,
                       const Workspace& ws, bool rectify, bool text, cudaStream_t st) {
  using C = Cfg<D, BKV>;
  CUtensorMap tq, tk, tv;
  if (!make_tmap(&tq, q, g, 128) || !make_tmap(&tk, k, g, BKV) || !make_tmap(&tv, v, g, BKV))
    return cudaErrorInvalidValue;
  TcParams P;
  P.g = g;
  P.ws = ws;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.lse = lse;
  P.rectify = rectify ? 1 : 0;
  P.text_tiles_per_head = (g.Tt + 127) / 128;
  P.n_text_tiles = text ? g.H * P.text_tiles_per_head : 0;
  P.video_tiles_per_head = (g.N * g.B + 127) / 128;
  P.scale_log2 = (float)(1.4426950408889634 / sqrt((double)g.d));
  auto kern = attn_tc_kernel<D, BKV>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  const int64_t tiles = P.n_text_tiles + g.H * P.video_tiles_per_head;
  kern<<<(unsigned)tiles, kThreads, C::SMEM, st>>>(tq, tk, tv, P);
  return cudaGetLastError();
}

}  // namespace

bool tc_supported(const Geometry& g) {
  return g.dtype == RSA_BF16 && (g.d == 64 || g.d == 128) && (g.B == 64 || g.B == 128) &&
         g.T * g.d < (int64_t(1) << 31) && g.H < 65536 && encode_fn() != nullptr;
}

cudaError_t launch_attn_tc(const Geometry& g, const void* q, const void* k, const void* v, void* out, float* lse,
                           const Workspace& ws, bool rectify, bool text, cudaStream_t st, int* launches) {
  ++*launches;
  if (g.d == 128 && g.B == 128) return launch_cfg<128, 128>(g, q, k, v, out, lse, ws, rectify, text, st);
  if (g.d == 128 && g.B == 64) return launch_cfg<128, 64>(g, q, k, v, out, lse, ws, rectify, text, st);
  if (g.d == 64 && g.B == 128) return launch_cfg<64, 128>(g, q, k, v, out, lse, ws, rectify, text, st);
  return launch_cfg<64, 64>(g, q, k, v, out, lse, ws, rectify, text, st);
}

}  // namespace rsa
