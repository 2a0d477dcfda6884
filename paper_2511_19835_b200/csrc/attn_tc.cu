// K3 + K4 (tensor-core variant): block-sparse flash attention on tcgen05 with
// the IPAR rescale and GAPR compensation fused into the epilogue.
//
// Reference semantics: _query_block_pass / block_sparse_attention /
// text_full_attention (pkg/src/rectattn/kernel.py:43-145) -- per query block
// an online softmax over the retained kv blocks in ascending order -- and
// apply_rectification (rectify.py:66-89): O' = R_n O + sum_applied a_pool v_pool.
//
// Two kernels, one per shape class:
//   attn_tc_pp_kernel          d = B = 128 (HunyuanVideo, Wan): two query tiles
//                              per CTA in independent ping-pong slots
//   attn_tc_persistent_kernel  B = 64 and/or d = 64 (and on request for
//                              d = B = 128): one query tile at a time per CTA
// Both are persistent (one CTA per SM) and walk 128-row query tiles head-major:
// video tiles over their kv lists, text tiles over every kv block in split-K
// chunks that text_combine_kernel merges.
#include "rsa_internal.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

#include <cuda.h>
#include <algorithm>
#include <cstdlib>
#include <cudaTypedefs.h>

namespace rsa {
namespace {

constexpr int kThreads = 384;   // 4 control warps + 8 softmax warps
constexpr float kRescaleThreshold = 12.0f;  // log2 units: rescale O only if the row max grows by > 2^12
                                            // (P <= 2^12 stays exact-range in bf16 / fp32; 8 measured ~1 % slower)
constexpr float kSpecSum = 8192.0f;         // paired-tile kernel: keep the running base while a block's row
                                            // sum of P stays <= 2^13 (so does every P)

// persistent kernel: Q resident in TMEM (A operand of the S MMAs), two S/P
// TMEM buffers, a K/V ring of NST stages in shared memory
template <int D, int BKV>
struct Cfg {
  static constexpr int NS = 2;
  static constexpr int NST = BKV * D * 2 <= 16384 ? 8 : 6;
  static constexpr int PANELS = D / 64;
  static constexpr int Q_PANEL = 128 * 128;     // bytes: 128 rows x 128 B
  static constexpr int KV_PANEL = BKV * 128;    // bytes: B rows x 128 B
  static constexpr int Q_BYTES = 128 * D * 2;
  static constexpr int STAGE = BKV * D * 2;
  static constexpr int O_COL = NS * BKV;
  static constexpr int Q_COL = NS * BKV + D;      // Q (bf16 pairs) resident in TMEM
  static constexpr int TMEM_USED = NS * BKV + D + D / 2;
  static constexpr int TMEM_COLS = TMEM_USED <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + NST * STAGE + 256 + 768 * 4;
  static constexpr uint32_t IDESC_S = ptx::idesc_bf16(128, BKV, false);
  static constexpr uint32_t IDESC_O = ptx::idesc_bf16(128, D, true);   // PV B operand: V tiles (MN-major)
};

struct TcParams {
  Geometry g;
  Workspace ws;
  __nv_bfloat16* out;
  const __nv_bfloat16* q;
  float* lse;
  const int32_t* perm;   // token permutation (video row r = original row perm[r]) or null
  float* text_part;   // [H][text tiles][chunks][128][D] unnormalised partial O
  float2* text_ml;    // [H][text tiles][chunks][128] (row max log2, row sum)
  int rectify;
  int64_t text_tiles_per_head;   // 128-row text query tiles per head (0: no text queries)
  int64_t text_chunks;           // kv-block chunks per text tile (split-K)
  int64_t chunk_blocks;          // kv blocks per chunk
  int64_t video_tiles_per_head;
  int64_t tiles_per_head;        // text_tiles_per_head * text_chunks + video_tiles_per_head
  float scale_log2;  // log2(e) / sqrt(d)
  int qring;         // persistent kernel: each tile's Q rows arrive by TMA in a K/V ring stage
};


// ============================================================================
// Persistent variant (production path): one CTA per SM walks the tiles
// blockIdx.x, blockIdx.x + gridDim.x, ... (head-major order, so the SMs work
// on ~one head's K/V at a time).  TMEM allocation, barrier set-up and the
// K/V ring persist across tiles; barrier phases and the S/P buffer index run
// on per-CTA step counters.  At a tile boundary the softmax warps store the
// next tile's Q rows into TMEM as soon as the last S of the current tile has
// been read, so the MMA warp starts the next tile's S_0, S_1 while the same
// warps run the current tile's epilogue; PV_0 of the next tile (which
// overwrites O) waits for its P_0, i.e. after that epilogue.  This removes the
// per-CTA launch gap (~8 us), set-up and Q-load latency of the one-tile
// kernel (profiles/r01j: 16 us of ~117 us per tile).
// ============================================================================
// 64 columns x box rows of head h starting at token row `row` (4-D tensor
// maps over (d, T, head of the batch entry, batch entry): any row-contiguous
// [B, H, T, d] or [B, T, H, d] view, see make_rows_tmap)
__device__ __forceinline__ void tma_rows(void* dst, const CUtensorMap* tm, uint64_t* bar, int col, int row, int64_t h,
                                         const Geometry& g, uint64_t policy) {
  const int hb = (int)g.hb, hh = (int)h;
  ptx::tma_load_4d_hint(dst, tm, bar, col, row, hh % hb, hh / hb, policy);
}

struct TileDesc {
  int64_t h, q_row0, rows_valid, count, m_first, part;
  const int32_t* list;
  bool text;
};

__device__ __forceinline__ TileDesc decode_tile(const TcParams& P, int64_t bid) {
  const Geometry& g = P.g;
  TileDesc t;
  t.h = bid / P.tiles_per_head;
  const int64_t r_in = bid % P.tiles_per_head;
  const int64_t n_text_ct = P.text_tiles_per_head * P.text_chunks;
  t.text = r_in < n_text_ct;
  t.m_first = 0;
  t.part = 0;
  t.list = nullptr;
  if (t.text) {
    const int64_t tt = r_in / P.text_chunks, c = r_in % P.text_chunks;
    t.q_row0 = g.Tv + tt * 128;
    t.rows_valid = min((int64_t)128, g.Tt - tt * 128);
    t.m_first = c * P.chunk_blocks;
    t.count = min(g.M, t.m_first + P.chunk_blocks) - t.m_first;
    t.part = (t.h * P.text_tiles_per_head + tt) * P.text_chunks + c;
  } else {
    const int64_t tt = r_in - n_text_ct;
    t.q_row0 = tt * 128;
    t.rows_valid = min((int64_t)128, g.Tv - t.q_row0);
    if (g.B == 128) {   // one query block per tile: its own kv list (tile_lists skipped)
      t.count = P.ws.kv_count[t.h * g.N + tt];
      t.list = P.ws.kv_list + (t.h * g.N + tt) * g.M;
    } else {
      t.count = P.ws.tile_count[t.h * P.video_tiles_per_head + tt];
      t.list = P.ws.tile_list + (t.h * P.video_tiles_per_head + tt) * g.M;
    }
  }
  return t;
}

template <int D, int BKV>
__device__ __forceinline__ void producer_loop(const CUtensorMap& tm_q, const CUtensorMap& tm_k, const CUtensorMap& tm_v, const TcParams& P,
                                   int64_t n_tiles, uint8_t* kv_s, uint64_t* q_full, uint64_t* kv_full,
                                   uint64_t* kv_empty, uint64_t* s_full, uint64_t* p_full, uint64_t* pv_done,
                                   uint32_t tmem, int lane) {
  using C = Cfg<D, BKV>;
  const Geometry& g = P.g;
  (void)g; (void)q_full; (void)s_full; (void)p_full; (void)pv_done; (void)tmem; (void)tm_v;
  // ===================== TMA producer: every tile's [Q] K_0 K_1 V_0 K_2 V_1 ... =====================
  if (lane == 0) {
    if (P.qring) ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    const uint64_t keep = ptx::policy_evict_last();   // K/V blocks are re-read by many tiles of the head
    const uint64_t once = ptx::policy_evict_first();  // Q rows are read by one tile
    int s = 0;
    uint32_t ph = 0;
    for (int64_t bid = blockIdx.x; bid < n_tiles; bid += gridDim.x) {
      const TileDesc t = decode_tile(P, bid);
      if (P.qring) {
        // the tile's Q rows take one ring stage ahead of its K/V, so they are
        // in shared memory long before the softmax warps move them into TMEM
        ptx::mbar_wait(kv_empty + s, ph ^ 1);
        ptx::mbar_expect_tx(kv_full + s, C::STAGE);
        uint8_t* dst = kv_s + s * C::STAGE;
#pragma unroll
        for (int p = 0; p < C::PANELS; ++p)
          tma_rows(dst + p * C::Q_PANEL, &tm_q, kv_full + s, 64 * p, (int)t.q_row0, (int)t.h, g, once);
        if (++s == C::NST) { s = 0; ph ^= 1; }
      }
      auto load = [&](int64_t j, bool is_v) {
        const int64_t m = t.list ? (t.list[j] & 0xFFFFFF) : t.m_first + j;
        ptx::mbar_wait(kv_empty + s, ph ^ 1);
        ptx::mbar_expect_tx(kv_full + s, C::STAGE);
        uint8_t* dst = kv_s + s * C::STAGE;
#pragma unroll
        for (int p = 0; p < C::PANELS; ++p)
          tma_rows(dst + p * C::KV_PANEL, is_v ? &tm_v : &tm_k, kv_full + s, 64 * p, (int)kv_row0(g, m), t.h, g,
                   keep);
        if (++s == C::NST) { s = 0; ph ^= 1; }
      };
      for (int64_t j = 0; j <= t.count; ++j) {
        if (j < t.count) load(j, false);
        if (j >= 1) load(j - 1, true);
      }
    }
  }
}

template <int D, int BKV>
__device__ __forceinline__ void mma_loop(const CUtensorMap& tm_k, const CUtensorMap& tm_v, const TcParams& P,
                                   int64_t n_tiles, uint8_t* kv_s, uint64_t* q_full, uint64_t* kv_full,
                                   uint64_t* kv_empty, uint64_t* s_full, uint64_t* p_full, uint64_t* pv_done,
                                   uint32_t tmem, int lane) {
  using C = Cfg<D, BKV>;
  const Geometry& g = P.g;
  (void)g; (void)q_full; (void)s_full; (void)p_full; (void)pv_done; (void)tmem; (void)tm_v;
  // ===================== MMA issuer (whole warp; one elected lane issues) =====================
  const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0);
  const uint32_t kv_addr = __shfl_sync(0xffffffffu, ptx::smem_u32(kv_s), 0);
  int s_kv = 0;
  uint32_t ph_kv = 0;
  int64_t gs = 0;          // S/P steps issued by this CTA before the current tile
  uint32_t tile_par = 0;
  auto advance = [&]() {
    if (++s_kv == C::NST) { s_kv = 0; ph_kv ^= 1u; }
  };
  for (int64_t bid = blockIdx.x; bid < n_tiles; bid += gridDim.x) {
    const int64_t count = decode_tile(P, bid).count;
    ptx::mbar_wait(q_full, tile_par);   // this tile's Q rows are in TMEM
    tile_par ^= 1u;
    ptx::tc_fence_after();
    if (P.qring) {
      // every softmax thread has copied its Q row out of the ring stage: free it
      if (lane == 0) ptx::mbar_arrive(kv_empty + s_kv);
      __syncwarp();
      advance();
    }
    for (int64_t j = 0; j <= count; ++j) {
      if (j < count) {
        const int64_t gj = gs + j;
        ptx::mbar_wait(kv_full + s_kv, ph_kv);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tm + (uint32_t)((gj % C::NS) * BKV);
        const uint32_t kb = kv_addr + (uint32_t)(s_kv * C::STAGE);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint64_t b = ptx::sw128_desc(kb + (k / 4) * C::KV_PANEL + (k % 4) * 32, 16, 1024);
            ptx::mma_ts(d_tmem, tm + C::Q_COL + k * 8, b, C::IDESC_S, k > 0);
          }
          ptx::tc_commit(kv_empty + s_kv);
          ptx::tc_commit(s_full + (gj % C::NS));
        }
        __syncwarp();
        advance();
      }
      if (j >= 1) {
        const int64_t gj = gs + j - 1;
        ptx::mbar_wait(p_full + (gj % C::NS), (uint32_t)((gj / C::NS) & 1));
        ptx::mbar_wait(kv_full + s_kv, ph_kv);
        ptx::tc_fence_after();
        const uint32_t a_tmem = tm + (uint32_t)((gj % C::NS) * BKV);
        const uint32_t vb = kv_addr + (uint32_t)(s_kv * C::STAGE);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < BKV / 16; ++k) {
            const uint64_t b = ptx::sw128_desc(vb + k * 2048, C::KV_PANEL, 1024);
            ptx::mma_ts(tm + C::O_COL, a_tmem + k * 8, b, C::IDESC_O, (j > 1 || k > 0) ? 1u : 0u);
          }
          ptx::tc_commit(kv_empty + s_kv);
          ptx::tc_commit(pv_done);
        }
        __syncwarp();
        advance();
      }
    }
    // the epilogue waits for this (one phase per tile: a per-PV parity wait is
    // exact only one phase ahead, and PV_{count-2} can still be running there)
    if (ptx::elect_one()) ptx::tc_commit(pv_done + 1);
    __syncwarp();
    gs += count;
  }
}

template <int D, int BKV, int WPQ>
__global__ void __launch_bounds__(128 + 128 * WPQ, 1)
attn_tc_persistent_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                          const __grid_constant__ CUtensorMap tm_v, const TcParams P, int64_t n_tiles) {
  using C = Cfg<D, BKV>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* kv_s = base;
  uint64_t* bars = reinterpret_cast<uint64_t*>(kv_s + C::NST * C::STAGE);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + C::NST;
  uint64_t* s_full = kv_empty + C::NST;    // [NS]
  uint64_t* p_full = s_full + C::NS;       // [NS]
  uint64_t* pv_done = p_full + C::NS;      // [1]
  uint64_t* o_full = pv_done + 1;          // [1] a tile's last PV is complete (one phase per tile)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);
  float* red_max = reinterpret_cast<float*>(bars + 32);   // [2][WPQ][128] row maxima + [WPQ][128] row sums

  const Geometry& g = P.g;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    ptx::mbar_init(q_full, 128 * WPQ);
    for (int i = 0; i < C::NST; ++i) {
      ptx::mbar_init(kv_full + i, 1);
      ptx::mbar_init(kv_empty + i, 1);
    }
    for (int i = 0; i < C::NS; ++i) {
      ptx::mbar_init(s_full + i, 1);
      ptx::mbar_init(p_full + i, 128 * WPQ);
    }
    ptx::mbar_init(pv_done, 1);
    ptx::mbar_init(o_full, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    producer_loop<D, BKV>(tm_q, tm_k, tm_v, P, n_tiles, kv_s, q_full, kv_full, kv_empty, s_full, p_full, pv_done, tmem, lane);
  } else if (warp == 1) {
    mma_loop<D, BKV>(tm_k, tm_v, P, n_tiles, kv_s, q_full, kv_full, kv_empty, s_full, p_full, pv_done, tmem, lane);
  } else if (warp >= 4) {
    // ===================== softmax + epilogue =====================
    // WPQ softmax warps per TMEM lane quadrant, each owning BKV / WPQ score
    // columns and D / WPQ output columns of its quadrant's 32 rows
    constexpr int HC = BKV / WPQ;   // score columns per thread
    constexpr int HD = D / WPQ;     // output columns per thread
    constexpr int QW = D / 2 / WPQ; // 32-bit Q words per thread
    constexpr int NB = 32 * WPQ;    // threads of a quadrant's named barrier
    static_assert(HC % 32 == 0 && HD % 32 == 0 && (QW == 16 || QW == 32), "column split");
    const int sw = warp - 4;
    const int quad = sw & 3, half = sw >> 2;   // half: column part 0..WPQ-1
    const int row = quad * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const int sub = row / (int)g.B;          // which member query block of the tile
    const float sl2 = P.scale_log2;
    const uint64_t once = ptx::policy_evict_first();   // Q rows and outputs are touched once
    // Q row -> TMEM lanes (A operand of S = Q K^T): this thread packs half of
    // its row's d columns, bf16 pairs per 32-bit column
    int64_t ring_pos = 0;   // K/V ring stages consumed before the current tile (qring)
    auto store_q = [&](const TileDesc& t) {
      uint32_t qw[QW];
      if (P.qring) {
        // this thread's D / WPQ columns of its row from the tile's Q ring stage
        // (TMA 128B-swizzled panels of 64 columns: 16-byte chunk c of row r at
        // chunk slot c ^ (r % 8))
        const int st = (int)(ring_pos % C::NST);
        ptx::mbar_wait(kv_full + st, (uint32_t)((ring_pos / C::NST) & 1));
        const uint8_t* stage = kv_s + st * C::STAGE;
#pragma unroll
        for (int i = 0; i < QW / 4; ++i) {
          const int col16 = half * (QW / 4) + i;             // 16-byte chunk of the row (8 per panel)
          const uint8_t* pan = stage + (col16 / 8) * C::Q_PANEL + row * 128;
          const uint4 x = *reinterpret_cast<const uint4*>(pan + (((col16 % 8) ^ (row % 8)) * 16));
          qw[4 * i] = x.x; qw[4 * i + 1] = x.y; qw[4 * i + 2] = x.z; qw[4 * i + 3] = x.w;
        }
        ring_pos += 1 + 2 * t.count;
      } else {
        const int64_t grow = t.q_row0 + row;
        // permuted problem: gather the query row from its original position
        const int64_t srow = (P.perm && grow < g.Tv) ? P.perm[grow] : grow;
        const uint4* src = reinterpret_cast<const uint4*>(P.q + row_off(g, t.h, srow) + half * (D / WPQ));
#pragma unroll
        for (int i = 0; i < QW / 4; ++i) {
          const uint4 x = grow < g.T ? ptx::ld_stream(src + i, once) : make_uint4(0, 0, 0, 0);
          qw[4 * i] = x.x; qw[4 * i + 1] = x.y; qw[4 * i + 2] = x.z; qw[4 * i + 3] = x.w;
        }
      }
      if constexpr (QW == 32) {
        ptx::tmem_st32(lane_base + C::Q_COL + half * QW, qw);
      } else {
        ptx::tmem_st16(lane_base + C::Q_COL + half * QW, qw);
      }
      ptx::tmem_st_wait();
      ptx::tc_fence_before();
      ptx::mbar_arrive(q_full);
    };
    int64_t gs = 0;
    int64_t bid = blockIdx.x;
    TileDesc t;
    if (bid < n_tiles) {
      t = decode_tile(P, bid);
      store_q(t);
    }
    int tix = 0;
    for (; bid < n_tiles; bid += gridDim.x, ++tix) {
      const int64_t count = t.count;
      float m_run = -INFINITY, l_part = 0.f;
      for (int64_t j = 0; j < count; ++j) {
        const int64_t gj = gs + j;
        int64_t m;
        bool member;
        if (t.list) {
          const int32_t e = t.list[j];
          m = e & 0xFFFFFF;
          member = BKV == 128 || ((e >> (24 + sub)) & 1);   // plain kv-list entries at B = 128
        } else {
          m = t.m_first + j;
          member = true;
        }
        const int len = (int)kv_len(g, m);
        ptx::mbar_wait(s_full + (gj % C::NS), (uint32_t)((gj / C::NS) & 1));
        ptx::tc_fence_after();
        const uint32_t s_addr = lane_base + (uint32_t)((gj % C::NS) * BKV);
        uint32_t sr[HC / 32][32];
#pragma unroll
        for (int c = 0; c < HC / 32; ++c) ptx::tmem_ld32(s_addr + half * HC + c * 32, sr[c]);
        ptx::tmem_ld_wait();
        if (!member || len < BKV) {
#pragma unroll
          for (int c = 0; c < HC / 32; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (!member || half * HC + c * 32 + i >= len) sr[c][i] = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < HC / 32; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) mx4[i & 3] = fmaxf(mx4[i & 3], __uint_as_float(sr[c][i]));
        float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
        red_max[(gj & 1) * (WPQ * 128) + half * 128 + row] = mx;
        asm volatile("bar.sync %0, %1;" ::"r"(1 + quad), "r"(NB) : "memory");   // the quad's warps only
#pragma unroll
        for (int p2 = 0; p2 < WPQ; ++p2) mx = fmaxf(mx, red_max[(gj & 1) * (WPQ * 128) + p2 * 128 + row]);
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
        const float2 sc2 = make_float2(sl2, sl2), nb2 = make_float2(-base_m, -base_m);
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < HC / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = ptx::ffma2(make_float2(__uint_as_float(sr[c][2 * i]), __uint_as_float(sr[c][2 * i + 1])),
                                        sc2, nb2);
            const float2 p = make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
            sum2[i & 1] = ptx::fadd2(sum2[i & 1], p);
            pk[i] = ptx::pack_bf16(p.x, p.y);
          }
          ptx::tmem_st16(s_addr + half * (HC / 2) + c * 16, pk);
        }
        const float2 st2 = ptx::fadd2(sum2[0], sum2[1]);
        l_part = l_part * alpha + (st2.x + st2.y);
        // Every pv_done phase is observed here (the one before the next PV's
        // commit): the rescale below needs O = PV_0..PV_{j-1} of this tile, and
        // an mbarrier phase nobody waits on is a synchronisation hazard
        // (compute-sanitizer synccheck).  PV_{gj-1} ran right behind S_gj, so
        // after the exps above the wait is normally already satisfied.
        if (gj >= 1) ptx::mbar_wait(pv_done, (uint32_t)((gj - 1) & 1));
        if (__any_sync(0xffffffffu, rescale_o)) {
          // O must hold exactly PV_0..PV_{j-1} of this tile before it is rescaled
          ptx::tc_fence_after();
          const float a = rescale_o ? alpha : 1.f;
#pragma unroll
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            const uint32_t oa = lane_base + C::O_COL + half * HD + c * 32;
            ptx::tmem_ld32(oa, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
            ptx::tmem_st32(oa, o);
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full + (gj % C::NS));
      }
      // every S of this tile has been read: Q's TMEM columns are free, so the
      // next tile's Q goes in now and its S_0, S_1 overlap this epilogue
      const TileDesc cur = t;
      const int64_t nb = bid + gridDim.x;
      if (nb < n_tiles) {
        t = decode_tile(P, nb);
        store_q(t);
      }

      // ---- epilogue: O / l, rectification (rectify.py:66-89), bf16 store, LSE ----
      red_max[2 * WPQ * 128 + half * 128 + row] = l_part;
      asm volatile("bar.sync %0, %1;" ::"r"(1 + quad), "r"(NB) : "memory");   // the quad's warps only
      float l_run = 0.f;
#pragma unroll
      for (int p2 = 0; p2 < WPQ; ++p2) l_run += red_max[2 * WPQ * 128 + p2 * 128 + row];
      ptx::mbar_wait(o_full, (uint32_t)(tix & 1));   // every PV of this tile is complete
      ptx::tc_fence_after();
      const bool valid = row < cur.rows_valid;
      const int64_t grow = cur.q_row0 + row;
      if (cur.text) {
        // split-K text chunk: unnormalised O (fp32), row max (log2) and row sum
        float* po = P.text_part + (cur.part * 128 + row) * D;
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          const int col0 = half * HD + c * 32;
          ptx::tmem_ld32(lane_base + C::O_COL + col0, o);
          ptx::tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int v4 = 0; v4 < 8; ++v4)
              *reinterpret_cast<uint4*>(po + col0 + v4 * 4) =
                  make_uint4(o[v4 * 4], o[v4 * 4 + 1], o[v4 * 4 + 2], o[v4 * 4 + 3]);
          }
        }
        if (valid && half == 0) P.text_ml[cur.part * 128 + row] = make_float2(m_run, l_run);
      } else {
        float rfac = 1.f;
        const double* comp = nullptr;
        if (P.rectify && valid) {
          const int64_t n_blk = grow / g.B;
          rfac = P.ws.r_eff[cur.h * g.N + n_blk];
          comp = P.ws.comp + (cur.h * g.N + n_blk) * D;
        }
        const float inv_l = (count > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
        // permuted problem: scatter the row back to its original position
        const int64_t orig = (P.perm && valid) ? P.perm[grow] : grow;
        __nv_bfloat16* orow = P.out + out_off(g, cur.h, orig);
#pragma unroll
        for (int c = 0; c < HD / 32; ++c) {
          uint32_t o[32];
          const int col0 = half * HD + c * 32;
          ptx::tmem_ld32(lane_base + C::O_COL + col0, o);
          ptx::tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int v8 = 0; v8 < 4; ++v8) {
              uint32_t w[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int col = col0 + v8 * 8 + 2 * i;
                float y0 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * i]) * inv_l * rfac;
                float y1 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * i + 1]) * inv_l * rfac;
                if (comp) {
                  y0 += (float)comp[col];
                  y1 += (float)comp[col + 1];
                }
                w[i] = ptx::pack_bf16(y0, y1);
              }
              ptx::st_stream(orow + col0 + v8 * 8, make_uint4(w[0], w[1], w[2], w[3]), once);
            }
          }
        }
        if (valid && half == 0 && P.lse)
          P.lse[cur.h * g.T + orig] = l_run > 0.f ? (log2f(l_run) + m_run) * 0.69314718055994531f : -INFINITY;
      }
      // O is read: the next tile's PV_0 (after its P_0 below) may overwrite it
      ptx::tc_fence_before();
      gs += count;
    }
  }

  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::TMEM_COLS>(tmem);
  }
}

// Split-K text tiles: merge the chunks' (O_c, m_c, l_c) of every text query
// row into the final row, O = sum_c 2^(m_c - m*) O_c / sum_c 2^(m_c - m*) l_c
// (the online-softmax merge, kernel.py:120-145 semantics), plus the LSE.
template <int D>
__global__ void __launch_bounds__(256) text_combine_kernel(const float* __restrict__ part,
                                                           const float2* __restrict__ ml,
                                                           __nv_bfloat16* __restrict__ out, float* lse,
                                                           Geometry g, int64_t tiles, int64_t chunks) {
  const int64_t ht = blockIdx.x;                 // (head, text tile)
  const int64_t h = ht / tiles, t = ht % tiles;
  const int row = threadIdx.x / 2, half = threadIdx.x % 2;
  const int64_t trow = t * 128 + row;
  if (trow >= g.Tt) return;
  const int64_t base = ht * chunks;
  float mx = -INFINITY;
  for (int64_t c = 0; c < chunks; ++c) mx = fmaxf(mx, ml[(base + c) * 128 + row].x);
  float acc[D / 2];
#pragma unroll
  for (int i = 0; i < D / 2; ++i) acc[i] = 0.f;
  float l = 0.f;
  for (int64_t c = 0; c < chunks; ++c) {
    const float2 e = ml[(base + c) * 128 + row];
    const float w = e.x == -INFINITY ? 0.f : exp2f(e.x - mx);
    l += w * e.y;
    const float4* po = reinterpret_cast<const float4*>(part + ((base + c) * 128 + row) * D + half * (D / 2));
#pragma unroll
    for (int i = 0; i < D / 8; ++i) {
      const float4 x = po[i];
      acc[4 * i] += w * x.x; acc[4 * i + 1] += w * x.y; acc[4 * i + 2] += w * x.z; acc[4 * i + 3] += w * x.w;
    }
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
  __nv_bfloat16* orow = out + out_off(g, h, g.Tv + trow) + half * (D / 2);
#pragma unroll
  for (int i = 0; i < D / 16; ++i) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = ptx::pack_bf16(acc[8 * i + 2 * k] * inv, acc[8 * i + 2 * k + 1] * inv);
    *reinterpret_cast<uint4*>(orow + 8 * i) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  if (lse && half == 0) lse[h * g.T + g.Tv + trow] = l > 0.f ? (log2f(l) + mx) * 0.69314718055994531f : -INFINITY;
}


// ============================================================================
// Ping-pong kernel (d = B = 128): two query tiles per CTA in
// independent "slots", FA4-style.  Each slot has its own Q (shared memory, SS
// MMA for S), K/V ring, S/P and O TMEM columns (2 x (128 + 128) = 512), TMA
// producer warp, MMA warp and softmax warpgroup with one thread per row (no
// row-max exchange), so one slot's softmax overlaps the other slot's MMAs and
// the MUFU pipe is fed by whichever slot is in its ex2 phase; a slot's
// epilogue overlaps the other slot's steps.  d = B = 128 only.
// Warps: 0/1 TMA producers (slot 0/1), 2/3 MMA issuers, 4-7 / 8-11 softmax.
// ============================================================================
struct CfgPP {
  static constexpr int D = 128, BKV = 128;
  static constexpr int NST = 2;                   // K/V stages per slot
  static constexpr int STAGE = BKV * D * 2;       // 32 KB
  static constexpr int KV_PANEL = BKV * 128;      // 16 KB: 128 rows x 128 B
  static constexpr int Q_PANEL = 128 * 128;
  static constexpr int Q_BYTES = 128 * D * 2;     // 32 KB
  static constexpr int SLOT_SMEM = Q_BYTES + NST * STAGE;
  static constexpr int SMEM = 1024 + 2 * SLOT_SMEM + 512 + 2 * 2 * 128 * 4;   // + parked compensation rows
  static constexpr uint32_t IDESC_S64 = ptx::idesc_bf16(128, 64, false);   // S sub-steps: 64 keys
  static constexpr uint32_t IDESC_O = ptx::idesc_bf16(128, D, true);   // V MN-major
  static constexpr int THREADS = 384;
};

__global__ void __launch_bounds__(384, 1)
attn_tc_pp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                  const __grid_constant__ CUtensorMap tm_v, const TcParams P, int64_t n_tiles) {
  using C = CfgPP;
  constexpr int D = C::D, BKV = C::BKV;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + 2 * C::SLOT_SMEM);
  // per slot: q_full, q_empty, kv_full[2], kv_empty[2], s_full[2], pv_done, p_full[2], o_full  (12 barriers)
  auto slot_bar = [&](int s, int i) { return bars + s * 12 + i; };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  float* comp_s = reinterpret_cast<float*>(bars + 64);   // [slot][tile parity][D] compensation rows

  const Geometry& g = P.g;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(slot_bar(s, 0), 1);     // q_full (TMA)
      ptx::mbar_init(slot_bar(s, 1), 1);     // q_empty (MMA commit after a tile's last S)
      for (int i = 0; i < 2; ++i) {
        ptx::mbar_init(slot_bar(s, 2 + i), 1);   // kv_full
        ptx::mbar_init(slot_bar(s, 4 + i), 1);   // kv_empty
      }
      ptx::mbar_init(slot_bar(s, 6), 1);     // s_full[0]
      ptx::mbar_init(slot_bar(s, 7), 1);     // s_full[1]
      ptx::mbar_init(slot_bar(s, 8), 1);     // pv_done
      ptx::mbar_init(slot_bar(s, 9), 128);   // p_full[0]
      ptx::mbar_init(slot_bar(s, 10), 128);  // p_full[1]
      ptx::mbar_init(slot_bar(s, 11), 1);    // o_full: the tile's last PV is complete
    }
    ptx::fence_barrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // slot s walks tiles (blockIdx.x + k * gridDim.x) * 2 + s
  const int64_t stride = 2 * (int64_t)gridDim.x;

  if (warp < 2) {
    // ===================== TMA producer of slot `warp` =====================
    const int s = warp;
    if (lane == 0) {
      ptx::prefetch_tmap(&tm_q);
      ptx::prefetch_tmap(&tm_k);
      ptx::prefetch_tmap(&tm_v);
      const uint64_t keep = ptx::policy_evict_last();
      const uint64_t once = ptx::policy_evict_first();
      uint8_t* qs = base + s * C::SLOT_SMEM;
      uint8_t* ring = qs + C::Q_BYTES;
      int st = 0;
      uint32_t ph = 0, qph = 0;
      for (int64_t bid = 2 * (int64_t)blockIdx.x + s; bid < n_tiles; bid += stride) {
        const TileDesc t = decode_tile(P, bid);
        ptx::mbar_wait(slot_bar(s, 1), qph ^ 1);    // previous tile's S MMAs have read Q
        qph ^= 1;
        ptx::mbar_expect_tx(slot_bar(s, 0), C::Q_BYTES);
#pragma unroll
        for (int p = 0; p < 2; ++p)
          tma_rows(qs + p * C::Q_PANEL, &tm_q, slot_bar(s, 0), 64 * p, (int)t.q_row0, t.h, g,
                   once);   // Q rows are read by one tile: keep L2 for K/V
        for (int64_t j = 0; j < t.count; ++j) {
          const int64_t m = t.list ? (t.list[j] & 0xFFFFFF) : t.m_first + j;
#pragma unroll
          for (int kv = 0; kv < 2; ++kv) {
            ptx::mbar_wait(slot_bar(s, 4 + st), ph ^ 1);
            ptx::mbar_expect_tx(slot_bar(s, 2 + st), C::STAGE);
            uint8_t* dst = ring + st * C::STAGE;
#pragma unroll
            for (int p = 0; p < 2; ++p)
              tma_rows(dst + p * C::KV_PANEL, kv ? &tm_v : &tm_k, slot_bar(s, 2 + st), 64 * p, (int)kv_row0(g, m),
                       t.h, g, keep);
            if (++st == C::NST) { st = 0; ph ^= 1; }
          }
        }
      }
    }
  } else if (warp < 4) {
    // ===================== MMA issuer of slot `warp - 2` =====================
    // 64-key sub-steps i (two per kv block) into S buffers i % 2 ([0,64) and
    // [64,128) of the slot's S columns): S_{i+1} runs while the softmax works
    // on S_i; S_{i+2} reuses buffer i % 2 after PV_i (in-order tensor pipe).
    const int s = warp - 2;
    const uint32_t tm = __shfl_sync(0xffffffffu, tmem, 0) + (uint32_t)(s * 256);
    const uint32_t q_addr = __shfl_sync(0xffffffffu, ptx::smem_u32(base + s * C::SLOT_SMEM), 0);
    const uint32_t ring = q_addr + C::Q_BYTES;
    int st = 0;          // ring stage of the current kv block's K (V is the next stage)
    uint32_t ph = 0, qph = 0;
    int64_t gi = 0;      // sub-steps before the current tile
    for (int64_t bid = 2 * (int64_t)blockIdx.x + s; bid < n_tiles; bid += stride) {
      const int64_t count = decode_tile(P, bid).count;
      const int64_t nsub = 2 * count;
      ptx::mbar_wait(slot_bar(s, 0), qph);
      qph ^= 1;
      ptx::tc_fence_after();
      // ring bookkeeping: block j's K at stage kst(j), V at the next stage
      int k_st = st;
      uint32_t k_ph = ph;
      auto issue_s = [&](int64_t i) {       // S_i, i = 2 j + half
        const int64_t j = i >> 1;
        const int half = (int)(i & 1);
        int kst = k_st;
        uint32_t kph = k_ph;
        // K of block j: ring slot (st0 + 2 j) mod NST
        const int64_t slot = (int64_t)kst + 2 * j;
        const int sj = (int)(slot % C::NST);
        const uint32_t pj = kph ^ (uint32_t)((slot / C::NST) & 1);
        if (half == 0) ptx::mbar_wait(slot_bar(s, 2 + sj), pj);
        ptx::tc_fence_after();
        const uint32_t kb = ring + (uint32_t)(sj * C::STAGE) + (uint32_t)(half * 64 * 128);
        const uint32_t d_tmem = tm + (uint32_t)(half * 64);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = (uint32_t)((k / 4) * C::Q_PANEL + (k % 4) * 32);
            const uint64_t a = ptx::sw128_desc(q_addr + off, 16, 1024);
            const uint64_t b = ptx::sw128_desc(kb + (k / 4) * C::KV_PANEL + (k % 4) * 32, 16, 1024);
            ptx::mma_ss(d_tmem, a, b, C::IDESC_S64, k > 0);
          }
          if (half == 1) ptx::tc_commit(slot_bar(s, 4 + sj));   // K_j fully read
          ptx::tc_commit(slot_bar(s, 6 + half));                  // s_full[half]
          if (i == nsub - 1) ptx::tc_commit(slot_bar(s, 1));      // Q may be replaced after this
        }
        __syncwarp();
      };
      if (nsub > 0) issue_s(0);
      if (nsub > 1) issue_s(1);
      // a tile with an empty kv list (the C ABI's mask seam flags it as
      // RSA_ERR_EMPTY_ROW) issues no S MMA: release its Q buffer here, or the
      // producer would wait for it forever
      if (nsub == 0) {
        if (ptx::elect_one()) ptx::tc_commit(slot_bar(s, 1));
        __syncwarp();
      }
      for (int64_t i = 0; i < nsub; ++i) {
        const int64_t gsub = gi + i;
        const int64_t j = i >> 1;
        const int half = (int)(i & 1);
        // O += P_i V_i[64 half rows] once the softmax has written P_i
        ptx::mbar_wait(slot_bar(s, 9 + half), (uint32_t)((gsub >> 1) & 1));
        const int64_t slot = (int64_t)k_st + 2 * j + 1;
        const int sv = (int)(slot % C::NST);
        const uint32_t pv = k_ph ^ (uint32_t)((slot / C::NST) & 1);
        if (half == 0) ptx::mbar_wait(slot_bar(s, 2 + sv), pv);
        ptx::tc_fence_after();
        const uint32_t vb = ring + (uint32_t)(sv * C::STAGE) + (uint32_t)(half * 64 * 128);
        if (ptx::elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t b = ptx::sw128_desc(vb + k * 2048, C::KV_PANEL, 1024);
            ptx::mma_ts(tm + 128, tm + (uint32_t)(half * 64) + k * 8, b, C::IDESC_O, (i > 0 || k > 0) ? 1u : 0u);
          }
          if (half == 1) ptx::tc_commit(slot_bar(s, 4 + sv));   // V_j fully read
          ptx::tc_commit(slot_bar(s, 8));                         // pv_done
        }
        __syncwarp();
        if (i + 2 < nsub) issue_s(i + 2);
      }
      if (ptx::elect_one()) ptx::tc_commit(slot_bar(s, 11));   // one phase per tile, for the epilogue
      __syncwarp();
      // advance the ring past this tile's 2 * count stages
      const int64_t used = (int64_t)st + 2 * count;
      ph ^= (uint32_t)((used / C::NST) & 1);
      st = (int)(used % C::NST);
      gi += nsub;
    }
  } else {
    // ===================== softmax + epilogue of slot s, one thread per row =====================
    const int s = (warp - 4) >> 2;
    const int quad = warp & 3;
    const int row = quad * 32 + lane;
    const uint32_t lane_base = tmem + (uint32_t)(s * 256) + ((uint32_t)(quad * 32) << 16);
    const float sl2 = P.scale_log2;
    const uint64_t once = ptx::policy_evict_first();
    int64_t gi = 0;
    int64_t tix_s = 0;   // tiles of this slot so far (o_full phases)
    for (int64_t bid = 2 * (int64_t)blockIdx.x + s; bid < n_tiles; bid += stride) {
      const TileDesc t = decode_tile(P, bid);
      const int64_t count = t.count, nsub = 2 * count;
      float m_run = -INFINITY, l_run = 0.f;
      // this tile's compensation row and factor (one query block per tile at
      // B = 128): fetched now, parked in shared memory (double-buffered by tile
      // parity), read by the epilogue after the slot's barrier
      float rpre = 1.f;
      float* comp_park = comp_s + (s * 2 + (int)(tix_s & 1)) * D;
      if (P.rectify && !t.text) {
        const int64_t n_blk = t.q_row0 / g.B;
        comp_park[row] = (float)P.ws.comp[(t.h * g.N + n_blk) * D + row];
        rpre = P.ws.r_eff[t.h * g.N + n_blk];
      }
      // the kv list entry (for the ragged-block masks) is fetched one block ahead:
      // a global load per sub-step sat on the softmax critical path
      int32_t ent_next = (t.list && count > 0) ? t.list[0] : 0;
      int blen = 0;
      for (int64_t i = 0; i < nsub; ++i) {
        const int64_t gsub = gi + i;
        const int half = (int)(i & 1);
        if (half == 0) {
          const int64_t jb = i >> 1;
          const int64_t m = t.list ? (ent_next & 0xFFFFFF) : t.m_first + jb;
          if (t.list && jb + 1 < count) ent_next = t.list[jb + 1];
          blen = (int)kv_len(g, m);
        }
        const int len = blen - half * 64;
        ptx::mbar_wait(slot_bar(s, 6 + half), (uint32_t)((gsub >> 1) & 1));
        ptx::tc_fence_after();
        const uint32_t sbuf = lane_base + (uint32_t)(half * 64);
        uint32_t sr[2][32];
        ptx::tmem_ld32(sbuf, sr[0]);
        ptx::tmem_ld32(sbuf + 32, sr[1]);
        ptx::tmem_ld_wait();
        if (len < 64) {
#pragma unroll
          for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int q2 = 0; q2 < 32; ++q2)
              if (c * 32 + q2 >= len) sr[c][q2] = __float_as_uint(-INFINITY);
        }
        float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int q2 = 0; q2 < 32; ++q2) mx4[q2 & 3] = fmaxf(mx4[q2 & 3], __uint_as_float(sr[c][q2]));
        const float m_blk = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
        float alpha = 1.f;
        bool rescale_o = false;
        if (m_blk > m_run + kRescaleThreshold || (m_run == -INFINITY && m_blk > -INFINITY)) {
          alpha = (m_run == -INFINITY) ? 0.f : ptx::ex2(m_run - m_blk);
          rescale_o = (m_run != -INFINITY) && i > 0;
          m_run = m_blk;
        }
        const float base_m = (m_run == -INFINITY) ? 0.f : m_run;
        const float2 sc2 = make_float2(sl2, sl2), nb2 = make_float2(-base_m, -base_m);
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int q2 = 0; q2 < 16; ++q2) {
            const float2 x = ptx::ffma2(make_float2(__uint_as_float(sr[c][2 * q2]), __uint_as_float(sr[c][2 * q2 + 1])),
                                        sc2, nb2);
            const float2 p = make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
            sum2[q2 & 1] = ptx::fadd2(sum2[q2 & 1], p);
            pk[q2] = ptx::pack_bf16(p.x, p.y);
          }
          ptx::tmem_st16(sbuf + c * 16, pk);
        }
        const float2 st2 = ptx::fadd2(sum2[0], sum2[1]);
        l_run = l_run * alpha + (st2.x + st2.y);
        // every pv_done phase is observed (see the persistent kernel)
        if (gsub >= 1) ptx::mbar_wait(slot_bar(s, 8), (uint32_t)((gsub - 1) & 1));   // O = PV_..i-1
        if (__any_sync(0xffffffffu, rescale_o)) {
          ptx::tc_fence_after();
          const float a = rescale_o ? alpha : 1.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            const uint32_t oa = lane_base + 128 + c * 32;
            ptx::tmem_ld32(oa, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int q2 = 0; q2 < 32; ++q2) o[q2] = __float_as_uint(__uint_as_float(o[q2]) * a);
            ptx::tmem_st32(oa, o);
          }
        }
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(slot_bar(s, 9 + half));
      }
      // ---- epilogue (overlaps the other slot's steps) ----
      // every PV of this tile is complete (one o_full phase per tile: a per-PV
      // parity wait is exact only one phase ahead, and the last two PVs -- both
      // halves of the last block -- can still be in flight here)
      ptx::mbar_wait(slot_bar(s, 11), (uint32_t)(tix_s & 1));
      ptx::tc_fence_after();
      ++tix_s;
      asm volatile("bar.sync %0, 128;" ::"r"(1 + s) : "memory");   // the slot's parked compensation row
      const bool valid = row < t.rows_valid;
      const int64_t grow = t.q_row0 + row;
      if (t.text) {
        float* po = P.text_part + (t.part * 128 + row) * D;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          ptx::tmem_ld32(lane_base + 128 + c * 32, o);
          ptx::tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int v4 = 0; v4 < 8; ++v4)
              *reinterpret_cast<uint4*>(po + c * 32 + v4 * 4) =
                  make_uint4(o[v4 * 4], o[v4 * 4 + 1], o[v4 * 4 + 2], o[v4 * 4 + 3]);
          }
        }
        if (valid) P.text_ml[t.part * 128 + row] = make_float2(m_run, l_run);
      } else {
        const float rfac = (P.rectify && valid) ? rpre : 1.f;
        const float* comp = (P.rectify && valid) ? comp_park : nullptr;
        const float inv_l = (nsub > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
        // permuted problem: scatter the row back to its original position
        const int64_t orig = (P.perm && valid) ? P.perm[grow] : grow;
        __nv_bfloat16* orow = P.out + out_off(g, t.h, orig);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          ptx::tmem_ld32(lane_base + 128 + c * 32, o);
          ptx::tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int v8 = 0; v8 < 4; ++v8) {
              uint32_t w[4];
#pragma unroll
              for (int q2 = 0; q2 < 4; ++q2) {
                const int col = c * 32 + v8 * 8 + 2 * q2;
                float y0 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * q2]) * inv_l * rfac;
                float y1 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * q2 + 1]) * inv_l * rfac;
                if (comp) {
                  y0 += (float)comp[col];
                  y1 += (float)comp[col + 1];
                }
                w[q2] = ptx::pack_bf16(y0, y1);
              }
              ptx::st_stream(orow + c * 32 + v8 * 8, make_uint4(w[0], w[1], w[2], w[3]), once);
            }
          }
        }
        if (valid && P.lse)
          P.lse[t.h * g.T + orig] = l_run > 0.f ? (log2f(l_run) + m_run) * 0.69314718055994531f : -INFINITY;
      }
      ptx::tc_fence_before();
      gi += nsub;
    }
  }

  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

// ============================================================================
// Paired-tile kernel (d = B = 128, the default): two 128-row query tiles per
// CTA, each walking its own kv list, and ONE MMA-issuing thread interleaving
// them in the order  S0_j, PV1_{j-1}, S1_j, PV0_j  (FA4-style), so each tile's
// softmax runs while the tensor pipe executes the other tile's two MMA groups,
// and every S is a full 128-key MMA group (no 64-key sub-steps: half the
// barrier round trips per FLOP of the ping-pong kernel, and the SS operand
// traffic stays at the shared-memory rate).
//   TMEM   S0 | S1 | O0 | O1 (4 x 128 fp32 columns); P_t is written as bf16
//          pairs over the first 64 columns of S_t (the TS-MMA A operand).
//   smem   Q0, Q1 (32 KB each) + a 5-stage ring of 32 KB K / V blocks,
//          filled in exactly the MMA consumption order.
//   warps  0 TMA producer (K/V ring), 1 MMA issuer (+ TMEM owner), 2-3 K/V
//          readiness checkers of tiles 0/1 (warpgroup 0 runs on 80 registers), 4-7 softmax +
//          epilogue of tile 0, 8-11 of tile 1 (one thread per row, 208
//          registers: all 128 scores of a row stay in registers).  The
//          setmaxnreg budgets move registers inside the CTA's own pool
//          (384 x 168 at launch): 128 x (168 - 80) >= 256 x (208 - 168).
// Ordering facts the pipeline relies on (no extra barriers):
//   * the tensor pipe executes one thread's MMAs in issue order, so S_t_{j+1}
//     (issued after PV_t_j) cannot overwrite P_t_j before PV_t_j read it;
//   * tcgen05.commit tracks every earlier MMA of the issuing thread, so the
//     s_full[t] phase of block j implies PV_t_{j-1} is complete: the softmax
//     may rescale O_t right there;
//   * a softmax group finishes its epilogue (reads of O_t) before it releases
//     P_t of its next tile, and the next tile's first PV_t waits on that P_t.
// Q_t of a slot's next tile is TMA-loaded by the slot's own softmax group as
// soon as the last S_t of the current tile has completed (Q_t is then free).
// ============================================================================
// tools-only timeline of CTA 0 (-DRSA_PAIR_TRACE; tools/pair_trace.py): region 0 the
// MMA thread (per MMA group: clock before its waits, after the P wait, after
// the K/V wait), regions 1-2 row 0 of each softmax group (per block: before the
// S wait, after it, after the P release), region 3 the producer (per K/V load:
// clock before the ring-slot wait, at the TMA issue)
#ifdef RSA_PAIR_TRACE
__device__ long long g_pair_trace[4][16384];
#define PAIR_TRACE(region, idx, v) \
  do { if (blockIdx.x == 0 && (idx) < 16384) g_pair_trace[region][idx] = (v); } while (0)
#else
#define PAIR_TRACE(region, idx, v) do {} while (0)
#endif

struct CfgPair {
  static constexpr int D = 128, BKV = 128;
#ifndef RSA_PAIR_NST
#define RSA_PAIR_NST 5
#endif
  static constexpr int NST = RSA_PAIR_NST;         // K/V ring stages
  static constexpr int STAGE = BKV * D * 2;        // 32 KB
  static constexpr int PANEL = 128 * 128;          // 16 KB: 128 rows x 128 B (64 columns)
  static constexpr int Q_BYTES = 128 * D * 2;      // 32 KB
  static constexpr int HEAD = 256 + 2 * 128 * 4;   // barriers + tmem slot | parked compensation rows [2][128]
  static constexpr int SMEM = HEAD + 1024 + 2 * Q_BYTES + NST * STAGE;   // 231,680 <= 232,448
  static constexpr uint32_t IDESC_S = ptx::idesc_bf16(128, 128, false);
  static constexpr uint32_t IDESC_O = ptx::idesc_bf16(128, D, true);   // V MN-major
  static constexpr int THREADS = 384;
};
#ifndef RSA_PAIR_POLY
#define RSA_PAIR_POLY 0   // column pairs per 32-column chunk whose 2^x runs on the FMA pipe
#endif
#ifndef RSA_PAIR_SPIN
#define RSA_PAIR_SPIN 1   // poll (test_wait) instead of try_wait: 1 the MMA thread's P waits (A/B over four
                          // rounds: -1.9 % K3), 2 the softmax S waits (no gain)
#endif
#ifndef RSA_PAIR_KV_HINT
#define RSA_PAIR_KV_HINT 0   // A/B: 1 = K/V loads without the evict_last L2 hint; 2 = only K, 3 = only V evict_last
#endif
#ifndef RSA_TMEM_ZERO
#define RSA_TMEM_ZERO 1   // paired-tile kernel: TMEM base as the constant 0 (checked); 0 = read it (A/B)
#endif
#ifndef RSA_PAIR_FASTLOOP
#define RSA_PAIR_FASTLOOP 1   // steady-state MMA loop without first/last flags (0: one general loop, A/B)
#endif
#ifndef RSA_DESC_ADD
#define RSA_DESC_ADD 1   // MMA descriptors as base + offset (1) or rebuilt per MMA (0, A/B)
#endif
#ifndef RSA_PAIR_L2PF
#define RSA_PAIR_L2PF 0   // iterations ahead whose K/V blocks the producer prefetches into L2 (0: off)
#endif

__global__ void __launch_bounds__(384, 1)
attn_tc_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const TcParams P, int64_t n_tiles) {
  using C = CfgPair;
  constexpr int D = C::D;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* q_full = bars;            // [2] tx: the slot's Q tile landed
  uint64_t* s_full = bars + 2;        // [2] commit: S_t complete (and every earlier MMA)
  uint64_t* p_full = bars + 4;        // [2] 129 arrivals: P_t written (O_t rescaled if needed), V_t_j and
                                      //     K_t_{j+1} landed
  uint64_t* o_full = bars + 6;        // [2] commit: the tile's last PV_t complete
  uint64_t* kv_full = bars + 8;       // [NST]
  uint64_t* kv_empty = bars + 8 + C::NST;   // [NST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8 + 2 * C::NST);
  float* comp_s = reinterpret_cast<float*>(smem_raw + 256);   // [slot][128] this tile's compensation row
  uint8_t* data = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw + C::HEAD) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* q_s = data;                       // [2][Q_BYTES]
  uint8_t* ring = data + 2 * C::Q_BYTES;     // [NST][STAGE]

  const Geometry& g = P.g;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t n_pairs = (n_tiles + 1) / 2;
  if (threadIdx.x == 0) {
    for (int t = 0; t < 2; ++t) {
      ptx::mbar_init(q_full + t, 1);
      ptx::mbar_init(s_full + t, 1);
      ptx::mbar_init(p_full + t, 129);   // the group's 128 rows + the K/V readiness checker
      ptx::mbar_init(o_full + t, 1);
    }
    for (int i = 0; i < C::NST; ++i) {
      ptx::mbar_init(kv_full + i, 1);
      ptx::mbar_init(kv_empty + i, 1);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<512>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
#if RSA_TMEM_ZERO
  // A CTA's only allocation of all 512 columns starts at lane 0, column 0: the
  // TMEM base is the constant 0, so every tcgen05 address below is a
  // compile-time constant (no vector -> uniform register moves on the MMA
  // thread between groups).  Checked once.
  if (*tmem_slot != 0u) __trap();
  constexpr uint32_t tmem = 0u;
#else
  const uint32_t tmem = *tmem_slot;
#endif

  if (warp < 4) {
    ptx::regs_dec<80>();
    if (warp == 0 && lane == 0) {
    // ===================== TMA producer: K/V blocks in MMA order =====================
      ptx::prefetch_tmap(&tm_k);
      ptx::prefetch_tmap(&tm_v);
      const uint64_t normal = ptx::policy_evict_normal();
      (void)normal;
#if RSA_PAIR_KV_HINT == 1
      const uint64_t keep = ptx::policy_evict_normal();
#else
      const uint64_t keep = ptx::policy_evict_last();   // K/V blocks are re-read by many tiles of the head
#endif
      int st = 0;
      uint32_t ph = 0;
      int ptr = 0;   // trace index (RSA_PAIR_TRACE)
      (void)ptr;
      for (int64_t pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
        const int64_t b1 = 2 * pr + 1;
        const TileDesc t0 = decode_tile(P, 2 * pr);
        const TileDesc t1 = b1 < n_tiles ? decode_tile(P, b1) : TileDesc{};
        const int c0 = (int)t0.count;
        const int c1 = b1 < n_tiles ? (int)t1.count : 0;
        const int h0 = (int)t0.h, h1 = (int)t1.h, f0 = (int)t0.m_first, f1 = (int)t1.m_first;
        const int32_t* l0 = t0.list;
        const int32_t* l1 = t1.list;
        const int cmax = c0 > c1 ? c0 : c1;
        // kv-list entries are read one iteration ahead: a dependent global load
        // between the kv_empty wait and the TMA issue would sit on the ring's
        // refill path (it did: ~300-cycle S waits)
        auto kv_of = [&](const int32_t* lst, int f, int jj) { return lst ? (__ldg(lst + jj) & 0xFFFFFF) : f + jj; };
        int m0 = c0 > 0 ? kv_of(l0, f0, 0) : 0, m1 = c1 > 0 ? kv_of(l1, f1, 0) : 0, m1_prev = 0;
        int pf0 = 0, pf1 = 0;   // (RSA_PAIR_L2PF) kv blocks of iteration j + RSA_PAIR_L2PF
        if (RSA_PAIR_L2PF > 0) {
          pf0 = RSA_PAIR_L2PF < c0 ? kv_of(l0, f0, RSA_PAIR_L2PF) : 0;
          pf1 = RSA_PAIR_L2PF < c1 ? kv_of(l1, f1, RSA_PAIR_L2PF) : 0;
        }
        (void)pf0; (void)pf1;
        for (int j = 0; j <= cmax; ++j) {
          const int n0 = j + 1 < c0 ? kv_of(l0, f0, j + 1) : 0;
          const int n1 = j + 1 < c1 ? kv_of(l1, f1, j + 1) : 0;
          if (RSA_PAIR_L2PF > 0) {
            const int jp = j + RSA_PAIR_L2PF;
            const int q0 = jp + 1 < c0 ? kv_of(l0, f0, jp + 1) : 0;
            const int q1 = jp + 1 < c1 ? kv_of(l1, f1, jp + 1) : 0;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
              if (jp < c0) {
                ptx::tma_prefetch_4d(&tm_k, 64 * p, (int)kv_row0(g, pf0), h0 % (int)g.hb, h0 / (int)g.hb);
                ptx::tma_prefetch_4d(&tm_v, 64 * p, (int)kv_row0(g, pf0), h0 % (int)g.hb, h0 / (int)g.hb);
              }
              if (jp < c1) {
                ptx::tma_prefetch_4d(&tm_k, 64 * p, (int)kv_row0(g, pf1), h1 % (int)g.hb, h1 / (int)g.hb);
                ptx::tma_prefetch_4d(&tm_v, 64 * p, (int)kv_row0(g, pf1), h1 % (int)g.hb, h1 / (int)g.hb);
              }
            }
            pf0 = q0;
            pf1 = q1;
          }
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            // MMA order: K0_j, V1_{j-1}, K1_j, V0_j
            const int tt = (q4 == 0 || q4 == 3) ? 0 : 1;
            const int jj = q4 == 1 ? j - 1 : j;
            const int cc = tt ? c1 : c0;
            if (jj < 0 || jj >= cc) continue;
            const int m = q4 == 1 ? m1_prev : (tt ? m1 : m0);
            PAIR_TRACE(3, ptr, clock64());
            ptx::mbar_wait(kv_empty + st, ph ^ 1);
            PAIR_TRACE(3, ptr + 1, clock64());
            ptr += 2;
            ptx::mbar_expect_tx(kv_full + st, C::STAGE);
            uint8_t* dst = ring + st * C::STAGE;
            const CUtensorMap* tmap = (q4 & 1) ? &tm_v : &tm_k;
            const int row0 = (int)kv_row0(g, m), hh = tt ? h1 : h0;
#pragma unroll
            for (int p = 0; p < 2; ++p)
              tma_rows(dst + p * C::PANEL, tmap, kv_full + st, 64 * p, row0, hh, g,
                       RSA_PAIR_KV_HINT >= 2 ? ((q4 & 1) == (RSA_PAIR_KV_HINT - 2) ? keep : normal) : keep);
            if (++st == C::NST) { st = 0; ph ^= 1; }
          }
          m1_prev = m1;
          m0 = n0;
          m1 = n1;
        }
      }
    } else if (warp == 1) {
    // ===================== MMA issuer: S0_j, PV1_{j-1}, S1_j, PV0_j =====================
    // In steady state the only waits are the two p_full phases per iteration:
    // p_full[t] of block j also certifies (checker warp 2 + t) that V_t_j and
    // K_t_{j+1} have landed, so each wait releases a PV group and the next S
    // group of the same tile back to back.  A wait on an mbarrier costs the
    // issuing thread ~250 cycles behind its queued MMAs, during which the
    // tensor pipe ran dry with one wait per group.
    const uint32_t q_addr = ptx::smem_u32(q_s);
    const uint32_t ring_addr = ptx::smem_u32(ring);
    int st = 0;
    uint32_t ph = 0;
    uint32_t pbits = 0, qbits = 0;   // p_full / q_full parity per slot (bit t)
    int tr = 0;   // trace index (RSA_PAIR_TRACE)
    (void)tr;
    auto issue_s = [&](int t, bool first_of_tile) {
      PAIR_TRACE(0, tr, (clock64() << 2) | (t ? 2 : 0));
      PAIR_TRACE(0, tr + 1, 0);
      if (first_of_tile) {   // Q_t and K_t_0 are nobody else's to certify
        ptx::mbar_wait(q_full + t, (qbits >> t) & 1u);
        qbits ^= 1u << t;
        ptx::mbar_wait(kv_full + st, ph);
        ptx::tc_fence_after();
      }
      PAIR_TRACE(0, tr + 2, clock64());
      tr += 3;
      const uint32_t kb = ring_addr + (uint32_t)(st * C::STAGE);
      const uint32_t qb = q_addr + (uint32_t)(t * C::Q_BYTES);
      if (ptx::elect_one()) {
#if RSA_DESC_ADD
        // descriptors of the k-th K slice = base descriptor + (byte offset >> 4)
        // (shared addresses < 2^18: the 14-bit address field never carries)
        const uint64_t qd = ptx::sw128_desc(qb, 16, 1024), kd = ptx::sw128_desc(kb, 16, 1024);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint64_t off = (uint64_t)(((k / 4) * C::PANEL + (k % 4) * 32) >> 4);
          ptx::mma_ss(tmem + (uint32_t)(t * 128), qd + off, kd + off, C::IDESC_S, k > 0);
        }
#else
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (uint32_t)((k / 4) * C::PANEL + (k % 4) * 32);
          ptx::mma_ss(tmem + (uint32_t)(t * 128), ptx::sw128_desc(qb + off, 16, 1024),
                      ptx::sw128_desc(kb + off, 16, 1024), C::IDESC_S, k > 0);
        }
#endif
        ptx::tc_commit(kv_empty + st);   // K block read
        ptx::tc_commit(s_full + t);
      }
      __syncwarp();
      if (++st == C::NST) { st = 0; ph ^= 1u; }
    };
    auto issue_pv = [&](int t, bool first, bool last) {
      PAIR_TRACE(0, tr, (clock64() << 2) | (t ? 1 : 3));
#if RSA_PAIR_SPIN & 1
      ptx::mbar_spin(p_full + t, (pbits >> t) & 1u);
#else
      ptx::mbar_wait(p_full + t, (pbits >> t) & 1u);   // P_t_j written, V_t_j (and K_t_{j+1}) landed
#endif
      pbits ^= 1u << t;
      ptx::tc_fence_after();
      PAIR_TRACE(0, tr + 1, clock64());
      PAIR_TRACE(0, tr + 2, clock64());
      tr += 3;
      const uint32_t vb = ring_addr + (uint32_t)(st * C::STAGE);
      if (ptx::elect_one()) {
#if RSA_DESC_ADD
        const uint64_t vd = ptx::sw128_desc(vb, C::PANEL, 1024);
#pragma unroll
        for (int k = 0; k < 128 / 16; ++k)
          ptx::mma_ts(tmem + 256u + (uint32_t)(t * 128), tmem + (uint32_t)(t * 128) + k * 8,
                      vd + (uint64_t)(k * (2048 >> 4)), C::IDESC_O, (!first || k > 0) ? 1u : 0u);
#else
#pragma unroll
        for (int k = 0; k < 128 / 16; ++k)
          ptx::mma_ts(tmem + 256u + (uint32_t)(t * 128), tmem + (uint32_t)(t * 128) + k * 8,
                      ptx::sw128_desc(vb + k * 2048, C::PANEL, 1024), C::IDESC_O, (!first || k > 0) ? 1u : 0u);
#endif
        ptx::tc_commit(kv_empty + st);   // V block read
        if (last) ptx::tc_commit(o_full + t);
      }
      __syncwarp();
      if (++st == C::NST) { st = 0; ph ^= 1u; }
    };
    for (int64_t pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
      const int64_t b1 = 2 * pr + 1;
      const bool e1 = b1 < n_tiles;
      const int c0 = (int)decode_tile(P, 2 * pr).count;
      const int c1 = e1 ? (int)decode_tile(P, b1).count : 0;
      const int cmax = c0 > c1 ? c0 : c1;
      if (c0 > 0) issue_s(0, true);
      auto general = [&](int j) {
        if (j >= 1 && j <= c1) issue_pv(1, j == 1, j == c1);
        if (j < c1) issue_s(1, j == 0);
        if (j < c0) {
          issue_pv(0, j == 0, j == c0 - 1);
          if (j + 1 < c0) issue_s(0, false);
        }
      };
#if RSA_PAIR_FASTLOOP
      // steady state (2 <= j < min(c1, c0 - 1)): all four groups, no first /
      // last flags -- a straight-line body with compile-time arguments keeps the
      // MMA thread's work between groups short (it sits on both tiles' chains)
      const int fast_end = c1 < c0 - 1 ? c1 : c0 - 1;
      int j = 0;
      for (; j <= cmax && j < 2; ++j) general(j);
      for (; j < fast_end; ++j) {
        issue_pv(1, false, false);
        issue_s(1, false);
        issue_pv(0, false, false);
        issue_s(0, false);
      }
      for (; j <= cmax; ++j) general(j);
#else
      for (int j = 0; j <= cmax; ++j) general(j);
#endif
      // a tile with an empty kv list (the C ABI's mask seam flags it as
      // RSA_ERR_EMPTY_ROW): its group still loaded Q and releases one P phase
      // after its previous epilogue; answer with the o_full phase (so o_full
      // can never run a phase ahead of the group).  Its Q phase is skipped, not
      // waited for: the group may already have started the next tile's Q load
      // on the same barrier (a parity wait here would alias that phase).
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if ((t == 0 ? c0 : c1) == 0 && (t == 0 || e1)) {
          qbits ^= 1u << t;
          ptx::mbar_wait(p_full + t, (pbits >> t) & 1u);
          pbits ^= 1u << t;
          if (ptx::elect_one()) ptx::tc_commit(o_full + t);
          __syncwarp();
        }
      }
    }
    } else if (lane == 0) {
    // ===================== K/V readiness checker of slot t = warp - 2 =====================
    // Adds its own arrival to p_full[t] of block j once V_t_j and K_t_{j+1}
    // have landed (the ring position of every load is a function of the pair's
    // two counts), then waits for that phase so it never arrives a phase early.
    const int t = warp - 2;
    uint32_t base = 0, pph = 0;
    for (int64_t pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
      const int64_t b1 = 2 * pr + 1;
      const bool e1 = b1 < n_tiles;
      const int c0 = (int)decode_tile(P, 2 * pr).count;
      const int c1 = e1 ? (int)decode_tile(P, b1).count : 0;
      if (t == 0 || e1) {
        // items in iterations [0, j): K0, V1_{i-1}, K1, V0 per iteration i
        auto cnt = [&](int j) { return 2 * min(j, c0) + min(j, c1) + max(0, min(j - 1, c1)); };
        auto wait_item = [&](uint32_t pos) {
          ptx::mbar_wait(kv_full + (pos % C::NST), (pos / C::NST) & 1u);
        };
        const int ct = t ? c1 : c0;
        for (int j = 0; j < ct; ++j) {
          uint32_t pv, pk;
          if (t == 0) {
            pv = base + cnt(j) + 1 + (j >= 1 && j <= c1) + (j < c1);        // V0_j
            pk = base + cnt(j + 1);                                          // K0_{j+1}
          } else {
            pv = base + cnt(j + 1) + (j + 1 < c0);                           // V1_j
            pk = base + cnt(j + 1) + (j + 1 < c0) + (j + 1 <= c1);           // K1_{j+1}
          }
          wait_item(pv);
          if (j + 1 < ct) wait_item(pk);
          ptx::mbar_arrive(p_full + t);
          ptx::mbar_wait(p_full + t, pph);
          pph ^= 1u;
        }
        if (ct == 0) {   // the empty tile's single P phase
          ptx::mbar_arrive(p_full + t);
          ptx::mbar_wait(p_full + t, pph);
          pph ^= 1u;
        }
      }
      base += 2u * (uint32_t)(c0 + c1);
    }
    }
  } else {
    ptx::regs_inc<208>();
    // ===================== softmax + epilogue of slot t, one thread per row =====================
    const int t = (warp - 4) >> 2;
    const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    const int wtid = row;                      // 0..127 within the group
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t s_addr = lane_base + (uint32_t)(t * 128);
    const uint32_t o_addr = lane_base + 256u + (uint32_t)(t * 128);
    const float sl2 = P.scale_log2;
    const uint64_t once = ptx::policy_evict_first();
    float* comp_t = comp_s + t * 128;
    uint8_t* q_dst = q_s + t * C::Q_BYTES;
    auto load_q = [&](int64_t bid) {   // one thread of the group
      const TileDesc nt = decode_tile(P, bid);
      ptx::mbar_expect_tx(q_full + t, C::Q_BYTES);
#pragma unroll
      for (int p = 0; p < 2; ++p)
        tma_rows(q_dst + p * C::PANEL, &tm_q, q_full + t, 64 * p, (int)nt.q_row0, (int)nt.h, g, once);
    };
    const int64_t stride = 2 * (int64_t)gridDim.x;
    int64_t bid = 2 * (int64_t)blockIdx.x + t;
    if (wtid == 0 && bid < n_tiles) {
      ptx::prefetch_tmap(&tm_q);
      load_q(bid);
    }
    uint32_t ns = 0, no = 0, nq = 0;   // s_full / o_full / q_full phases seen by this group
    int tr = 0;   // trace index (RSA_PAIR_TRACE)
    (void)tr;
    for (; bid < n_tiles; bid += stride, ++nq) {
      const TileDesc T = decode_tile(P, bid);
      const int count = (int)T.count;
      const bool next = bid + stride < n_tiles;
      // park this tile's compensation row (the previous epilogue's readers are done)
      asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");
      float rpre = 1.f;
      if (P.rectify && !T.text) {
        const int64_t n_blk = T.q_row0 / g.B;
        comp_t[row] = (float)P.ws.comp[(T.h * g.N + n_blk) * D + row];
        rpre = P.ws.r_eff[T.h * g.N + n_blk];
      }
      const int32_t* list = T.list;
      const int m_first = (int)T.m_first;
      float m_run = -INFINITY, l_run = 0.f;
      int32_t ent_next = (list && count > 0) ? list[0] : 0;
      for (int j = 0; j < count; ++j) {
        const int m = list ? (ent_next & 0xFFFFFF) : m_first + j;
        if (list && j + 1 < count) ent_next = list[j + 1];
        const int len = (int)kv_len(g, m);
        if (wtid == 0) PAIR_TRACE(1 + t, tr, clock64());
#if RSA_PAIR_SPIN & 2
        ptx::mbar_spin(s_full + t, ns & 1u);
#else
        ptx::mbar_wait(s_full + t, ns & 1u);
#endif
        ++ns;
        ptx::tc_fence_after();
        if (wtid == 0) PAIR_TRACE(1 + t, tr + 1, clock64());
        // the tile's last S has read Q_t: bring in the next tile's Q now
        if (j == count - 1 && next && wtid == 0) load_q(bid + stride);
        uint32_t sr[4][32];
        float2 sum2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sc2 = make_float2(sl2, sl2);
        // P = 2^(s * scale - base) of 32 columns -> bf16 pairs in TMEM columns [16c, 16c + 16)
        auto exp_chunk = [&](int c, float2 nb2) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = ptx::ffma2(make_float2(__uint_as_float(sr[c][2 * i]), __uint_as_float(sr[c][2 * i + 1])),
                                        sc2, nb2);
            const float2 p = (i < RSA_PAIR_POLY) ? ptx::ex2_poly2(x) : make_float2(ptx::ex2(x.x), ptx::ex2(x.y));
            sum2[i & 1] = ptx::fadd2(sum2[i & 1], p);
            pk[i] = ptx::pack_bf16(p.x, p.y);
          }
          ptx::tmem_st16(s_addr + c * 16, pk);
        };
        auto max2 = [&](int c0_, float mx) {   // max over columns [32 c0_, 32 c0_ + 64)
          float a4[4] = {mx, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
          for (int c = c0_; c < c0_ + 2; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) a4[i & 3] = fmaxf(a4[i & 3], __uint_as_float(sr[c][i]));
          return fmaxf(fmaxf(a4[0], a4[1]), fmaxf(a4[2], a4[3]));
        };
        float alpha = 1.f;
        bool rescale_o = false;
        // TMEM -> registers runs at ~64 B/clk per SMSP (16 KB per block per
        // warp): only the first 32 columns are waited for before the exps start
        ptx::tmem_ld32(s_addr, sr[0]);
        ptx::tmem_ld_wait();
        if (wtid == 0) PAIR_TRACE(1 + t, tr + 2, clock64());
        if (len == 128 && __all_sync(0xffffffffu, m_run != -INFINITY)) {
          // Speculative: exponentiate against the running base m_run while the
          // second half of S is still loading, with no row max on the critical
          // path.  The base is kept while this block's P stays bounded: a row
          // sum <= 2^kSpecSumLog2 implies every P <= 2^kSpecSumLog2 (fine for
          // bf16 P and fp32 O / l).  Otherwise (rarely; warp-wide, because
          // tcgen05.st is warp-collective) the block is redone against its true
          // row max, as the max-first path would -- any base gives the same
          // softmax, the choice only moves rounding.
          ptx::tmem_ld32(s_addr + 32, sr[1]);
          ptx::tmem_ld32(s_addr + 64, sr[2]);
          ptx::tmem_ld32(s_addr + 96, sr[3]);
          const float2 nb2 = make_float2(-m_run, -m_run);
          if (wtid == 0) PAIR_TRACE(1 + t, tr + 3, clock64());
          exp_chunk(0, nb2);
          ptx::tmem_ld_wait();
          exp_chunk(1, nb2);
          exp_chunk(2, nb2);
          exp_chunk(3, nb2);
          const float2 ps = ptx::fadd2(sum2[0], sum2[1]);
          const bool redo = !(ps.x + ps.y <= kSpecSum);   // (NaN-safe)
          if (__any_sync(0xffffffffu, redo)) {
            if (redo) {
              const float m_blk = max2(2, max2(0, -INFINITY)) * sl2;
              alpha = ptx::ex2(m_run - m_blk);
              rescale_o = true;
              m_run = m_blk;
            }
            sum2[0] = sum2[1] = make_float2(0.f, 0.f);
            const float2 nb = make_float2(-m_run, -m_run);
            ptx::tmem_st_wait();   // the speculative P stores land before they are overwritten
#pragma unroll
            for (int c = 0; c < 4; ++c) exp_chunk(c, nb);
          }
        } else {
          // first block of the tile (or a ragged block): row max first
          ptx::tmem_ld32(s_addr + 32, sr[1]);
          ptx::tmem_ld32(s_addr + 64, sr[2]);
          ptx::tmem_ld32(s_addr + 96, sr[3]);
          ptx::tmem_ld_wait();
          if (len < 128) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (c * 32 + i >= len) sr[c][i] = __float_as_uint(-INFINITY);
          }
          const float m_blk = max2(2, max2(0, -INFINITY)) * sl2;
          if (m_blk > m_run + kRescaleThreshold || (m_run == -INFINITY && m_blk > -INFINITY)) {
            alpha = (m_run == -INFINITY) ? 0.f : ptx::ex2(m_run - m_blk);
            rescale_o = (m_run != -INFINITY) && j > 0;
            m_run = m_blk;
          }
          const float base_m = (m_run == -INFINITY) ? 0.f : m_run;
          const float2 nb2 = make_float2(-base_m, -base_m);
          if (wtid == 0) PAIR_TRACE(1 + t, tr + 3, clock64());
#pragma unroll
          for (int c = 0; c < 4; ++c) exp_chunk(c, nb2);
        }
        if (__any_sync(0xffffffffu, rescale_o)) {
          // O_t holds exactly PV_t_0 .. PV_t_{j-1} (this s_full phase implies
          // it) and PV_t_j waits for the P release below
          const float a = rescale_o ? alpha : 1.f;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            ptx::tmem_ld32(o_addr + c * 32, o);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * a);
            ptx::tmem_st32(o_addr + c * 32, o);
          }
        }
        if (wtid == 0) PAIR_TRACE(1 + t, tr + 4, clock64());
        ptx::tmem_st_wait();
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full + t);
        if (wtid == 0) PAIR_TRACE(1 + t, tr + 5, clock64());
        tr += 6;
        const float2 st2 = ptx::fadd2(sum2[0], sum2[1]);
        l_run = l_run * alpha + (st2.x + st2.y);
      }
      if (count == 0) {
        // empty kv list: no S read Q_t; once its load has landed the next Q
        // can go in.  One P phase tells the MMA warp this group is past its
        // previous epilogue.
        if (next && wtid == 0) {
          ptx::mbar_wait(q_full + t, nq & 1u);
          load_q(bid + stride);
        }
        ptx::tc_fence_before();
        ptx::mbar_arrive(p_full + t);
      }
      // ---- epilogue: O / l, rectification (rectify.py:66-89), bf16 store, LSE ----
      ptx::mbar_wait(o_full + t, no & 1u);
      ++no;
      ptx::tc_fence_after();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + t) : "memory");   // the parked compensation row
      const bool valid = row < T.rows_valid;
      const int64_t grow = T.q_row0 + row;
      if (T.text) {
        float* po = P.text_part + (T.part * 128 + row) * D;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          ptx::tmem_ld32(o_addr + c * 32, o);
          ptx::tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int v4 = 0; v4 < 8; ++v4)
              *reinterpret_cast<uint4*>(po + c * 32 + v4 * 4) =
                  make_uint4(o[v4 * 4], o[v4 * 4 + 1], o[v4 * 4 + 2], o[v4 * 4 + 3]);
          }
        }
        if (valid) P.text_ml[T.part * 128 + row] = make_float2(m_run, l_run);
      } else {
        const float rfac = (P.rectify && valid) ? rpre : 1.f;
        const bool comp = P.rectify && valid;
        const float inv_l = (count > 0 && l_run > 0.f) ? 1.f / l_run : 0.f;
        const int64_t orig = (P.perm && valid) ? P.perm[grow] : grow;
        __nv_bfloat16* orow = P.out + out_off(g, T.h, orig);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t o[32];
          ptx::tmem_ld32(o_addr + c * 32, o);
          ptx::tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int v8 = 0; v8 < 4; ++v8) {
              uint32_t w[4];
#pragma unroll
              for (int q2 = 0; q2 < 4; ++q2) {
                const int col = c * 32 + v8 * 8 + 2 * q2;
                float y0 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * q2]) * inv_l * rfac;
                float y1 = inv_l == 0.f ? 0.f : __uint_as_float(o[v8 * 8 + 2 * q2 + 1]) * inv_l * rfac;
                if (comp) {
                  y0 += comp_t[col];
                  y1 += comp_t[col + 1];
                }
                w[q2] = ptx::pack_bf16(y0, y1);
              }
              ptx::st_stream(orow + c * 32 + v8 * 8, make_uint4(w[0], w[1], w[2], w[3]), once);
            }
          }
        }
        if (valid && P.lse)
          P.lse[T.h * g.T + orig] = l_run > 0.f ? (log2f(l_run) + m_run) * 0.69314718055994531f : -INFINITY;
      }
      // the O_t reads above complete before this group's next P_t release
      ptx::tc_fence_before();
    }
  }

  __syncwarp();
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<512>(tmem);
  }
}

cudaError_t launch_pair(const Geometry& g, const void* q, const void* k, const void* v, void* out, float* lse,
                        const Workspace& ws, bool rectify, bool text, cudaStream_t st, const int32_t* perm) {
  using C = CfgPair;
  CUtensorMap tq, tk, tv;
  if (!make_rows_tmap(&tq, q, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_rows_tmap(&tk, k, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_rows_tmap(&tv, v, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  TcParams P{};
  P.g = g;
  P.ws = ws;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.q = static_cast<const __nv_bfloat16*>(q);
  P.lse = lse;
  P.perm = perm;   // (q is then the permuted copy; outputs are scattered back)
  P.rectify = rectify ? 1 : 0;
  P.text_tiles_per_head = text ? (g.Tt + 127) / 128 : 0;
  P.text_chunks = text_chunks(g);
  P.chunk_blocks = (g.M + P.text_chunks - 1) / P.text_chunks;
  P.video_tiles_per_head = (g.N * g.B + 127) / 128;
  P.tiles_per_head = P.text_tiles_per_head * P.text_chunks + P.video_tiles_per_head;
  P.text_part = ws.text_part;
  P.text_ml = reinterpret_cast<float2*>(ws.text_ml);
  P.scale_log2 = (float)(1.4426950408889634 / sqrt((double)g.d));
  cudaError_t e = cudaFuncSetAttribute(attn_tc_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_tiles = g.H * P.tiles_per_head;
  attn_tc_pair_kernel<<<(unsigned)std::min<int64_t>((n_tiles + 1) / 2, sms), C::THREADS, C::SMEM, st>>>(
      tq, tk, tv, P, n_tiles);
  e = cudaGetLastError();
  if (e != cudaSuccess || P.text_tiles_per_head == 0) return e;
  text_combine_kernel<128><<<(unsigned)(g.H * P.text_tiles_per_head), 256, 0, st>>>(
      P.text_part, P.text_ml, P.out, lse, g, P.text_tiles_per_head, P.text_chunks);
  return cudaGetLastError();
}

cudaError_t launch_pp(const Geometry& g, const void* q, const void* k, const void* v, void* out, float* lse,
                      const Workspace& ws, bool rectify, bool text, cudaStream_t st, const int32_t* perm) {
  using C = CfgPP;
  CUtensorMap tq, tk, tv;
  if (!make_rows_tmap(&tq, q, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_rows_tmap(&tk, k, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_rows_tmap(&tv, v, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  TcParams P{};
  P.g = g;
  P.ws = ws;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.q = static_cast<const __nv_bfloat16*>(q);
  P.lse = lse;
  P.perm = perm;   // (q is then the permuted copy; outputs are scattered back)
  P.rectify = rectify ? 1 : 0;
  P.text_tiles_per_head = text ? (g.Tt + 127) / 128 : 0;
  P.text_chunks = text_chunks(g);
  P.chunk_blocks = (g.M + P.text_chunks - 1) / P.text_chunks;
  P.video_tiles_per_head = (g.N * g.B + 127) / 128;
  P.tiles_per_head = P.text_tiles_per_head * P.text_chunks + P.video_tiles_per_head;
  P.text_part = ws.text_part;
  P.text_ml = reinterpret_cast<float2*>(ws.text_ml);
  P.scale_log2 = (float)(1.4426950408889634 / sqrt((double)g.d));
  cudaError_t e = cudaFuncSetAttribute(attn_tc_pp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_tiles = g.H * P.tiles_per_head;
  attn_tc_pp_kernel<<<(unsigned)std::min<int64_t>((n_tiles + 1) / 2, sms), C::THREADS, C::SMEM, st>>>(tq, tk, tv, P,
                                                                                                        n_tiles);
  e = cudaGetLastError();
  if (e != cudaSuccess || P.text_tiles_per_head == 0) return e;
  text_combine_kernel<128><<<(unsigned)(g.H * P.text_tiles_per_head), 256, 0, st>>>(
      P.text_part, P.text_ml, P.out, lse, g, P.text_tiles_per_head, P.text_chunks);
  return cudaGetLastError();
}

template <int D, int BKV, int WPQ>
cudaError_t launch_persistent(const Geometry& g, const void* q, const void* k, const void* v, void* out,
                              float* lse, const Workspace& ws, bool rectify, bool text, cudaStream_t st,
                              const int32_t* perm) {
  using C = Cfg<D, BKV>;
  CUtensorMap tq, tk, tv;
  if (!make_rows_tmap(&tq, q, g, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_rows_tmap(&tk, k, g, 64, BKV, CU_TENSOR_MAP_SWIZZLE_128B) ||
      !make_rows_tmap(&tv, v, g, 64, BKV, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  TcParams P{};
  // Q through the ring when a Q tile is exactly one stage (BKV = 128) and rows
  // are not gathered through a permutation
  P.qring = (C::STAGE == C::Q_BYTES && perm == nullptr) ? 1 : 0;
  P.g = g;
  P.ws = ws;
  P.out = static_cast<__nv_bfloat16*>(out);
  P.q = static_cast<const __nv_bfloat16*>(q);
  P.lse = lse;
  P.perm = perm;
  P.rectify = rectify ? 1 : 0;
  P.text_tiles_per_head = text ? (g.Tt + 127) / 128 : 0;
  P.text_chunks = text_chunks(g);
  P.chunk_blocks = (g.M + P.text_chunks - 1) / P.text_chunks;
  P.video_tiles_per_head = (g.N * g.B + 127) / 128;
  P.tiles_per_head = P.text_tiles_per_head * P.text_chunks + P.video_tiles_per_head;
  P.text_part = ws.text_part;
  P.text_ml = reinterpret_cast<float2*>(ws.text_ml);
  P.scale_log2 = (float)(1.4426950408889634 / sqrt((double)g.d));
  auto kern = attn_tc_persistent_kernel<D, BKV, WPQ>;
  const int smem = C::SMEM - 768 * 4 + 3 * WPQ * 128 * 4;   // row-max / row-sum exchange area
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_tiles = g.H * P.tiles_per_head;
  kern<<<(unsigned)std::min<int64_t>(n_tiles, sms), 128 + 128 * WPQ, smem, st>>>(tq, tk, tv, P, n_tiles);
  e = cudaGetLastError();
  if (e != cudaSuccess || P.text_tiles_per_head == 0) return e;
  text_combine_kernel<D><<<(unsigned)(g.H * P.text_tiles_per_head), 256, 0, st>>>(
      P.text_part, P.text_ml, P.out, lse, g, P.text_tiles_per_head, P.text_chunks);
  return cudaGetLastError();
}


}  // namespace

#ifdef RSA_PAIR_TRACE
extern "C" int rsa_debug_pair_trace(long long* dst, int n) {
  return (int)cudaMemcpyFromSymbol(dst, g_pair_trace, sizeof(long long) * (size_t)std::min(n, 4 * 16384));
}
#endif

bool tc_supported(const Geometry& g) {
  return g.dtype == RSA_BF16 && (g.d == 64 || g.d == 128) && (g.B == 64 || g.B == 128) &&
         g.T * g.d < (int64_t(1) << 31) && g.H < 65536 && tmap_encode_fn() != nullptr;
}

cudaError_t launch_attn_tc(const Geometry& g, const void* q, const void* k, const void* v, void* out, float* lse,
                           const Workspace& ws, bool rectify, bool text, cudaStream_t st, int* launches,
                           const int32_t* perm, const void* q_perm, int kernel) {
  *launches += 1 + (text && g.Tt > 0 ? 1 : 0);   // attention (+ text combine)
  // d = B = 128: the ping-pong kernel (the permuted problem runs on it with the
  // permuted Q copy K1 wrote); RSA_KERNEL_TCGEN05_PERSISTENT asks for the
  // one-tile persistent kernel instead (cross-checks)
  if (g.d == 128 && g.B == 128 && kernel != RSA_KERNEL_TCGEN05_PERSISTENT && (!perm || q_perm)) {
    if (kernel == RSA_KERNEL_TCGEN05_PINGPONG)
      return launch_pp(g, perm ? q_perm : q, k, v, out, lse, ws, rectify, text, st, perm);
    return launch_pair(g, perm ? q_perm : q, k, v, out, lse, ws, rectify, text, st, perm);
  }
#define RSA_TC_P(DD, BB) \
  if (g.d == DD && g.B == BB) return launch_persistent<DD, BB, 2>(g, q, k, v, out, lse, ws, rectify, text, st, perm);
  RSA_TC_P(128, 128)
  RSA_TC_P(128, 64)
  RSA_TC_P(64, 128)
  RSA_TC_P(64, 64)
#undef RSA_TC_P
  return cudaErrorInvalidValue;
}

}  // namespace rsa
