// K1: exactly rounded fp64 block pooling (HBM-bound streaming reduction).
//
// Reference: block_pool / block_sums (pkg/src/rectattn/core.py:154-189) use
// math.fsum per column, pool_problem (core.py:192-201) pools Q video blocks,
// K video blocks and all V blocks; _pool_rows (masks.py:130-135) pools the
// text keys per (possibly ragged) text block; pooling_error (masks.py:165-171)
// needs the deficits sum - len * mean.
//
// Two kernels.  bf16 (the model path): pool_bulk_kernel below, TMA-streamed.
// f32 / f64 (the reference's own precisions) and unaligned bf16: pool_kernel,
// one CTA per (block, segment, head); 256 threads stream the block's rows with
// 128-bit non-allocating loads, each thread owning a column chunk and a row
// phase.  For bf16/f32 data the sums are plain fp64 adds, proven exact per
// block from its magnitude range (see pass 1 below); otherwise (f64 data, or a
// block spanning too many binades) each column is summed by Shewchuk's
// algorithm (fsum_exact).  Either way the result is the exactly rounded sum,
// bit-identical to math.fsum, and independent of launch geometry.
#include "rsa_internal.cuh"
#include "tc_ptx.cuh"
#include "tmap.cuh"

#include <cfloat>

#include <algorithm>

namespace rsa {
namespace {

constexpr int kThreads = 256;

// Shewchuk's exactly rounded sum (CPython math.fsum, including its half-even
// correction) of n finite doubles at(0..n-1).
template <typename F>
__device__ double fsum_exact(int64_t n, F at) {
  double p[48];   // non-overlapping partials, increasing magnitude (<= 40 for doubles)
  int np = 0;
  for (int64_t i = 0; i < n; ++i) {
    double x = at(i);
    int j = 0;
    for (int k = 0; k < np; ++k) {
      double y = p[k];
      if (fabs(x) < fabs(y)) { const double t = x; x = y; y = t; }
      const double hi = __dadd_rn(x, y);
      const double lo = __dsub_rn(y, __dsub_rn(hi, x));
      if (lo != 0.0) p[j++] = lo;
      x = hi;
    }
    p[j] = x;
    np = j + 1;
  }
  if (np == 0) return 0.0;
  int n2 = np;
  double hi = p[--n2], lo = 0.0;
  while (n2 > 0) {
    const double x = hi, y = p[--n2];
    hi = __dadd_rn(x, y);
    const double yr = __dsub_rn(hi, x);
    lo = __dsub_rn(y, yr);
    if (lo != 0.0) break;
  }
  if (n2 > 0 && ((lo < 0.0 && p[n2 - 1] < 0.0) || (lo > 0.0 && p[n2 - 1] > 0.0))) {
    const double y = __dmul_rn(lo, 2.0), x = __dadd_rn(hi, y);
    if (y == __dsub_rn(x, hi)) hi = x;
  }
  return hi;
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
  const int64_t row0 = kv_row0(g, blk);  // text blocks follow the video blocks contiguously
  const int64_t len = kv_len(g, blk);
  const T* src = (seg == 0 ? q : seg == 1 ? k : v) + (h * g.T + row0) * d;

  __shared__ double s_hi[2048];

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
  bool nonfinite = false;
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
            nonfinite |= !(ax <= FLT_MAX);
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
          nonfinite |= !(ax <= FLT_MAX);
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
  if (!exact && rg < rg_count) {
    // (the column sums come from fsum_exact below; this pass flags non-finite
    // values and, for f64 data, copies the raw text keys)
    for (int64_t r = rg; r < len; r += rg_count) {
      double x[VEC];
      load_vec<T, VEC>(src + r * d + c * VEC, x);
#pragma unroll
      for (int i = 0; i < VEC; ++i) nonfinite |= !(fabs(x[i]) <= DBL_MAX);
      if (raw_out && !kTryPlain) {
#pragma unroll
        for (int i = 0; i < VEC; ++i) raw_out[r * d + c * VEC + i] = x[i];
      }
    }
  }
  if (nonfinite) atomicOr(ws.status + ST_NONFINITE, 1);
  __syncthreads();

  for (int64_t col = t; col < d; col += kThreads) {
    const int64_t slot = (col % VEC) * tpr + col / VEC;
    double sum;
    if (exact) {
      sum = 0.0;   // exact partial sums: plain adds stay exact (same bound)
      for (int p = 0; p < rg_count; ++p) sum += s_hi[p * d + slot];
    } else {
      // correctly rounded (math.fsum) column sum, one thread per column
      sum = fsum_exact(len, [&](int64_t r) { return to_f64(src[r * d + col]); });
    }
    const double flen = (double)len;
    const double mean = sum / flen;           // core.py:172 fsum(...) / length
    // numpy rounds the product first (no FMA contraction): masks.py:166 / masks.py:171
    const double deficit = __dsub_rn(sum, __dmul_rn(flen, mean));
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

// ---------------------------------------------------------------------------
// bf16 path: persistent CTAs (2 per SM) walk the pooling items -- one
// (head, segment, block) = B rows x d bf16 -- and stream each into a
// shared-memory ring with ONE TMA tensor load (a [d x B] box of the 4-D row
// map, so any row strides work), STAGES items in flight per CTA.  Per item:
//  phase A (all threads; 8 columns x B/RP rows each, 16-byte shared loads):
//    every bf16 x is re-encoded EXACTLY as the fp64 value x * 2^-896 with two
//    or three integer ops -- its f32 bit pattern shifted right by 3 with the
//    sign kept: the 8-bit exponent lands in the low bits of the f64 exponent,
//    the 7 significand bits at the top of the f64 significand; 0 -> +-0,
//    subnormals -> f64 subnormals, one scale for all -- instead of a
//    bf16->f64 conversion per element on the XU pipe (what bound round 1's
//    kernel); fp64 adds; packed 16x2 integer max / min of the |x| bit
//    patterns (3-input DPX min/max).  Lanes sharing columns merge by shuffle;
//    one barrier.
//  decision (every thread): the plain sums are exact iff
//    e_max - e_min + 8 + ceil(log2 len) < 53 (e_min over nonzero values: a
//    thread that saw an exact zero recomputes its minimum without zeros);
//  phase B (d threads): the column's 8 warp partials, unscaled by 2^896
//    (exact), mean / deficit.  A block failing the test (never for sane data)
//    is re-summed per column with Shewchuk's algorithm -- the algorithm of
//    math.fsum, correctly rounded -- from the same shared-memory copy.
// Result: bit-identical to the reference's math.fsum pooling (core.py:154-189).
// ---------------------------------------------------------------------------
constexpr int kBulkThreads = 256;

// f32 bit pattern of a bf16 value (low 16 bits zero) -> the fp64 x * 2^-896, exactly
__device__ __forceinline__ double bf16_scaled(uint32_t f32_bits) {
  return __hiloint2double((int)(((int)f32_bits >> 3) & 0x8FFFE000), 0);
}
__device__ __forceinline__ double unscale_896(double x) {
  return __dmul_rn(x, __hiloint2double(0x77F00000, 0));   // * 2^896
}

struct PoolItem {
  int64_t h, blk;
  int seg;
};

// items: per head [N Q video blocks][M K blocks][M V blocks]
__device__ __forceinline__ PoolItem pool_item(const Geometry& g, int64_t i) {
  const int64_t per_head = g.N + 2 * g.M;
  PoolItem it;
  it.h = i / per_head;
  int64_t r = i % per_head;
  if (r < g.N) { it.seg = 0; it.blk = r; }
  else if (r < g.N + g.M) { it.seg = 1; it.blk = r - g.N; }
  else { it.seg = 2; it.blk = r - g.N - g.M; }
  return it;
}

template <int D, int STAGES>
__global__ void __launch_bounds__(kBulkThreads, 2)
pool_bulk_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const __nv_bfloat16* __restrict__ q,
                 const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, Workspace ws,
                 Geometry g, int64_t n_items, const int32_t* __restrict__ perm, __nv_bfloat16* kp,
                 __nv_bfloat16* vp, __nv_bfloat16* qp) {
  constexpr int TPR = D / 8;                   // threads per row: 16 bytes (8 bf16) each
  constexpr int RP = kBulkThreads / TPR;       // row phases
  constexpr int WARPS = kBulkThreads / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = (int)(g.B * D * 2);
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  double* s_part = reinterpret_cast<double*>(full + STAGES);        // [2][WARPS][D]
  uint32_t* s_rng = reinterpret_cast<uint32_t*>(s_part + 2 * WARPS * D);   // [2][WARPS][2]

  const int t = threadIdx.x, lane = t % 32, warp = t / 32;
  const int tc = t % TPR, rp = t / TPR;
  if (t == 0) {
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    for (int st = 0; st < STAGES; ++st) ptx::mbar_init(full + st, 1);
    ptx::fence_barrier_init();
  }
  __syncthreads();
  // item i -> ring stage st (thread 0): one TMA box of B rows (rows past the
  // block -- the next block, or zero fill past T -- are ignored)
  auto fetch = [&](int64_t i, int st) {
    const PoolItem it = pool_item(g, i);
    ptx::mbar_expect_tx(full + st, (uint32_t)stage_bytes);
    ptx::tma_load_4d(ring + st * stage_bytes, it.seg == 0 ? &tm_q : it.seg == 1 ? &tm_k : &tm_v, full + st, 0,
                     (int)kv_row0(g, it.blk), (int)(it.h % g.hb), (int)(it.h / g.hb));
  };
  // permuted (Morton) problem: every thread gathers 16-byte pieces of the
  // block's rows (cp.async groups)
  constexpr int CPR = D * 2 / 16;
  auto fetch_rows = [&](int64_t i, int st) {
    const PoolItem it = pool_item(g, i);
    const int64_t len = kv_len(g, it.blk);
    const __nv_bfloat16* base = it.seg == 0 ? q : it.seg == 1 ? k : v;
    uint8_t* dst = ring + st * stage_bytes;
    for (int64_t c = t; c < len * CPR; c += kBulkThreads) {
      const int64_t r = c / CPR, cc = c % CPR;
      const int64_t row = it.blk < g.N ? perm[it.blk * g.B + r] : kv_row0(g, it.blk) + r;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst + r * D * 2 + cc * 16)),
                   "l"(base + row_off(g, it.h, row) + cc * 8)
                   : "memory");
    }
  };
  if (perm) {
    for (int st = 0; st < STAGES; ++st) {
      const int64_t i = blockIdx.x + (int64_t)st * gridDim.x;
      if (i < n_items) fetch_rows(i, st);
      asm volatile("cp.async.commit_group;" ::: "memory");   // one group per stage, even if empty
    }
  } else if (t == 0) {
    for (int st = 0; st < STAGES; ++st) {
      const int64_t i = blockIdx.x + (int64_t)st * gridDim.x;
      if (i < n_items) fetch(i, st);
    }
  }
  int64_t kk = 0;
  for (int64_t i = blockIdx.x; i < n_items; i += gridDim.x, ++kk) {
    const int st = (int)(kk % STAGES);
    const int buf = (int)(kk & 1);
    const PoolItem it = pool_item(g, i);
    const int64_t len = kv_len(g, it.blk);
    if (perm) {
      asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
      __syncthreads();
    } else {
      ptx::mbar_wait(full + st, (uint32_t)((kk / STAGES) & 1));
    }
    const uint8_t* blk = ring + st * stage_bytes;
    if (kp && (it.seg > 0 || qp) && t == 0) {
      if (perm) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> bulk read
      // the permuted Q / K / V block, contiguous [H][T][d], for K3's TMA
      __nv_bfloat16* dstp = (it.seg == 0 ? qp : it.seg == 1 ? kp : vp) + (it.h * g.T + kv_row0(g, it.blk)) * D;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                   "cp.async.bulk.commit_group;" ::"l"(dstp),
                   "r"((uint32_t)__cvta_generic_to_shared(blk)), "r"((uint32_t)(len * D * 2))
                   : "memory");
    }
    // ---- phase A ----
    const bool text_k = (it.seg == 1) && (it.blk >= g.N);
    double* raw_out = text_k ? ws.k_cat + (it.h * g.n_cols + g.N + (kv_row0(g, it.blk) - g.Tv)) * D : nullptr;
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    uint32_t pmax = 0, pmin = 0x7FFF7FFFu;
#pragma unroll 4
    for (int64_t r = rp; r < len; r += RP) {
      const uint4 w4 = *reinterpret_cast<const uint4*>(blk + r * D * 2 + tc * 16);
      const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[2 * j] += bf16_scaled(w[j] << 16);
        acc[2 * j + 1] += bf16_scaled(w[j]);   // (the low half is masked off by the encoding)
      }
      const uint32_t m0 = w4.x & 0x7FFF7FFFu, m1 = w4.y & 0x7FFF7FFFu, m2 = w4.z & 0x7FFF7FFFu,
                     m3 = w4.w & 0x7FFF7FFFu;
      pmax = __vimax3_u16x2(pmax, __vimax3_u16x2(m0, m1, m2), m3);
      pmin = __vimin3_u16x2(pmin, __vimin3_u16x2(m0, m1, m2), m3);
      if (raw_out) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          raw_out[r * D + tc * 8 + 2 * j] = (double)__uint_as_float(w[j] << 16);
          raw_out[r * D + tc * 8 + 2 * j + 1] = (double)__uint_as_float(w[j] & 0xFFFF0000u);
        }
      }
    }
    uint32_t tmax = max(pmax & 0xFFFFu, pmax >> 16);
    uint32_t tmin = min(pmin & 0xFFFFu, pmin >> 16);
    if (tmin == 0) {
      // an exact zero: the minimum over NONZERO magnitudes (0 -> 0x7FFF key)
      uint32_t kmin = 0x7FFF7FFFu;
      for (int64_t r = rp; r < len; r += RP) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(blk + r * D * 2 + tc * 16);
        const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) kmin = __vminu2(kmin, ((w[j] & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x7FFF7FFFu);
      }
      const uint32_t km = min(kmin & 0xFFFFu, kmin >> 16);
      tmin = km == 0x7FFFu ? 0xFFFFu : km + 1;   // 0xFFFF: no nonzero value
    }
    // lanes holding the same 8 columns (other row phases) merge their sums
#pragma unroll
    for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tmax = max(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
      tmin = min(tmin, __shfl_xor_sync(0xffffffffu, tmin, o));
    }
    if (lane < TPR) {
      double2* dst = reinterpret_cast<double2*>(s_part + (buf * WARPS + warp) * D + tc * 8);
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = make_double2(acc[2 * j], acc[2 * j + 1]);
    }
    if (lane == 0) {
      s_rng[(buf * WARPS + warp) * 2] = tmax;
      s_rng[(buf * WARPS + warp) * 2 + 1] = tmin;
    }
    if (t == 0 && kp) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // permuted copy read out
    __syncthreads();
    // ---- decision (uniform) ----
    uint32_t mx = 0, mn = 0xFFFFu;
#pragma unroll
    for (int w2 = 0; w2 < WARPS; ++w2) {
      mx = max(mx, s_rng[(buf * WARPS + w2) * 2]);
      mn = min(mn, s_rng[(buf * WARPS + w2) * 2 + 1]);
    }
    if (t == 0 && mx >= 0x7F80u) atomicOr(ws.status + ST_NONFINITE, 1);   // exponent field 0xFF: inf / NaN
    const int lg = len > 1 ? 32 - __clz((int)(len - 1)) : 0;
    // exponent fields (bits >> 7); subnormals (field 0) count as exponent 1
    const int emax = max(1, (int)(mx >> 7)), emin = max(1, (int)(mn >> 7));
    const bool exact = (mn == 0xFFFFu) || (emax - emin + 8 + lg < 53);
    double sum = 0.0;
    if (!exact) {
      if (t < D)
        sum = fsum_exact(len, [&](int64_t r) {
          return (double)__bfloat162float(reinterpret_cast<const __nv_bfloat16*>(blk)[r * D + t]);
        });
      __syncthreads();   // every column has been read from the stage
    }
    // ---- refill stage st with this CTA's item STAGES ahead ----
    {
      const int64_t nx = i + (int64_t)STAGES * gridDim.x;
      if (perm) {
        if (nx < n_items) fetch_rows(nx, st);
        asm volatile("cp.async.commit_group;" ::: "memory");
      } else if (t == 0 && nx < n_items) {
        fetch(nx, st);
      }
    }
    // ---- phase B ----
    if (t < D) {
      const int col = t;
      if (exact) {
#pragma unroll
        for (int w2 = 0; w2 < WARPS; ++w2) sum += s_part[(buf * WARPS + w2) * D + col];
        sum = unscale_896(sum);
      }
      const double flen = (double)len;
      const double mean = sum / flen;            // core.py:172 fsum(...) / length
      // numpy rounds the product first (no FMA contraction): masks.py:166 / masks.py:171
      const double deficit = __dsub_rn(sum, __dmul_rn(flen, mean));
      if (it.seg == 0) {
        ws.q_pool[(it.h * g.N + it.blk) * D + col] = mean;
        ws.q_def[(it.h * g.N + it.blk) * D + col] = deficit;
      } else if (it.seg == 1) {
        const int64_t kc_row = it.blk < g.N ? it.blk : g.N + g.Tt + (it.blk - g.N);
        ws.k_cat[(it.h * g.n_cols + kc_row) * D + col] = mean;
        ws.k_def[(it.h * g.M + it.blk) * D + col] = deficit;
      } else {
        ws.v_pool[(it.h * g.M + it.blk) * D + col] = mean;
      }
      if (it.seg < 2 && deficit != 0.0) atomicOr(ws.status + ST_DEFICIT, 1);
    }
  }
  if (t == 0 && kp) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int D>
cudaError_t launch_bulk(const Geometry& g, const void* q, const void* k, const void* v, const Workspace& ws,
                        cudaStream_t st, const int32_t* perm, void* kp, void* vp, void* qp) {
  constexpr int STAGES = 3;
  constexpr int WARPS = kBulkThreads / 32;
  const size_t smem = (size_t)STAGES * g.B * D * 2 + STAGES * 8 + 2 * WARPS * D * 8 + 2 * WARPS * 2 * 4;
  CUtensorMap tq, tk, tv;
  if (!make_rows_tmap(&tq, q, g, D, (int)g.B, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_rows_tmap(&tk, k, g, D, (int)g.B, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_rows_tmap(&tv, v, g, D, (int)g.B, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  auto kern = pool_bulk_kernel<D, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_items = g.H * (g.N + 2 * g.M);
  const int64_t grid = std::min<int64_t>(n_items, (int64_t)sms * 2);
  kern<<<(unsigned)grid, kBulkThreads, smem, st>>>(tq, tk, tv, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                                   (const __nv_bfloat16*)v, ws, g, n_items, perm,
                                                   (__nv_bfloat16*)kp, (__nv_bfloat16*)vp, (__nv_bfloat16*)qp);
  return cudaGetLastError();
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
                        const Workspace& ws, cudaStream_t st, int* launches, const int32_t* perm,
                        void* kp, void* vp, void* qp) {
  ++*launches;
  switch (g.dtype) {
    case RSA_BF16: {
      // bulk-copy streaming path when a block is one 16-byte-aligned range
      // that fits two ring stages per CTA, three CTAs per SM
      const bool aligned = ((uintptr_t)q % 16 == 0) && ((uintptr_t)k % 16 == 0) && ((uintptr_t)v % 16 == 0);
      // rows 16-byte aligned for TMA; three ring stages + partials fit two CTAs per SM
      const bool fits = g.B * g.d * 2 * 3 <= 96 * 1024 && g.B <= 256 && (g.s_tok * 2) % 16 == 0 &&
                        (g.s_head * 2) % 16 == 0 && (g.s_batch * 2) % 16 == 0;
      if (aligned && fits && g.d == 128) return launch_bulk<128>(g, q, k, v, ws, st, perm, kp, vp, qp);
      if (aligned && fits && g.d == 64) return launch_bulk<64>(g, q, k, v, ws, st, perm, kp, vp, qp);
      if (perm) return cudaErrorNotSupported;
      return launch_typed<__nv_bfloat16>(g, q, k, v, ws, st);
    }
    case RSA_F32: if (perm) return cudaErrorNotSupported; return launch_typed<float>(g, q, k, v, ws, st);
    default: if (perm) return cudaErrorNotSupported; return launch_typed<double>(g, q, k, v, ws, st);
  }
}

}  // namespace rsa
