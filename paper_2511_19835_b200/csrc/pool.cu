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
  const T* src = (seg == 0 ? q : seg == 1 ? k : v) + row_off(g, h, row0);   // rows g.s_tok apart
  const int64_t ts = g.s_tok;

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
        for (int u = 0; u < 8; ++u) load_vec_f32<T, VEC>(src + (r + u * rg_count) * ts + c * VEC, x[u]);
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
        load_vec_f32<T, VEC>(src + r * ts + c * VEC, x);
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
      load_vec<T, VEC>(src + r * ts + c * VEC, x);
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
      sum = fsum_exact(len, [&](int64_t r) { return to_f64(src[r * ts + col]); });
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
// bf16 path (pool_warp_kernel below): every pooling item -- one (head,
// segment, block) = B rows x d bf16 -- is reduced by ONE warp from a TMA-fed
// shared-memory ring (a [d x SR] box of the 4-D row map, so any row strides
// work).  Per element:
//    the bf16 x is re-encoded EXACTLY as the fp64 value x * 2^-896 with two
//    or three integer ops -- its f32 bit pattern shifted right by 3 with the
//    sign kept: the 8-bit exponent lands in the low bits of the f64 exponent,
//    the 7 significand bits at the top of the f64 significand; 0 -> +-0,
//    subnormals -> f64 subnormals, one scale for all -- instead of a
//    bf16->f64 conversion per element on the XU pipe (what bound round 1's
//    kernel); an fp64 add; packed 16x2 integer max / min of the |x| bit
//    patterns (3-input DPX min/max).
// Per item: lanes sharing columns merge by shuffle, the magnitude range by
// warp REDUX; the plain sums are exact iff e_max - e_min + 8 + ceil(log2 len)
// < 53 (e_min over nonzero values: a part with an exact zero recomputes its
// minimum without zeros), and are then unscaled by 2^896 (exact).  A block
// failing the test (never for sane data) is re-summed per column with
// Shewchuk's algorithm -- the algorithm of math.fsum, correctly rounded.
// Result: bit-identical to the reference's math.fsum pooling (core.py:154-189).
// ---------------------------------------------------------------------------

// f32 bit pattern of a bf16 value (low 16 bits zero) -> the fp64 x * 2^-896, exactly
__device__ __forceinline__ double bf16_scaled(uint32_t f32_bits) {
  return __hiloint2double((int)(((int)f32_bits >> 3) & 0x8FFFE000), 0);
}
__device__ __forceinline__ double unscale_896(double x) {
  return __dmul_rn(x, __hiloint2double(0x77F00000, 0));   // * 2^896
}

struct PoolItem {
  int h, blk, seg;
};

// items: per head [N Q video blocks][M K blocks][M V blocks] (32-bit: the
// launcher checks H (N + 2M) < 2^31)
__device__ __forceinline__ PoolItem pool_item(int per_head, int n_q, int n_kv, int i) {
  PoolItem it;
  it.h = i / per_head;
  const int r = i - it.h * per_head;
  if (r < n_q) { it.seg = 0; it.blk = r; }
  else if (r < n_q + n_kv) { it.seg = 1; it.blk = r - n_q; }
  else { it.seg = 2; it.blk = r - n_q - n_kv; }
  return it;
}

// One warp per CTA, one pooling item (block) at a time, no block-wide
// synchronisation: the warp's lane 0 streams the item in 8 KB parts (a TMA
// box of SR rows; four parts per 32 KB block) through a 2-stage ring of its
// own, the 32 lanes reduce every part as it lands (lanes l and l + 16 take
// alternate rows of the same 8 columns at d = 128), and the item's column sums,
// exactness test (warp REDUX of the magnitude range) and outputs stay in the
// warp.  Twelve such CTAs per SM keep 192 KB of HBM reads in flight (A/B over
// part size x stages x CTAs/SM: 8 KB x 2 x 12 best).
#ifndef RSA_K1_PART_BYTES
#define RSA_K1_PART_BYTES 8192   // one TMA part (rows x d x 2 bytes)
#endif
#ifndef RSA_K1_CTAS_PER_SM
#define RSA_K1_CTAS_PER_SM 12    // one warp each
#endif
#ifndef RSA_K1_STAGES
#define RSA_K1_STAGES 2
#endif

template <int D>
__global__ void __launch_bounds__(32, RSA_K1_CTAS_PER_SM)
pool_warp_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                 const __grid_constant__ CUtensorMap tm_v, const __nv_bfloat16* __restrict__ q,
                 const __nv_bfloat16* __restrict__ k, const __nv_bfloat16* __restrict__ v, Workspace ws,
                 Geometry g, int n_items, int stage_rows, const int32_t* __restrict__ perm, __nv_bfloat16* kp,
                 __nv_bfloat16* vp, __nv_bfloat16* qp) {
  constexpr int TPR = D / 8;          // lanes per row: 16 bytes (8 bf16) each
  constexpr int RPI = 32 / TPR;       // rows per warp iteration
  constexpr int NST = RSA_K1_STAGES;
  extern __shared__ __align__(128) uint8_t smem[];
  const int SR = stage_rows;
  const int stage_bytes = SR * D * 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * stage_bytes);
  const int lane = threadIdx.x, tc = lane % TPR, rl = lane / TPR;
  const int n_q = (int)g.N, n_kv = (int)g.M, per_head = n_q + 2 * n_kv;
  const int B = (int)g.B;
  const int parts = (B + SR - 1) / SR;
  const __nv_bfloat16* bases[3] = {q, k, v};

  // fetch cursor: (item, part) of the next stage load
  int fi = blockIdx.x, fpart = 0;
  constexpr int CPR = D * 2 / 16;
  auto issue = [&](int st) {
    if (fi >= n_items) return;
    const PoolItem it = pool_item(per_head, n_q, n_kv, fi);
    const int r0 = fpart * SR;
    if (perm) {   // permuted (Morton) rows: every lane gathers 16-byte pieces (cp.async)
      const int len = (int)kv_len(g, it.blk);
      const int rows = min(SR, len - r0);
      uint8_t* dst = smem + st * stage_bytes;
      for (int c = lane; c < rows * CPR; c += 32) {
        const int r = c / CPR, cc = c % CPR;
        const int64_t row = it.blk < n_q ? perm[(int64_t)it.blk * B + r0 + r] : kv_row0(g, it.blk) + r0 + r;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(dst + r * D * 2 + cc * 16)),
                     "l"(bases[it.seg] + row_off(g, it.h, row) + cc * 8)
                     : "memory");
      }
    } else if (lane == 0) {
      ptx::mbar_expect_tx(full + st, (uint32_t)stage_bytes);
      ptx::tma_load_4d(smem + st * stage_bytes, it.seg == 0 ? &tm_q : it.seg == 1 ? &tm_k : &tm_v, full + st, 0,
                       (int)kv_row0(g, it.blk) + r0, it.h % (int)g.hb, it.h / (int)g.hb);
    }
    if (++fpart == parts) { fpart = 0; fi += gridDim.x; }
  };
  if (lane == 0) {
    ptx::prefetch_tmap(&tm_q);
    ptx::prefetch_tmap(&tm_k);
    ptx::prefetch_tmap(&tm_v);
    for (int st = 0; st < NST; ++st) ptx::mbar_init(full + st, 1);
    ptx::fence_barrier_init();
  }
  __syncwarp();
  for (int st = 0; st < NST; ++st) {
    issue(st);
    if (perm) asm volatile("cp.async.commit_group;" ::: "memory");   // one group per stage, even if empty
  }
  int u = 0;   // stage loads consumed
  for (int i = blockIdx.x; i < n_items; i += gridDim.x) {
    const PoolItem it = pool_item(per_head, n_q, n_kv, i);
    const int len = (int)kv_len(g, it.blk);
    const bool text_k = it.seg == 1 && it.blk >= n_q;
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    // packed 16x2 |x| bit patterns: max, and min over NONZERO values (0xFFFF: none)
    uint32_t pmax = 0, nzmin = 0xFFFFFFFFu;
    for (int part = 0; part < parts; ++part, ++u) {
      const int st = u % NST;
      if (perm) {
        asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
        __syncwarp();
      } else {
        ptx::mbar_wait(full + st, (uint32_t)((u / NST) & 1));
      }
      const uint8_t* stage = smem + st * stage_bytes;
      const int r0 = part * SR;
      const int rows = min(SR, len - r0);   // (<= 0: a short block's unused part)
      if (kp && (it.seg > 0 || qp) && lane == 0 && rows > 0) {
        if (perm) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> bulk read
        // the permuted Q / K / V rows, contiguous [H][T][d], for K3's TMA
        __nv_bfloat16* dstp =
            (it.seg == 0 ? qp : it.seg == 1 ? kp : vp) + ((int64_t)it.h * g.T + kv_row0(g, it.blk) + r0) * D;
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                     "cp.async.bulk.commit_group;" ::"l"(dstp),
                     "r"((uint32_t)__cvta_generic_to_shared(stage)), "r"((uint32_t)(rows * D * 2))
                     : "memory");
      }
      uint32_t pmin = 0xFFFFFFFFu;   // this part's min, zeros included
      const uint8_t* rowp = stage + rl * D * 2 + tc * 16;
#pragma unroll 4
      for (int r = rl; r < rows; r += RPI, rowp += RPI * D * 2) {
        const uint4 w4 = *reinterpret_cast<const uint4*>(rowp);
        acc[0] += bf16_scaled(w4.x << 16);
        acc[1] += bf16_scaled(w4.x);   // (the low half is masked off by the encoding)
        acc[2] += bf16_scaled(w4.y << 16);
        acc[3] += bf16_scaled(w4.y);
        acc[4] += bf16_scaled(w4.z << 16);
        acc[5] += bf16_scaled(w4.z);
        acc[6] += bf16_scaled(w4.w << 16);
        acc[7] += bf16_scaled(w4.w);
        const uint32_t m0 = w4.x & 0x7FFF7FFFu, m1 = w4.y & 0x7FFF7FFFu, m2 = w4.z & 0x7FFF7FFFu,
                       m3 = w4.w & 0x7FFF7FFFu;
        pmax = __vimax3_u16x2(pmax, __vimax3_u16x2(m0, m1, m2), m3);
        pmin = __vimin3_u16x2(pmin, __vimin3_u16x2(m0, m1, m2), m3);
      }
      const bool zero_here = (pmin & 0xFFFFu) == 0 || (pmin >> 16) == 0;
      if (text_k || zero_here) {
        // text keys also go to k_cat raw (fp64; 2 blocks per head); an exact
        // zero: this part's minimum over NONZERO magnitudes (0 -> 0x7FFF key)
        double* raw_out =
            text_k ? ws.k_cat + ((int64_t)it.h * g.n_cols + n_q + (kv_row0(g, it.blk) - g.Tv) + r0) * D : nullptr;
        uint32_t kmin = 0x7FFF7FFFu;
        for (int r = rl; r < rows; r += RPI) {
          const uint4 w4 = *reinterpret_cast<const uint4*>(stage + r * D * 2 + tc * 16);
          const uint32_t w[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            kmin = __vminu2(kmin, ((w[j] & 0x7FFF7FFFu) + 0x7FFF7FFFu) & 0x7FFF7FFFu);
            if (raw_out) {
              raw_out[r * D + tc * 8 + 2 * j] = (double)__uint_as_float(w[j] << 16);
              raw_out[r * D + tc * 8 + 2 * j + 1] = (double)__uint_as_float(w[j] & 0xFFFF0000u);
            }
          }
        }
        if (zero_here) {
          // this part's nonzero minimum: key + 1 (a 0x7FFF key: only zeros -> 0xFFFF, none)
          const uint32_t k0 = kmin & 0xFFFFu, k1 = kmin >> 16;
          const uint32_t n0 = k0 == 0x7FFFu ? 0xFFFFu : k0 + 1, n1 = k1 == 0x7FFFu ? 0xFFFFu : k1 + 1;
          pmin = (n1 << 16) | n0;
        }
      }
      nzmin = __vminu2(nzmin, pmin);
      if (kp && (it.seg > 0 || qp) && lane == 0 && rows > 0)
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");   // permuted copy read out
      __syncwarp();
      // stage st is consumed: refill it with the load NST ahead
      if (!perm && lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(st);
      if (perm) asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // ---- this item's column sums, exactness, outputs (all in the warp) ----
#pragma unroll
    for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    uint32_t tmax = max(pmax & 0xFFFFu, pmax >> 16);
    uint32_t tmin = min(nzmin & 0xFFFFu, nzmin >> 16);
    tmax = __reduce_max_sync(0xffffffffu, tmax);
    tmin = __reduce_min_sync(0xffffffffu, tmin);
    if (lane == 0 && tmax >= 0x7F80u) atomicOr(ws.status + ST_NONFINITE, 1);   // exponent 0xFF: inf / NaN
    const int lg = len > 1 ? 32 - __clz(len - 1) : 0;
    // exponent fields (bits >> 7); subnormals (field 0) count as exponent 1
    const int emax = max(1, (int)(tmax >> 7)), emin = max(1, (int)(tmin >> 7));
    const bool exact = (tmin >= 0xFFFFu) || (emax - emin + 8 + lg < 53);
    const bool pow2 = (len & (len - 1)) == 0;
    const int64_t h = it.h;
    double* dst_mean;
    double* dst_def = nullptr;
    if (it.seg == 0) {
      dst_mean = ws.q_pool + (h * g.N + it.blk) * D;
      dst_def = ws.q_def + (h * g.N + it.blk) * D;
    } else if (it.seg == 1) {
      const int64_t kc_row = it.blk < n_q ? it.blk : g.N + g.Tt + (it.blk - n_q);
      dst_mean = ws.k_cat + (h * g.n_cols + kc_row) * D;
      dst_def = ws.k_def + (h * g.M + it.blk) * D;
    } else {
      dst_mean = ws.v_pool + (h * g.M + it.blk) * D;
    }
    bool nonzero_def = false;
    auto finish = [&](int col, double sum) {
      // core.py:172 fsum(...) / length; a power-of-two length divides exactly
      // by its reciprocal (and then the deficit is exactly 0)
      const double mean = pow2 ? __dmul_rn(sum, 1.0 / (double)len) : sum / (double)len;
      // numpy rounds the product first (no FMA contraction): masks.py:166 / masks.py:171
      const double deficit = pow2 ? 0.0 : __dsub_rn(sum, __dmul_rn((double)len, mean));
      dst_mean[col] = mean;
      if (dst_def) dst_def[col] = deficit;
      nonzero_def |= deficit != 0.0;
    };
    if (exact) {
      if (lane < TPR) {
#pragma unroll
        for (int j = 0; j < 8; ++j) finish(tc * 8 + j, unscale_896(acc[j]));
      }
    } else {
      // correctly rounded column sums (math.fsum), re-read from global memory
      const __nv_bfloat16* src = bases[it.seg];
      for (int col = lane; col < D; col += 32) {
        const double sum = fsum_exact(len, [&](int64_t r) {
          const int64_t row = (perm && it.blk < n_q) ? perm[(int64_t)it.blk * B + r] : kv_row0(g, it.blk) + r;
          return (double)__bfloat162float(src[row_off(g, it.h, row) + col]);
        });
        finish(col, sum);
      }
    }
    if (it.seg < 2 && __any_sync(0xffffffffu, nonzero_def) && lane == 0) atomicOr(ws.status + ST_DEFICIT, 1);
  }
  if (lane == 0 && kp) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int D>
cudaError_t launch_bulk(const Geometry& g, const void* q, const void* k, const void* v, const Workspace& ws,
                        cudaStream_t st, const int32_t* perm, void* kp, void* vp, void* qp) {
  const int stage_rows = (int)std::min<int64_t>(g.B, RSA_K1_PART_BYTES / (D * 2));
  const size_t smem = (size_t)RSA_K1_STAGES * stage_rows * D * 2 + RSA_K1_STAGES * 8;
  if (g.H * (g.N + 2 * g.M) >= ((int64_t)1 << 31)) return cudaErrorNotSupported;
  CUtensorMap tq, tk, tv;
  if (!make_rows_tmap(&tq, q, g, D, stage_rows, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_rows_tmap(&tk, k, g, D, stage_rows, CU_TENSOR_MAP_SWIZZLE_NONE) ||
      !make_rows_tmap(&tv, v, g, D, stage_rows, CU_TENSOR_MAP_SWIZZLE_NONE))
    return cudaErrorInvalidValue;
  auto kern = pool_warp_kernel<D>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int n_items = (int)(g.H * (g.N + 2 * g.M));
  const int grid = (int)std::min<int64_t>(n_items, (int64_t)sms * RSA_K1_CTAS_PER_SM);
  kern<<<(unsigned)grid, 32, smem, st>>>(tq, tk, tv, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
                                          (const __nv_bfloat16*)v, ws, g, n_items, stage_rows, perm,
                                          (__nv_bfloat16*)kp, (__nv_bfloat16*)vp, (__nv_bfloat16*)qp);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_typed(const Geometry& g, const void* q, const void* k, const void* v,
                         const Workspace& ws, cudaStream_t st) {
  dim3 grid((unsigned)g.M, 3, (unsigned)g.H);
  constexpr int V16 = 16 / sizeof(T);
  const bool aligned = (g.d % V16 == 0) && ((uintptr_t)q % 16 == 0) &&
                       ((uintptr_t)k % 16 == 0) && ((uintptr_t)v % 16 == 0) && g.s_tok % V16 == 0 &&
                       g.s_head % V16 == 0 && g.s_batch % V16 == 0;
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
      const bool fits = g.B * g.d * 2 <= 32 * 1024 && g.B <= 256 && (g.s_tok * 2) % 16 == 0 &&
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
