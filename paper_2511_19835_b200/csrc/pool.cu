// K1: exactly rounded fp64 block pooling (HBM-bound streaming reduction).
//
// Reference: block_pool / block_sums (pkg/src/rectattn/core.py:154-189) use
// math.fsum per column, pool_problem (core.py:192-201) pools Q video blocks,
// K video blocks and all V blocks; _pool_rows (masks.py:130-135) pools the
// text keys per (possibly ragged) text block; pooling_error (masks.py:165-171)
// needs the deficits sum - len * mean.
//
// Layout: one CTA per (block, segment, head); 256 threads stream the block's
// rows with 128-bit non-allocating loads (8 bf16 / 4 f32 / 2 f64 per load),
// each thread owning a column chunk and a row phase.  For bf16/f32 data the
// sums are plain fp64 adds, proven exact per block from its magnitude range
// (see pass 1 below); otherwise (f64 data, or a block spanning too many
// binades) partial sums are (hi, lo) TwoSum pairs.  Either way the merged
// result is the exactly rounded sum, i.e. bit-identical to math.fsum, and
// independent of launch geometry.
#include "rsa_internal.cuh"

#include <cfloat>

#include <algorithm>

namespace rsa {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
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
  __shared__ double s_lo[2048];

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
  if (!exact) {
    double hi[VEC], lo[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) { hi[i] = 0.0; lo[i] = 0.0; }
    if (rg < rg_count) {
      for (int64_t r = rg; r < len; r += rg_count) {
        double x[VEC];
        load_vec<T, VEC>(src + r * d + c * VEC, x);
#pragma unroll
        for (int i = 0; i < VEC; ++i) {
          nonfinite |= !(fabs(x[i]) <= DBL_MAX);
          double sm, e;
          two_sum(hi[i], x[i], sm, e);
          hi[i] = sm;
          lo[i] += e;
        }
        if (raw_out && !kTryPlain) {
#pragma unroll
          for (int i = 0; i < VEC; ++i) raw_out[r * d + c * VEC + i] = x[i];
        }
      }
#pragma unroll
      for (int i = 0; i < VEC; ++i) {
        s_hi[rg * d + i * tpr + c] = hi[i];
        s_lo[rg * d + i * tpr + c] = lo[i];
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
      double S = 0.0, E = 0.0;
      for (int p = 0; p < rg_count; ++p) {
        double s, e;
        two_sum(S, s_hi[p * d + slot], s, e);
        S = s;
        E += e + s_lo[p * d + slot];
      }
      sum = S + E;                            // exactly rounded block sum
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
// bf16 fast path: persistent CTAs stream whole blocks (B rows x d bf16, one
// contiguous B*d*2-byte range of [H][T][d]) into a shared-memory ring with 1-D
// bulk async copies (cp.async.bulk, TMA engine), several blocks in flight per
// CTA, and reduce them from shared memory.  The exactness argument is the one
// of pool_kernel (pass 1): bf16 values have p = 8 significant bits, so fp64
// partial sums are exact while e_max - e_min + 8 + ceil(log2 len) < 53; a
// block that fails the test (never for sane data) is re-summed from the same
// shared-memory copy with TwoSum pairs.  Bit-identical to math.fsum either way.
// ---------------------------------------------------------------------------
constexpr int kBulkThreads = 256;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(parity)
        : "memory");
  }
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
__global__ void __launch_bounds__(kBulkThreads, 3)
pool_bulk_kernel(const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k,
                 const __nv_bfloat16* __restrict__ v, Workspace ws, Geometry g, int64_t n_items,
                 const int32_t* __restrict__ perm, __nv_bfloat16* kp, __nv_bfloat16* vp,
                 __nv_bfloat16* qp) {
  constexpr int WPR = D / 2;                   // 32-bit words (bf16 pairs) per row
  constexpr int RP = kBulkThreads / WPR;       // row phases
  extern __shared__ __align__(128) uint8_t smem[];
  const int stage_bytes = (int)(g.B * D * 2);
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * stage_bytes);
  double* s_part = reinterpret_cast<double*>(full + STAGES);     // [RP][D] hi (+ [RP][D] lo)
  float* s_rng = reinterpret_cast<float*>(s_part + 2 * RP * D);  // [8 warps][2]
  __shared__ int s_exact;

  const int t = threadIdx.x;
  const int word = t % WPR, rp = t / WPR;
  auto src_of = [&](const PoolItem& it, uint32_t& bytes) -> const void* {
    const int64_t len = kv_len(g, it.blk);
    bytes = (uint32_t)(len * D * 2);
    const __nv_bfloat16* base = it.seg == 0 ? q : it.seg == 1 ? k : v;
    return base + (it.h * g.T + kv_row0(g, it.blk)) * D;
  };
  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) bar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Stage item i into ring slot s (thread 0): one contiguous bulk copy.
  auto fetch = [&](int64_t i, int s) {
    const PoolItem it = pool_item(g, i);
    uint32_t bytes;
    const void* src = src_of(it, bytes);
    uint8_t* dst = ring + s * stage_bytes;
    if (t == 0) {
      bar_expect_tx(full + s, bytes);
      bulk_g2s(dst, src, bytes, full + s);
    }
  };
  // Permuted problem: every thread gathers 16-byte pieces of the block's rows
  // (LDGSTS, cp.async groups) -- 128 row-sized bulk copies per block keep the
  // TMA engine busy issuing instead of moving bytes.
  constexpr int CPR = D * 2 / 16;   // 16-byte pieces per row
  auto fetch_rows = [&](int64_t i, int s) {
    const PoolItem it = pool_item(g, i);
    const int64_t len = kv_len(g, it.blk);
    const __nv_bfloat16* base = (it.seg == 0 ? q : it.seg == 1 ? k : v) + it.h * g.T * D;
    uint8_t* dst = ring + s * stage_bytes;
    for (int64_t c = t; c < len * CPR; c += kBulkThreads) {
      const int64_t r = c / CPR, cc = c % CPR;
      const int64_t row = it.blk < g.N ? perm[it.blk * g.B + r] : kv_row0(g, it.blk) + r;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                       (uint32_t)__cvta_generic_to_shared(dst + r * D * 2 + cc * 16)),
                   "l"(base + row * D + cc * 8)
                   : "memory");
    }
  };
  if (perm) {
    for (int s = 0; s < STAGES; ++s) {
      const int64_t i = blockIdx.x + (int64_t)s * gridDim.x;
      if (i < n_items) fetch_rows(i, s);
      asm volatile("cp.async.commit_group;" ::: "memory");   // one group per stage, even if empty
    }
  } else if (t < 32) {
    for (int s = 0; s < STAGES; ++s) {
      const int64_t i = blockIdx.x + (int64_t)s * gridDim.x;
      if (i >= n_items) break;
      fetch(i, s);
    }
  }
  int64_t kk = 0;
  for (int64_t i = blockIdx.x; i < n_items; i += gridDim.x, ++kk) {
    const int s = (int)(kk % STAGES);
    const PoolItem it = pool_item(g, i);
    const int64_t len = kv_len(g, it.blk);
    if (perm) {
      // this item's group (committed STAGES groups ago) has landed, all threads' pieces
      asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");
      __syncthreads();
    } else {
      bar_wait(full + s, (uint32_t)((kk / STAGES) & 1));
    }
    const uint32_t* blk = reinterpret_cast<const uint32_t*>(ring + s * stage_bytes);
    if (kp && (it.seg > 0 || qp) && t == 0) {
      if (perm) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> bulk read
      // the permuted Q / K / V block, contiguous, for K3's TMA (shared -> global bulk copy)
      __nv_bfloat16* dstp = (it.seg == 0 ? qp : it.seg == 1 ? kp : vp) + (it.h * g.T + kv_row0(g, it.blk)) * D;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n\t"
                   "cp.async.bulk.commit_group;" ::"l"(dstp),
                   "r"((uint32_t)__cvta_generic_to_shared(blk)), "r"((uint32_t)(len * D * 2))
                   : "memory");
    }
    // pass 1: plain fp64 sums of this thread's column pair over its row phase,
    // plus the magnitude range (bf16 bits & 0x7FFF is monotonic in |x|)
    double a0 = 0.0, a1 = 0.0;
    // packed 16x2 magnitude tracking: max of (bits & 0x7FFF); min over
    // nonzero values through the key (mag + 0x7FFF) & 0x7FFF (0 -> 0x7FFF,
    // x -> x - 1; no carry crosses the halves)
    uint32_t pmax = 0, pmin = 0x7FFF7FFFu;
    const bool text_k = (it.seg == 1) && (it.blk >= g.N);
    double* raw_out = text_k ? ws.k_cat + (it.h * g.n_cols + g.N + (kv_row0(g, it.blk) - g.Tv)) * D : nullptr;
#pragma unroll 8
    for (int64_t r = rp; r < len; r += RP) {
      const uint32_t w = blk[r * WPR + word];
      const float x0 = __uint_as_float(w << 16), x1 = __uint_as_float(w & 0xFFFF0000u);
      a0 += (double)x0;
      a1 += (double)x1;
      const uint32_t mag = w & 0x7FFF7FFFu;
      pmax = __vmaxu2(pmax, mag);
      pmin = __vminu2(pmin, (mag + 0x7FFF7FFFu) & 0x7FFF7FFFu);
      if (raw_out) {
        raw_out[r * D + 2 * word] = (double)x0;
        raw_out[r * D + 2 * word + 1] = (double)x1;
      }
    }
    s_part[rp * D + 2 * word] = a0;
    s_part[rp * D + 2 * word + 1] = a1;
    uint32_t bmax = max(pmax & 0xFFFFu, pmax >> 16);
    const uint32_t kmin = min(pmin & 0xFFFFu, pmin >> 16);
    uint32_t bmin = kmin == 0x7FFFu ? 0xFFFFu : kmin + 1;   // 0xFFFF: no nonzero value
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      bmax = max(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
      bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
    }
    if (t % 32 == 0) {
      reinterpret_cast<uint32_t*>(s_rng)[2 * (t / 32)] = bmax;
      reinterpret_cast<uint32_t*>(s_rng)[2 * (t / 32) + 1] = bmin;
    }
    __syncthreads();
    if (t == 0) {
      uint32_t mx = 0, mn = 0xFFFFu;
      for (int w = 0; w < kBulkThreads / 32; ++w) {
        mx = max(mx, reinterpret_cast<uint32_t*>(s_rng)[2 * w]);
        mn = min(mn, reinterpret_cast<uint32_t*>(s_rng)[2 * w + 1]);
      }
      if (mx >= 0x7F80u) atomicOr(ws.status + ST_NONFINITE, 1);   // exponent field 0xFF: inf / NaN
      int lg = 0;
      while ((int64_t(1) << lg) < len) ++lg;
      // exponent fields (bits >> 7); subnormals (field 0) count as exponent 1
      const int emax = max(1, (int)(mx >> 7)), emin = max(1, (int)(mn >> 7));
      s_exact = (mn == 0xFFFFu) || (emax - emin + 8 + lg < 53);
    }
    __syncthreads();
    const bool exact = s_exact != 0;
    if (!exact) {
      // TwoSum (hi, lo) pairs over the same shared-memory copy
      double h0 = 0.0, l0 = 0.0, h1 = 0.0, l1 = 0.0;
      for (int64_t r = rp; r < len; r += RP) {
        const uint32_t w = blk[r * WPR + word];
        double sm, e;
        two_sum(h0, (double)__uint_as_float(w << 16), sm, e); h0 = sm; l0 += e;
        two_sum(h1, (double)__uint_as_float(w & 0xFFFF0000u), sm, e); h1 = sm; l1 += e;
      }
      s_part[rp * D + 2 * word] = h0;
      s_part[rp * D + 2 * word + 1] = h1;
      s_part[RP * D + rp * D + 2 * word] = l0;
      s_part[RP * D + rp * D + 2 * word + 1] = l1;
      __syncthreads();
    }
    // stage s is free (its permuted copy, if any, has been read out): refill
    // it with this CTA's item STAGES ahead
    if (perm) {
      if (t == 0 && kp) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncthreads();
      const int64_t nx = i + (int64_t)STAGES * gridDim.x;
      if (nx < n_items) fetch_rows(nx, s);
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else if (t < 32) {
      if (t == 0 && kp) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
      const int64_t nx = i + (int64_t)STAGES * gridDim.x;
      if (nx < n_items) fetch(nx, s);
    }
    for (int col = t; col < D; col += kBulkThreads) {
      double sum;
      if (exact) {
        sum = 0.0;
        for (int p = 0; p < RP; ++p) sum += s_part[p * D + col];
      } else {
        double S = 0.0, E = 0.0;
        for (int p = 0; p < RP; ++p) {
          double sm, e;
          two_sum(S, s_part[p * D + col], sm, e);
          S = sm;
          E += e + s_part[RP * D + p * D + col];
        }
        sum = S + E;
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
    __syncthreads();
  }
  if (t == 0 && kp) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int D>
cudaError_t launch_bulk(const Geometry& g, const void* q, const void* k, const void* v, const Workspace& ws,
                        cudaStream_t st, const int32_t* perm, void* kp, void* vp, void* qp) {
  constexpr int STAGES = 2;
  constexpr int RP = kBulkThreads / (D / 2);
  const size_t smem = (size_t)STAGES * g.B * D * 2 + STAGES * 8 + 2 * RP * D * 8 + 64;
  auto kern = pool_bulk_kernel<D, STAGES>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n_items = g.H * (g.N + 2 * g.M);
  const int64_t grid = std::min<int64_t>(n_items, (int64_t)sms * 3);
  kern<<<(unsigned)grid, kBulkThreads, smem, st>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)k,
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
      const bool fits = g.B * g.d * 2 * 2 <= 64 * 1024;
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
