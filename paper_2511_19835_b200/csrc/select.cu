// K2: pooled scoring, IPAR, deterministic block selection, GAPR gate,
// rectification factors, compensation rows and the kv-block lists K3 walks.
//
// Reference (pkg/src/rectattn):
//   mixed_pooled_scores  ipar.py:36-42     scores = q_pool k_mix^T / sqrt(d), softmax
//   reallocate           ipar.py:45-66     D = B*sum(A_v) + sum(A_t)
//   implicit_full_attn   ipar.py:69-86     text re-aggregation -> a_pool (N x M)
//   build_sparse_mask    masks.py:83-117   stable argsort(-a), sequential cumsum,
//                                          count = clip(max(ceil(fM), first_p), 1, M)
//   pooled_scores        masks.py:120-127  video columns == mixed video columns
//   attention_gain       masks.py:138-146  |B * len_m * s_pool|
//   pooling_error        masks.py:149-176  closed form from the K1 deficits
//   compensation_mask    masks.py:179-186  gain > error (ties -> False)
//   rectification_factors rectify.py:56-63 R = 1 - excluded mass
//   apply_rectification  rectify.py:84-87  (a_pool masked to applied) @ v_pool
//
// Everything is fp64 (the bit-exact mask needs it).  The
// two GEMM-shaped stages (N x n_cols x d scores, N x d x M compensation) run a
// register-tiled fp64 GEMM; the per-row stage (softmax, reallocation, sort,
// cumsum, gate, lists) runs one CTA per query block with a shared-memory
// bitonic sort on the composite key (weight desc, block index asc) -- exactly
// numpy's stable argsort of -a_pool.
#include "rsa_internal.cuh"


#include <algorithm>
#include <cfloat>
#include <cstdlib>

namespace rsa {
namespace {

// ----------------------------------------------------------------------------
// block-wide deterministic reductions (fixed tree order)
// ----------------------------------------------------------------------------
constexpr int RT = 128;

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}
__device__ double block_sum(double x, double* red) {
  x = warp_sum(x);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  double y = (threadIdx.x < RT / 32) ? red[threadIdx.x] : 0.0;
  if (w == 0) y = warp_sum(y);
  if (threadIdx.x == 0) red[0] = y;
  __syncthreads();
  return red[0];
}
__device__ double block_max(double x, double* red) {
  x = warp_max(x);
  const int w = threadIdx.x / 32, l = threadIdx.x % 32;
  __syncthreads();
  if (l == 0) red[w] = x;
  __syncthreads();
  double y = (threadIdx.x < RT / 32) ? red[threadIdx.x] : -DBL_MAX;
  if (w == 0) y = warp_max(y);
  if (threadIdx.x == 0) red[0] = y;
  __syncthreads();
  return red[0];
}
__device__ int block_excl_scan(int x, int* tmp, int* total) {
  // Hillis-Steele over 256 threads (deterministic, integer)
  tmp[threadIdx.x] = x;
  __syncthreads();
  for (int o = 1; o < RT; o <<= 1) {
    int y = threadIdx.x >= o ? tmp[threadIdx.x - o] : 0;
    __syncthreads();
    tmp[threadIdx.x] += y;
    __syncthreads();
  }
  const int incl = tmp[threadIdx.x];
  *total = tmp[RT - 1];
  __syncthreads();
  return incl - x;
}

struct SelectParams {
  Geometry g;
  Workspace ws;
  double p;
  int64_t k_floor;
  int radius;
  int force_text;
  int variant;
  double inv_sqrt_d;
  double sqrt_d;
  int p2;  // power of two >= M for the sort
  int use_sort;  // 1: top-K from one full bitonic sort of the row (no radix select)
};

// (value desc, index asc) ordering == numpy argsort(-a, kind="stable")
__device__ __forceinline__ bool before(double va, int ia, double vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

// in-place bitonic sort of n (power of two) (value, index) pairs in shared
// memory into (value desc, index asc) order
__device__ void bitonic_sort(double* sv, int* si, int n) {
  for (int kk = 2; kk <= n; kk <<= 1) {
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      for (int i = threadIdx.x; i < n; i += RT) {
        const int ixj = i ^ jj;
        if (ixj > i) {
          const bool up = (i & kk) == 0;
          const double va = sv[i], vb = sv[ixj];
          const int ia = si[i], ib = si[ixj];
          const bool swap = up ? before(vb, ib, va, ia) : before(va, ia, vb, ib);
          if (swap) { sv[i] = vb; sv[ixj] = va; si[i] = ib; si[ixj] = ia; }
        }
      }
      __syncthreads();
    }
  }
}

// Sequential cumsum of v[0..n) in order, exactly numpy.cumsum's rounding
// (masks.py:99): the first k with v[0] + ... + v[k-1] >= p, or 0 if none.
// One thread; loads batched ahead of the dependent adds (shared-memory latency
// would otherwise serialise with every add).
__device__ int seq_first_reach(const double* v, int n, double p) {
  double cum = 0.0;
  int j = 0;
  for (; j + 8 <= n; j += 8) {
    double x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = v[j + u];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      cum += x[u];
      if (cum >= p) return j + u + 1;
    }
  }
  for (; j < n; ++j) {
    cum += v[j];
    if (cum >= p) return j + 1;
  }
  return 0;
}

__global__ void __launch_bounds__(RT) select_rows_kernel(SelectParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const Geometry& g = P.g;
  const Workspace& ws = P.ws;
  const int64_t n = blockIdx.x, h = blockIdx.y;
  const int64_t N = g.N, M = g.M, Tt = g.Tt, n_cols = g.n_cols;
  const int64_t n_mix = N + Tt;
  // sa is dead once the a_pool row is built, so the sort values alias it
  // (keeps M = 8192 kv blocks with p > 0 inside 227 KB of shared memory)
  const int64_t sa_len = n_mix > P.p2 ? n_mix : P.p2;
  double* sa = reinterpret_cast<double*>(smem_raw);     // [n_mix] a_mix / a_hat
  double* sv = sa;                                       // [p2] sort values (after a_pool)
  double* ap = sa + sa_len;                              // [M] a_pool row
  int* si = reinterpret_cast<int*>(ap + M);              // [p2] sort indices
  uint8_t* bits = reinterpret_cast<uint8_t*>(si + P.p2); // [M]
  __shared__ double red[RT / 32];
  __shared__ int scan_tmp[RT];
  __shared__ int sh_count;
  __shared__ unsigned hist[256];
  __shared__ int sh_digit, sh_rem;

  // the scores GEMM (cuBLAS) leaves q_pool . k_cat^T; divide by sqrt(d) here
  // (ipar.py:41, masks.py:127 divide, they do not multiply by 1/sqrt(d))
  double* srow = ws.scores + (h * N + n) * n_cols;

  // ---- IPAR: softmax over the mixed row (core.py:204-208) ----
  double mx = -DBL_MAX;
  for (int64_t j = threadIdx.x; j < n_cols; j += RT) {
    const double s = srow[j] / P.sqrt_d;
    srow[j] = s;
    if (j < n_mix) { sa[j] = s; mx = fmax(mx, s); }
  }
  mx = block_max(mx, red);
  double part = 0.0;
  for (int64_t j = threadIdx.x; j < n_mix; j += RT) { const double e = exp(sa[j] - mx); sa[j] = e; part += e; }
  const double tot = block_sum(part, red);
  for (int64_t j = threadIdx.x; j < n_mix; j += RT) sa[j] = sa[j] / tot;
  __syncthreads();

  // ---- reallocation (ipar.py:45-66) ----
  if (Tt > 0 && g.B > 1) {
    // a ragged final video block stands for q_last tokens, not B:
    // D = B * sum_{n<N-1} A_v + q_last * A_v[N-1] + sum A_t
    const bool ragged = g.q_last != g.B;
    double pv = 0.0, pt = 0.0;
    for (int64_t j = threadIdx.x; j < n_mix; j += RT) {
      if (j < N) { if (!(ragged && j == N - 1)) pv += sa[j]; } else pt += sa[j];
    }
    const double sum_v = block_sum(pv, red);
    const double sum_t = block_sum(pt, red);
    const double D = ragged ? ((double)g.B * sum_v + (double)g.q_last * sa[N - 1]) + sum_t
                            : (double)g.B * sum_v + sum_t;
    if (D <= 0.0) { if (threadIdx.x == 0) atomicOr(ws.status + ST_DEGENERATE, 1); }
    __syncthreads();   // every thread has read sa[N - 1]
    for (int64_t j = threadIdx.x; j < n_mix; j += RT)
      sa[j] = (j < N) ? ((double)q_len(g, j) * sa[j]) / D : sa[j] / D;
    __syncthreads();
  }
  // ---- a_pool row: video part + text re-aggregation (ipar.py:76-83) ----
  for (int64_t m = threadIdx.x; m < N; m += RT) ap[m] = sa[m];
  for (int64_t j = 0; j < g.n_text; ++j) {
    const int64_t lo = N + j * g.B, hi = min(N + (j + 1) * g.B, n_mix);
    double pj = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += RT) pj += sa[i];
    const double sj = block_sum(pj, red);
    if (threadIdx.x == 0) ap[N + j] = sj;
  }
  __syncthreads();
  double* ap_out = ws.a_pool + (h * N + n) * M;
  for (int64_t m = threadIdx.x; m < M; m += RT) { ap_out[m] = ap[m]; bits[m] = 0; }
  __syncthreads();

  // ---- selection (masks.py:83-117) ----
  const bool full = P.variant == RSA_VARIANT_FULL;
  if (full) {
    for (int64_t m = threadIdx.x; m < M; m += RT) bits[m] = BIT_MASK | BIT_IMPORTANCE;
  } else {
    // Exact top-K (K = ceil(f*M), masks.py:100) by MSB-first radix select on
    // the fp64 bit patterns (a_pool >= 0, so unsigned order == value order),
    // ties resolved by ascending block index -- the set numpy's stable
    // argsort(-a) puts first.  The cumulative-weight rule (masks.py:101-103)
    // can only enlarge the count beyond K when the sequential cumsum of the
    // sorted top-K stays below p; only then is the full sort needed.
    const int64_t K = P.k_floor < M ? P.k_floor : M;
    bool need_full_sort = P.use_sort != 0;
    if (!need_full_sort) {
    uint64_t prefix = 0, pmask = 0;
    int remaining = (int)K;
    // skip the leading bytes every key shares (a_pool in [0, 1]: sign and
    // high exponent bits agree) -- one dominant histogram bin otherwise
    // serialises its shared-memory atomics
    uint64_t k_and = ~0ull, k_or = 0ull;
    for (int64_t m = threadIdx.x; m < M; m += RT) {
      const uint64_t key = (uint64_t)__double_as_longlong(ap[m]);
      k_and &= key;
      k_or |= key;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      k_and &= __shfl_xor_sync(0xffffffffu, k_and, o);
      k_or |= __shfl_xor_sync(0xffffffffu, k_or, o);
    }
    __shared__ unsigned long long s_and[RT / 32], s_or[RT / 32];
    __shared__ int sh_done;
    if (threadIdx.x % 32 == 0) { s_and[threadIdx.x / 32] = k_and; s_or[threadIdx.x / 32] = k_or; }
    __syncthreads();
    k_and = ~0ull;
    k_or = 0ull;
    for (int w = 0; w < RT / 32; ++w) { k_and &= s_and[w]; k_or |= s_or[w]; }
    const uint64_t differ = k_and ^ k_or;
    int top = 56;
    while (top > 0 && ((differ >> top) & 0xFF) == 0) top -= 8;
    if (top < 56) {
      pmask = ~0ull << (top + 8);
      prefix = k_and & pmask;
    }
    if (threadIdx.x == 0) sh_done = 0;
    for (int shift = top; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += RT) hist[i] = 0u;
      __syncthreads();
      for (int64_t m = threadIdx.x; m < M; m += RT) {
        const uint64_t key = (uint64_t)__double_as_longlong(ap[m]);
        if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 0xFF], 1u);
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        unsigned c[8], tot = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) { c[i] = hist[255 - 8 * lane - i]; tot += c[i]; }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned excl = incl - tot;
        if (excl < (unsigned)remaining && incl >= (unsigned)remaining) {
          unsigned run = excl;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (run + c[i] >= (unsigned)remaining) {
              sh_digit = 255 - 8 * lane - i;
              sh_rem = remaining - (int)run;
              // the whole boundary bin is selected: no lower digit can matter
              sh_done = (run + c[i] == (unsigned)remaining);
              break;
            }
            run += c[i];
          }
        }
      }
      __syncthreads();
      prefix |= (uint64_t)sh_digit << shift;
      pmask |= (uint64_t)0xFF << shift;
      remaining = sh_rem;
      if (sh_done) break;
    }
    {
      // keys > v* are in; the first `remaining` keys == v* (ascending index) too
      const int64_t chunk = (M + RT - 1) / RT;
      const int64_t lo = threadIdx.x * chunk, hi = min(lo + chunk, M);
      int eq = 0;
      // keys compared on the resolved digits only (all of them unless the
      // boundary bin was taken whole, where ties below cannot matter)
      for (int64_t m = lo; m < hi; ++m) eq += ((uint64_t)__double_as_longlong(ap[m]) & pmask) == prefix;
      int tot_eq;
      int rank = block_excl_scan(eq, scan_tmp, &tot_eq);
      for (int64_t m = lo; m < hi; ++m) {
        const uint64_t key = (uint64_t)__double_as_longlong(ap[m]) & pmask;
        if (key > prefix || (key == prefix && rank++ < remaining)) bits[m] = BIT_IMPORTANCE;
      }
    }
    __syncthreads();
    if (P.p > 0.0) {
      // sequential cumsum of the top-K in sorted order (masks.py:99): gather, sort, sum
      int kp2 = 1;
      while (kp2 < K) kp2 <<= 1;
      const int64_t chunk = (M + RT - 1) / RT;
      const int64_t lo = threadIdx.x * chunk, hi = min(lo + chunk, M);
      int mine = 0;
      for (int64_t m = lo; m < hi; ++m) mine += bits[m] & BIT_IMPORTANCE ? 1 : 0;
      int tot_k;
      int off = block_excl_scan(mine, scan_tmp, &tot_k);
      for (int64_t m = lo; m < hi; ++m)
        if (bits[m] & BIT_IMPORTANCE) { sv[off] = ap[m]; si[off] = (int)m; ++off; }
      for (int i = tot_k + threadIdx.x; i < kp2; i += RT) { sv[i] = -1.0; si[i] = 0x7fffffff; }
      __syncthreads();
      bitonic_sort(sv, si, kp2);
      if (threadIdx.x == 0) sh_count = seq_first_reach(sv, (int)K, P.p) ? 0 : 1;
      __syncthreads();
      need_full_sort = sh_count != 0;
    }
    }
    if (need_full_sort) {
      for (int i = threadIdx.x; i < P.p2; i += RT) {
        sv[i] = i < M ? ap[i] : -1.0;
        si[i] = i < M ? i : 0x7fffffff;
      }
      for (int64_t m = threadIdx.x; m < M; m += RT) bits[m] = 0;
      __syncthreads();
      bitonic_sort(sv, si, P.p2);
      if (threadIdx.x == 0) {
        // sequential cumsum in sorted order, exactly as numpy.cumsum (masks.py:99-102)
        const int reach = seq_first_reach(sv, (int)M, P.p);
        const int64_t first_p = reach ? reach : M;
        int64_t count = first_p > P.k_floor ? first_p : P.k_floor;
        count = count < 1 ? 1 : (count > M ? M : count);
        sh_count = (int)count;
      }
      __syncthreads();
      for (int i = threadIdx.x; i < sh_count; i += RT) bits[si[i]] = BIT_IMPORTANCE;
      __syncthreads();
    }
    for (int64_t m = threadIdx.x; m < M; m += RT) {
      uint8_t b = bits[m];
      const int64_t dist = m > n ? m - n : n - m;
      if (dist <= P.radius) b |= BIT_ADJ;
      if ((b & (BIT_IMPORTANCE | BIT_ADJ)) || (P.force_text && M > N && m >= N)) b |= BIT_MASK;
      bits[m] = b;
    }
  }
  __syncthreads();

  // ---- R = 1 - excluded mass (rectify.py:56-63) ----
  double ex = 0.0;
  for (int64_t m = threadIdx.x; m < M; m += RT) ex += (bits[m] & BIT_MASK) ? 0.0 : ap[m];
  const double R = 1.0 - block_sum(ex, red);

  // ---- GAPR gate: gain vs first-order error (masks.py:138-186) ----
  const bool deficit = ws.status[ST_DEFICIT] != 0;
  const int64_t d = g.d;
  for (int64_t m = threadIdx.x; m < M; m += RT) {
    const double len = (double)kv_len(g, m);
    const double bq = (double)q_len(g, n);   // query block tokens (masks.py:146: B)
    const double s = (m < N) ? srow[m] : srow[N + Tt + (m - N)];
    const double gain = fabs((bq * len) * s);
    double err = 0.0;
    if (deficit) {
      const int64_t krow = (m < N) ? m : N + Tt + (m - N);
      const double* kp = ws.k_cat + (h * n_cols + krow) * d;
      const double* kd = ws.k_def + (h * M + m) * d;
      const double* qp = ws.q_pool + (h * N + n) * d;
      const double* qd = ws.q_def + (h * N + n) * d;
      double d1 = 0.0, d2 = 0.0;
      for (int64_t c = 0; c < d; ++c) { d1 = fma(qd[c], kp[c], d1); d2 = fma(qp[c], kd[c], d2); }
      const double t1 = (d1 * len) * P.inv_sqrt_d;
      const double t2 = (bq * d2) * P.inv_sqrt_d;
      err = fabs(t1 + t2);
    }
    uint8_t b = bits[m];
    if (gain > err) b |= BIT_COMP;
    const bool masked = b & BIT_MASK;
    bool applied = false;
    if (P.variant == RSA_VARIANT_SPARSE_RECTIFIED) applied = !masked && (b & BIT_COMP);
    else if (P.variant == RSA_VARIANT_COMPENSATE_ALL) applied = !masked;
    if (applied) b |= BIT_APPLIED;
    bits[m] = b;
  }
  __syncthreads();
  uint8_t* bits_out = ws.mask_bits + (h * N + n) * M;
  double* applied_out = ws.a_applied + (h * N + n) * M;   // operand of the compensation GEMM
  for (int64_t m = threadIdx.x; m < M; m += RT) {
    bits_out[m] = bits[m];
    applied_out[m] = (bits[m] & BIT_APPLIED) ? ap[m] : 0.0;
  }
  if (threadIdx.x == 0) {
    ws.r[h * N + n] = R;
    const bool rect = P.variant == RSA_VARIANT_SPARSE_RECTIFIED ||
                      P.variant == RSA_VARIANT_SPARSE_RECTIFIED_NO_GAPR ||
                      P.variant == RSA_VARIANT_COMPENSATE_ALL;
    ws.r_eff[h * N + n] = rect ? (float)R : 1.0f;
  }

  // ---- ascending kv list (kernel.py:92 np.flatnonzero) ----
  const int64_t chunk = (M + RT - 1) / RT;
  const int64_t lo = threadIdx.x * chunk, hi = min(lo + chunk, M);
  int local = 0;
  for (int64_t m = lo; m < hi; ++m) local += (bits[m] & BIT_MASK) ? 1 : 0;
  int total;
  int off = block_excl_scan(local, scan_tmp, &total);
  int32_t* list = ws.kv_list + (h * N + n) * M;
  for (int64_t m = lo; m < hi; ++m)
    if (bits[m] & BIT_MASK) list[off++] = (int32_t)m;
  if (threadIdx.x == 0) {
    ws.kv_count[h * N + n] = total;
    if (total == 0) atomicOr(ws.status + ST_EMPTY_ROW, 1);
  }
}

// ----------------------------------------------------------------------------
// Register-resident select_rows (n_cols <= RT * PER, p == 0): same arithmetic,
// element for element, as select_rows_kernel, with 32-bit indices, the row in
// registers (strided for the softmax, blocked for the selection so ascending
// index order is thread order), shuffle scans and one barrier per reduction.
// ----------------------------------------------------------------------------
constexpr int NW = RT / 32;

template <typename F>
__device__ __forceinline__ double block_reduce(double x, double* slot, F op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = op(x, __shfl_xor_sync(0xffffffffu, x, o));
  if ((threadIdx.x & 31) == 0) slot[threadIdx.x >> 5] = x;
  __syncthreads();
  double y = slot[0];
#pragma unroll
  for (int w = 1; w < NW; ++w) y = op(y, slot[w]);
  return y;
}

// exclusive prefix of x over the block in thread order; *total = sum
__device__ __forceinline__ int block_scan(int x, int* slot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) slot[warp] = incl;
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int c = slot[w];
    before += w < warp ? c : 0;
    all += c;
  }
  *total = all;
  return before + incl - x;
}

// resident CTAs per SM the register budget is held to (8 at PER <= 10: measured
// 1.07 vs 1.46 ms for the whole K2 at HunyuanVideo size with the compiler's 96 registers)
constexpr int sel_min_blocks(int per) { return per <= 10 ? 8 : per <= 12 ? 6 : 4; }

// CUM: the cumulative-weight rule is on (p > 0).  The top-K found by the radix
// select already satisfies it when its sum clears p by more than any summation
// order can move it (K * eps relative); otherwise the row is sorted in shared
// memory and the sequential cumsum decides the count exactly (masks.py:99-103).
template <int PER, bool CUM>
__global__ void __launch_bounds__(RT, sel_min_blocks(PER)) select_rows_reg_kernel(SelectParams P) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int N = (int)P.g.N, M = (int)P.g.M, Tt = (int)P.g.Tt, n_cols = (int)P.g.n_cols;
  const int B = (int)P.g.B, n_text = (int)P.g.n_text;
  const int n_mix = N + Tt;
  const int n = blockIdx.x, h = blockIdx.y;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const size_t row = (size_t)h * N + n;
  double* sc = reinterpret_cast<double*>(smem_raw);   // [n_cols] scores / sqrt(d)
  double* sa = sc + n_cols;                            // [n_mix] a_hat
  double* at = sa + n_mix;                             // [n_text] text a_pool columns
  uint8_t* sb = reinterpret_cast<uint8_t*>(at + n_text);  // [M] mask bits
  // CUM only: [p2] sort values, [p2] sort indices, [M] importance flags
  double* sv = reinterpret_cast<double*>(((uintptr_t)(sb + M) + 15) & ~(uintptr_t)15);
  int* si = reinterpret_cast<int*>(sv + P.p2);
  uint8_t* simp = reinterpret_cast<uint8_t*>(si + P.p2);
  __shared__ double red[7][NW];
  __shared__ int sh_count;
  __shared__ int ired[2][NW];
  __shared__ unsigned hist[2][256];
  __shared__ unsigned long long s_and[NW], s_or[NW];
  __shared__ int sh_digit, sh_rem, sh_done;

  for (int k = t; k < 256; k += RT) hist[0][k] = 0u;

  // ---- scores / sqrt(d) and the IPAR softmax (ipar.py:36-42), strided ----
  double* srow = P.ws.scores + row * n_cols;
  double v[PER];
  double mx = -DBL_MAX;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = t + i * RT;
    v[i] = 0.0;
    if (j < n_cols) {
      const double s = srow[j] / P.sqrt_d;
      srow[j] = s;
      sc[j] = s;
      v[i] = s;
      if (j < n_mix) mx = fmax(mx, s);
    }
  }
  mx = block_reduce(mx, red[0], [](double a, double b) { return fmax(a, b); });
  double part = 0.0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int j = t + i * RT;
    if (j < n_mix) { v[i] = exp(v[i] - mx); part += v[i]; }
  }
  const auto add = [](double a, double b) { return a + b; };
  const double tot = block_reduce(part, red[1], add);
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (t + i * RT < n_mix) v[i] = v[i] / tot;
  // ---- reallocation (ipar.py:45-66) ----
  if (Tt > 0 && B > 1) {
    const int q_last = (int)P.g.q_last;
    const bool ragged = q_last != B;   // see select_rows_kernel
    double pv = 0.0, pt = 0.0, pl = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = t + i * RT;
      if (ragged && j == N - 1) pl = v[i];
      else if (j < N) pv += v[i];
      else if (j < n_mix) pt += v[i];
    }
    const double sum_v = block_reduce(pv, red[2], add);
    const double sum_t = block_reduce(pt, red[3], add);
    double D;
    if (ragged) {
      const double a_last = block_reduce(pl, red[5], add);   // one non-zero term: exact
      D = ((double)B * sum_v + (double)q_last * a_last) + sum_t;
    } else {
      D = (double)B * sum_v + sum_t;
    }
    if (D <= 0.0 && t == 0) atomicOr(P.ws.status + ST_DEGENERATE, 1);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int j = t + i * RT;
      if (j < n_mix) v[i] = (j < N) ? ((double)(j == N - 1 ? q_last : B) * v[i]) / D : v[i] / D;
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (t + i * RT < n_mix) sa[t + i * RT] = v[i];
  __syncthreads();
  // ---- text re-aggregation (ipar.py:76-83): one warp per text block ----
  for (int jt = warp; jt < n_text; jt += NW) {
    const int lo = N + jt * B, hi = min(lo + B, n_mix);
    double pj = 0.0;
    for (int i = lo + lane; i < hi; i += 32) pj += sa[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pj += __shfl_xor_sync(0xffffffffu, pj, o);
    if (lane == 0) at[jt] = pj;
  }
  __syncthreads();
  double* ap_out = P.ws.a_pool + row * M;
  for (int m = t; m < M; m += RT) ap_out[m] = m < N ? sa[m] : at[m - N];

  // ---- the a_pool row, blocked: thread t owns m = t * PER + i ----
  const int m0 = t * PER;
  double a[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int m = m0 + i;
    a[i] = m < M ? (m < N ? sa[m] : at[m - N]) : 0.0;
  }
  uint8_t b[PER];
  if (P.variant == RSA_VARIANT_FULL) {
#pragma unroll
    for (int i = 0; i < PER; ++i) b[i] = BIT_MASK | BIT_IMPORTANCE;
  } else {
    // exact top-K by MSB-first radix select on the fp64 bit patterns, ties by
    // ascending index (see select_rows_kernel)
    const int K = (int)(P.k_floor < M ? P.k_floor : M);
    uint64_t k_and = ~0ull, k_or = 0ull;
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (m0 + i < M) {
        const uint64_t key = (uint64_t)__double_as_longlong(a[i]);
        k_and &= key;
        k_or |= key;
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      k_and &= __shfl_xor_sync(0xffffffffu, k_and, o);
      k_or |= __shfl_xor_sync(0xffffffffu, k_or, o);
    }
    if (lane == 0) { s_and[warp] = k_and; s_or[warp] = k_or; }
    __syncthreads();
    k_and = ~0ull;
    k_or = 0ull;
#pragma unroll
    for (int w = 0; w < NW; ++w) { k_and &= s_and[w]; k_or |= s_or[w]; }
    const uint64_t differ = k_and ^ k_or;
    int top = 56;
    while (top > 0 && ((differ >> top) & 0xFF) == 0) top -= 8;
    uint64_t prefix = 0, pmask = 0;
    if (top < 56) {
      pmask = ~0ull << (top + 8);
      prefix = k_and & pmask;
    }
    int remaining = K, hb = 0;
    for (int shift = top; shift >= 0; shift -= 8) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const uint64_t key = (uint64_t)__double_as_longlong(a[i]);
        if (m0 + i < M && (key & pmask) == prefix) atomicAdd(&hist[hb][(key >> shift) & 0xFF], 1u);
      }
      for (int k = t; k < 256; k += RT) hist[hb ^ 1][k] = 0u;   // next pass's bins
      __syncthreads();
      if (warp == 0) {
        unsigned c[8], cnt = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) { c[i] = hist[hb][255 - 8 * lane - i]; cnt += c[i]; }
        unsigned incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const unsigned excl = incl - cnt;
        if (excl < (unsigned)remaining && incl >= (unsigned)remaining) {
          unsigned run = excl;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (run + c[i] >= (unsigned)remaining) {
              sh_digit = 255 - 8 * lane - i;
              sh_rem = remaining - (int)run;
              sh_done = (run + c[i] == (unsigned)remaining);
              break;
            }
            run += c[i];
          }
        }
      }
      __syncthreads();
      prefix |= (uint64_t)sh_digit << shift;
      pmask |= (uint64_t)0xFF << shift;
      remaining = sh_rem;
      hb ^= 1;
      if (sh_done) break;
    }
    // keys > v* are in; the first `remaining` keys == v* in ascending index too
    int eq = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i)
      eq += (m0 + i < M && ((uint64_t)__double_as_longlong(a[i]) & pmask) == prefix) ? 1 : 0;
    int tot_eq;
    int rank = block_scan(eq, ired[0], &tot_eq);
    bool sel[PER];
    double top_sum = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int m = m0 + i;
      const uint64_t key = (uint64_t)__double_as_longlong(a[i]) & pmask;
      sel[i] = false;
      if (m < M) sel[i] = key > prefix || (key == prefix && rank++ < remaining);
      top_sum += sel[i] ? a[i] : 0.0;
    }
    if (CUM) {
      const double S = block_reduce(top_sum, red[6], [](double x, double y) { return x + y; });
      if (!(S - 4.0 * (double)K * DBL_EPSILON * S >= P.p)) {
        // p may bind: sort the whole row (value desc, index asc) and take the
        // sequential cumsum, as the general kernel does
        for (int j = t; j < P.p2; j += RT) {
          const int src = j;
          sv[j] = src < M ? (src < N ? sa[src] : at[src - N]) : -1.0;
          si[j] = src < M ? src : 0x7fffffff;
        }
        for (int j = t; j < M; j += RT) simp[j] = 0;
        __syncthreads();
        bitonic_sort(sv, si, P.p2);
        if (t == 0) {
          const int reach = seq_first_reach(sv, M, P.p);
          const int first_p = reach ? reach : M;
          int count = first_p > K ? first_p : K;
          sh_count = count < 1 ? 1 : (count > M ? M : count);
        }
        __syncthreads();
        for (int j = t; j < sh_count; j += RT) simp[si[j]] = 1;
        __syncthreads();
#pragma unroll
        for (int i = 0; i < PER; ++i) sel[i] = m0 + i < M && simp[m0 + i];
      }
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int m = m0 + i;
      uint8_t bb = sel[i] ? BIT_IMPORTANCE : 0;
      const int dist = m > n ? m - n : n - m;
      if (dist <= P.radius) bb |= BIT_ADJ;
      if ((bb & (BIT_IMPORTANCE | BIT_ADJ)) || (P.force_text && M > N && m >= N)) bb |= BIT_MASK;
      b[i] = bb;
    }
  }

  // ---- R = 1 - excluded mass (rectify.py:56-63) ----
  double ex = 0.0;
#pragma unroll
  for (int i = 0; i < PER; ++i) ex += (m0 + i < M && !(b[i] & BIT_MASK)) ? a[i] : 0.0;
  const double R = 1.0 - block_reduce(ex, red[4], add);

  // ---- GAPR gate (masks.py:138-186) ----
  const bool deficit = P.ws.status[ST_DEFICIT] != 0;
  const int d = (int)P.g.d;
  const double bq = (double)q_len(P.g, n);   // query block tokens (masks.py:146: B)
  int kv_local = 0;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int m = m0 + i;
    if (m >= M) continue;
    const double len = (double)kv_len(P.g, m);
    const double s = (m < N) ? sc[m] : sc[N + Tt + (m - N)];
    const double gain = fabs((bq * len) * s);
    double err = 0.0;
    if (deficit) {
      const int krow = (m < N) ? m : N + Tt + (m - N);
      const double* kp = P.ws.k_cat + ((size_t)h * n_cols + krow) * d;
      const double* kd = P.ws.k_def + ((size_t)h * M + m) * d;
      const double* qp = P.ws.q_pool + row * d;
      const double* qd = P.ws.q_def + row * d;
      double d1 = 0.0, d2 = 0.0;
      for (int c = 0; c < d; ++c) { d1 = fma(qd[c], kp[c], d1); d2 = fma(qp[c], kd[c], d2); }
      const double t1 = (d1 * len) * P.inv_sqrt_d;
      const double t2 = (bq * d2) * P.inv_sqrt_d;
      err = fabs(t1 + t2);
    }
    uint8_t bb = b[i];
    if (gain > err) bb |= BIT_COMP;
    const bool masked = bb & BIT_MASK;
    bool applied = false;
    if (P.variant == RSA_VARIANT_SPARSE_RECTIFIED) applied = !masked && (bb & BIT_COMP);
    else if (P.variant == RSA_VARIANT_COMPENSATE_ALL) applied = !masked;
    if (applied) bb |= BIT_APPLIED;
    sb[m] = bb;
    kv_local += masked ? 1 : 0;
    b[i] = bb;
  }
  // ---- ascending kv list (kernel.py:92 np.flatnonzero) ----
  int total;
  int off = block_scan(kv_local, ired[1], &total);   // its barrier also publishes sb
  int32_t* list = P.ws.kv_list + row * M;
#pragma unroll
  for (int i = 0; i < PER; ++i)
    if (m0 + i < M && (b[i] & BIT_MASK)) list[off++] = m0 + i;
  uint8_t* bits_out = P.ws.mask_bits + row * M;
  double* applied_out = P.ws.a_applied + row * M;   // operand of the compensation GEMM
  for (int m = t; m < M; m += RT) {
    const uint8_t bb = sb[m];
    bits_out[m] = bb;
    applied_out[m] = (bb & BIT_APPLIED) ? (m < N ? sa[m] : at[m - N]) : 0.0;
  }
  if (t == 0) {
    P.ws.r[row] = R;
    const bool rect = P.variant == RSA_VARIANT_SPARSE_RECTIFIED ||
                      P.variant == RSA_VARIANT_SPARSE_RECTIFIED_NO_GAPR ||
                      P.variant == RSA_VARIANT_COMPENSATE_ALL;
    P.ws.r_eff[row] = rect ? (float)R : 1.0f;
    P.ws.kv_count[row] = total;
    if (total == 0) atomicOr(P.ws.status + ST_EMPTY_ROW, 1);
  }
}

// kv lists from an explicit caller mask (kernel-only seam)
__global__ void __launch_bounds__(RT) lists_from_mask_kernel(const uint8_t* __restrict__ mask,
                                                             Workspace ws, Geometry g) {
  __shared__ int scan_tmp[RT];
  const int64_t n = blockIdx.x, h = blockIdx.y, M = g.M;
  const uint8_t* row = mask + (h * g.N + n) * M;
  uint8_t* bits_out = ws.mask_bits + (h * g.N + n) * M;
  const int64_t chunk = (M + RT - 1) / RT;
  const int64_t lo = threadIdx.x * chunk, hi = min(lo + chunk, M);
  int local = 0;
  for (int64_t m = lo; m < hi; ++m) {
    const bool on = row[m] != 0;
    bits_out[m] = on ? BIT_MASK : 0;
    local += on;
  }
  int total;
  int off = block_excl_scan(local, scan_tmp, &total);
  int32_t* list = ws.kv_list + (h * g.N + n) * M;
  for (int64_t m = lo; m < hi; ++m)
    if (row[m]) list[off++] = (int32_t)m;
  if (threadIdx.x == 0) {
    ws.kv_count[h * g.N + n] = total;
    ws.r_eff[h * g.N + n] = 1.0f;
    if (total == 0) atomicOr(ws.status + ST_EMPTY_ROW, 1);
  }
}

// Per 128-row tcgen05 tile: union of the G = 128/B member query blocks' kv
// lists, ascending, each entry (kv id | member-bit mask << 24).  One warp per tile.
__global__ void tile_lists_kernel(Workspace ws, Geometry g) {
  const int G = (int)(kTcTileRows / g.B);
  const int64_t tiles_per_head = (g.N + G - 1) / G;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (warp >= tiles_per_head * g.H) return;
  const int64_t h = warp / tiles_per_head, t = warp % tiles_per_head;
  const int gcount = (int)min((int64_t)G, g.N - t * G);
  const uint8_t* rows = ws.mask_bits + (h * g.N + t * G) * g.M;
  int32_t* out = ws.tile_list + (h * tiles_per_head + t) * g.M;
  int count = 0;
  for (int64_t m0 = 0; m0 < g.M; m0 += 32) {
    const int64_t m = m0 + lane;
    uint32_t member = 0;
    if (m < g.M)
      for (int gg = 0; gg < gcount; ++gg) member |= (rows[gg * g.M + m] & BIT_MASK) ? (1u << gg) : 0u;
    const uint32_t ballot = __ballot_sync(0xffffffffu, member != 0);
    if (member) out[count + __popc(ballot & ((1u << lane) - 1))] = (int32_t)(m | (member << 24));
    count += __popc(ballot);
  }
  if (lane == 0) ws.tile_count[h * tiles_per_head + t] = count;
}

}  // namespace

cudaError_t launch_select(const Geometry& g, const rsa_config& cfg, int64_t k_floor,
                          const Workspace& ws, cudaStream_t st, int* launches) {
  const double sqrt_d = sqrt((double)g.d);
  // scores = q_pool @ k_cat^T (select_rows divides by sqrt(d), ipar.py:41):
  // [N][n_cols] per head, our DMMA GEMM
  cudaError_t e = launch_dgemm(g.H, g.N, g.n_cols, g.d, ws.q_pool, g.d, g.N * g.d, ws.k_cat, g.d,
                               g.n_cols * g.d, true, ws.scores, g.n_cols, g.N * g.n_cols, st);
  if (e != cudaSuccess) return e;
  ++*launches;
  SelectParams P;
  P.g = g;
  P.ws = ws;
  P.p = cfg.weight_threshold;
  P.k_floor = k_floor;
  P.radius = cfg.adjacency_radius;
  P.force_text = cfg.force_text_blocks;
  P.variant = cfg.variant;
  P.inv_sqrt_d = 1.0 / sqrt_d;
  P.sqrt_d = sqrt_d;
  int p2 = 1;
  while (p2 < g.M) p2 <<= 1;
  P.p2 = p2;
  P.use_sort = 0;   // radix select (a full bitonic sort of every row measured 2x slower)
  // the register-resident kernel covers rows up to 16 * RT columns; wider
  // rows take the general shared-memory kernel
  const int per = (int)((g.n_cols + RT - 1) / RT);
  const bool cum = P.p > 0.0;
  const bool reg = !P.use_sort && per <= 16;
  if (reg) {
    size_t smem = (size_t)(g.n_cols + g.N + g.Tt + g.n_text) * 8 + (size_t)g.M + 16;
    if (cum) smem += 16 + (size_t)p2 * 12 + (size_t)g.M;
    auto launch = [&](auto kern) -> cudaError_t {
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
      }
      kern<<<dim3((unsigned)g.N, (unsigned)g.H), RT, smem, st>>>(P);
      return cudaSuccess;
    };
    if (cum)
      e = per <= 4 ? launch(select_rows_reg_kernel<4, true>)
        : per <= 8 ? launch(select_rows_reg_kernel<8, true>)
        : per <= 10 ? launch(select_rows_reg_kernel<10, true>)
        : per <= 12 ? launch(select_rows_reg_kernel<12, true>)
        : launch(select_rows_reg_kernel<16, true>);
    else
      e = per <= 4 ? launch(select_rows_reg_kernel<4, false>)
        : per <= 6 ? launch(select_rows_reg_kernel<6, false>)
        : per <= 8 ? launch(select_rows_reg_kernel<8, false>)
        : per <= 10 ? launch(select_rows_reg_kernel<10, false>)
        : per <= 12 ? launch(select_rows_reg_kernel<12, false>)
        : launch(select_rows_reg_kernel<16, false>);
    if (e != cudaSuccess) return e;
  } else {
    const size_t sa_len = std::max<size_t>((size_t)(g.N + g.Tt), (size_t)p2);
    const size_t smem = sa_len * 8 + (size_t)g.M * 8 + (size_t)p2 * 4 + (size_t)g.M + 16;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(select_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    select_rows_kernel<<<dim3((unsigned)g.N, (unsigned)g.H), RT, smem, st>>>(P);
  }
  ++*launches;
  // compensation rows: (a_pool masked to applied) @ v_pool (rectify.py:84-87);
  // select_rows wrote the masked operand.  [N][d] per head
  e = launch_dgemm(g.H, g.N, g.d, g.M, ws.a_applied, g.M, g.N * g.M, ws.v_pool, g.d, g.M * g.d, false,
                   ws.comp, g.d, g.N * g.d, st);
  if (e != cudaSuccess) return e;
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_lists_from_mask(const Geometry& g, const uint8_t* mask, const Workspace& ws,
                                   cudaStream_t st, int* launches) {
  lists_from_mask_kernel<<<dim3((unsigned)g.N, (unsigned)g.H), RT, 0, st>>>(mask, ws, g);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_tile_lists(const Geometry& g, const Workspace& ws, cudaStream_t st,
                              int* launches) {
  // B = 128: a 128-row tile is one query block, K3 walks its kv list directly
  if (g.B == kTcTileRows) return cudaSuccess;
  const int64_t G = kTcTileRows / g.B;
  const int64_t tiles = g.H * ((g.N + G - 1) / G);
  const int64_t threads = tiles * 32;
  tile_lists_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(ws, g);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace rsa
