// Token reordering for the permuted (Morton) problem.
//
// Reference: morton_code_3d / morton_permutation / reorder_morton /
// inverse_permutation (pkg/src/rectattn/core.py:263-325) and the harness's
// `morton_reorder` option (harness.py:172-173), which runs the pipeline on the
// reordered problem.  The permutation depends only on the grid, so it is built
// once on the host (std::stable_sort of the codes == numpy's stable argsort);
// the row moves run on the device.  rsa_forward_permuted fuses the moves into
// K1 (gather + permuted K/V write) and the K3 epilogue (scatter) instead.
#include "rsa_internal.cuh"

#include <algorithm>
#include <numeric>
#include <vector>

namespace rsa {
namespace {

uint64_t part1by2(uint64_t n) {   // core.py:266-273
  n &= 0x1FFFFF;
  n = (n | (n << 32)) & 0x1F00000000FFFFull;
  n = (n | (n << 16)) & 0x1F0000FF0000FFull;
  n = (n | (n << 8)) & 0x100F00F00F00F00Full;
  n = (n | (n << 4)) & 0x10C30C30C30C30C3ull;
  n = (n | (n << 2)) & 0x1249249249249249ull;
  return n;
}

// dst row r <- src row perm[r] (inverse: dst row perm[r] <- src row r) for the
// video rows of every head; text rows copied.  One warp per row, 16-byte moves.
__global__ void permute_rows_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                    const int32_t* __restrict__ perm, int64_t H, int64_t T, int64_t Tv,
                                    int64_t row_vec, int inverse) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (warp >= H * T) return;
  const int64_t h = warp / T, r = warp % T;
  int64_t from = r, to = r;
  if (r < Tv) {
    if (inverse) to = perm[r];
    else from = perm[r];
  }
  const uint4* s = src + (h * T + from) * row_vec;
  uint4* d = dst + (h * T + to) * row_vec;
  for (int64_t i = lane; i < row_vec; i += 32) d[i] = s[i];
}

}  // namespace

void morton_permutation_host(int64_t t, int64_t h, int64_t w, int32_t* perm) {
  const int64_t n = t * h * w;
  std::vector<uint64_t> codes((size_t)n);
  int64_t i = 0;
  for (int64_t tt = 0; tt < t; ++tt)
    for (int64_t yy = 0; yy < h; ++yy)
      for (int64_t xx = 0; xx < w; ++xx)   // core.py:279-281 row-major, w fastest
        codes[(size_t)i++] = (part1by2((uint64_t)tt) << 2) | (part1by2((uint64_t)yy) << 1) | part1by2((uint64_t)xx);
  std::vector<int32_t> idx((size_t)n);
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) { return codes[(size_t)a] < codes[(size_t)b]; });
  std::copy(idx.begin(), idx.end(), perm);
}

cudaError_t launch_permute_rows(const Geometry& g, const int32_t* perm, const void* src, void* dst, bool inverse,
                                cudaStream_t st) {
  const size_t esz = g.dtype == RSA_BF16 ? 2 : g.dtype == RSA_F32 ? 4 : 8;
  const size_t row_bytes = (size_t)g.d * esz;
  if (row_bytes % 16 || (uintptr_t)src % 16 || (uintptr_t)dst % 16) return cudaErrorInvalidValue;
  const int64_t rows = g.H * g.T;
  const int64_t threads = rows * 32;
  permute_rows_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      static_cast<const uint4*>(src), static_cast<uint4*>(dst), perm, g.H, g.T, g.Tv, (int64_t)(row_bytes / 16),
      inverse ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace rsa
