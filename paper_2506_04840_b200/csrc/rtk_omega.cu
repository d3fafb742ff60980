// Appendix D sketch types: a uniform U[-1, 1] Omega_k and the Khatri-Rao
// products of standard Gaussian / uniform matrices, materialised row-major ([j][l], fp32) for the
// sketch kernels (rtk_tile.cu, rtk_tc.cu, rtk_fused.cu read it through sketch_pair()).
//
// Frozen generators (readings C2, C19; the oracle implements the same written spec in
// oracle/gauss.py, no shared code):
//   RTK-UNIF-1  Philox4x32-10 on counter (c/4, lo32 j, hi32 j, 0x55000000 | k), key (lo32 seed,
//               hi32 seed); word t -> column 4 (c/4) + t:  2u - 1 = (2 (x >> 8) + 1 - 2^24) 2^-24
//   RTK-KR-1    Omega_k(j, c) = fl32( prod_{m != k, ascending} F_m(i_m, c) ), product in binary64,
//               j = sum_m i_m stride_m over the column modes (lower modes fastest);
//               F_m (n_m x l) drawn like Omega with counter word 3 = 0x4B000000 | (m << 8) | k
//               (Gaussian: RTK-GAUSS-2 pairs) or 0x4C000000 | (m << 8) | k (uniform: RTK-UNIF-1).
// The Gaussian Khatri-Rao factors are tiny (sum n_m l values), so the per-element cost is d - 1
// table reads and products instead of a Philox block and a Box-Muller transform.
#include <cuda_runtime.h>

#include <algorithm>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"

namespace rtk {
namespace {

constexpr int kMaxF = 7;   // d <= 8: at most 7 column modes

struct KrSpec {
  int nf;                      // column modes (d - 1)
  int64_t ext[kMaxF];          // their extents, fastest first
  int64_t off[kMaxF];          // offsets of their tables in tabs ([i][l] row-major)
};

// F(i, c) for rows i < n, columns c < l of one Philox stream (word3), [i][l] row-major
__global__ void kr_factor_kernel(uint64_t seed, uint32_t word3, int uniform, int64_t n, int l,
                                 float* __restrict__ out) {
  const int n4 = (l + 3) / 4;
  const int64_t tot = n * n4;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < tot; it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = it / n4;
    const int c4 = (int)(it - i * n4);
    const uint4 x = omega_bits(seed, word3, (uint64_t)i, (uint32_t)c4);
    float z[4];
    if (uniform) {
      z[0] = unif_sym(x.x); z[1] = unif_sym(x.y); z[2] = unif_sym(x.z); z[3] = unif_sym(x.w);
    } else {
      const float2 a = box_muller(x.x, x.y), b = box_muller(x.z, x.w);
      z[0] = a.x; z[1] = a.y; z[2] = b.x; z[3] = b.y;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * c4 + t < l) out[i * l + 4 * c4 + t] = z[t];
  }
}

// rows [row0, row0 + rows) of Omega_k: kind 1 uniform (Philox in place), 2/3 Khatri-Rao (tables)
__global__ void omega_fill_kernel(int kind, uint64_t seed, uint32_t mode1, int64_t row0, int64_t rows, int l,
                                  KrSpec kr, const float* __restrict__ tabs, float* __restrict__ out) {
  const int n4 = (l + 3) / 4;
  const int64_t tot = rows * n4;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < tot; it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jr = it / n4;
    const int c4 = (int)(it - jr * n4);
    const int64_t j = row0 + jr;
    float z[4];
    if (kind == 1) {
      const uint4 x = omega_bits(seed, 0x55000000u | mode1, (uint64_t)j, (uint32_t)c4);
      z[0] = unif_sym(x.x); z[1] = unif_sym(x.y); z[2] = unif_sym(x.z); z[3] = unif_sym(x.w);
    } else {
      double p[4] = {1.0, 1.0, 1.0, 1.0};
      int64_t rest = j;
      for (int f = 0; f < kr.nf; ++f) {
        const int64_t i = rest % kr.ext[f];
        rest /= kr.ext[f];
        const float* row = tabs + kr.off[f] + i * l + 4 * c4;
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * c4 + t < l) p[t] = __dmul_rn(p[t], (double)row[t]);
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) z[t] = __double2float_rn(p[t]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (4 * c4 + t < l) out[jr * l + 4 * c4 + t] = z[t];
  }
}

}  // namespace

size_t sketch_tab_floats(const int64_t* dims, int d, int mode1, int l) {
  size_t s = 0;
  for (int m = 0; m < d; ++m)
    if (m + 1 != mode1) s += (size_t)dims[m] * l;
  return s;
}

cudaError_t sketch_materialize(int kind, uint64_t seed, int mode1, const int64_t* dims, int d, int64_t row0,
                               int64_t rows, int l, float* tabs, float* out, cudaStream_t st) {
  if (kind < 1 || kind > 3 || d < 2 || d > kMaxF + 1 || mode1 < 1 || mode1 > d) return cudaErrorInvalidValue;
  KrSpec kr = {};
  if (kind >= 2) {
    int64_t off = 0;
    for (int m = 0; m < d; ++m) {
      if (m + 1 == mode1) continue;
      const uint32_t w3 = (kind == 3 ? 0x4C000000u : 0x4B000000u) | ((uint32_t)(m + 1) << 8) | (uint32_t)mode1;
      const int64_t n4 = (int64_t)dims[m] * ((l + 3) / 4);
      kr_factor_kernel<<<(unsigned)std::min<int64_t>((n4 + 255) / 256, 4096), 256, 0, st>>>(
          seed, w3, kind == 3 ? 1 : 0, dims[m], l, tabs + off);
      kr.ext[kr.nf] = dims[m];
      kr.off[kr.nf] = off;
      ++kr.nf;
      off += (int64_t)dims[m] * l;
    }
  }
  const int64_t tot = rows * ((l + 3) / 4);
  if (tot > 0)
    omega_fill_kernel<<<(unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 64), 256, 0, st>>>(
        kind, seed, (uint32_t)mode1, row0, rows, l, kr, tabs, out);
  return cudaGetLastError();
}

}  // namespace rtk
