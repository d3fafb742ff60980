// rtk_solve.cu -- low-latency float64 "small solves" of one sketch / power step, l <= 64.
//
// After a streaming kernel has produced per-CTA fp32 partial sums of M (M^T Q) (or M Omega_k),
// one step of Alg. 3/4 finishes in TWO launches:
//
//   reduce_gram_kernel  (whole GPU, 8 rows per CTA, 512 threads)
//       Y = sum_g Ypart[g] - alpha Q           fixed g order, fp64 (Alg. 3/4 line 7's "- alpha Q")
//       per-block packed upper Gram  Y_b^T Y_b
//   step_kernel         (one thread-block cluster of C <= 8 CTAs, 256 threads each)
//       G = sum_b Gram_b                        (cluster-parallel sum, fixed order)
//       every CTA redundantly (identical inputs -> identical results) factors the l x l G:
//         span path   (sketch / non-final power step):  G = R^T R, T = R^{-1};
//                      a second CholQR pass only if eps * kappa_F(R)^2 > 1e-7 (C20)
//         shift       (power steps): Sigma_ll = sqrt(lambda_min(G)) by Householder
//                      tridiagonalisation + Sturm multisection; alpha <- (Sigma_ll + alpha)/2
//                      if Sigma_ll > alpha (degenerate guard SPEC.md:347)
//         eigen path  (final step, or Cholesky breakdown): G = V Lambda V^T via tridiagonalisation,
//                      all-eigenvalue Sturm bisection, inverse iteration and back-transformation;
//                      T = V Lambda^{-1/2} in descending order (left singular vectors of Y, which
//                      U_k = Q(:,1:r_k) needs); null columns completed by a Philox
//                      block; always followed by a second CholQR pass
//       each CTA: Q = Y T (and Q1 T2) on its own rows; outputs fp64 Q, fp32 shadow, the 3xTF32
//       B-operand planes of the next power step, and (final step) U_k with the SPEC.md:232 sign
//       pin (cluster-wide argmax).
//
// All arithmetic is float64; every reduction has a fixed order, so repeated
// runs are bit-identical.  Cross-CTA data goes through global memory (L2) ordered by
// barrier.cluster (release/acquire), read with ld.global.cg.
#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdio>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"
#include "rtk_sm100.cuh"

namespace cg = cooperative_groups;

namespace rtk {

constexpr int kSL = 64;        // max l of this solver
constexpr int kLD = 65;        // leading dimension of the l x l fp64 shared matrices
constexpr int kMLD = 66;       // leading dimension of T (even: 16-byte double2 rows)
constexpr int kST = 256;       // threads per CTA
constexpr int kRBr = 8;        // rows per reduce_gram CTA
#ifndef RTK_RGC
#define RTK_RGC 4
#endif
constexpr int kRGC = RTK_RGC;   // reduce_gram cluster: one Gram partial per kRGC * kRBr = 32 rows (8-CTA clusters
                                // launch ~8 us slower: C5 reduce 22 -> 14.5 us, solve 9.60 -> 9.42 ms)
constexpr int kChunk = 64;     // rows per product chunk in step_kernel
constexpr int kMaxC = 32;      // step-kernel CTAs (a cluster up to 8 / 16 (non-portable); beyond 8 the grid barrier)
constexpr double kPinTie = 1e-5;   // sign pin: |entries| within this (relative) of the max are tied (C6)

__device__ __forceinline__ void unpack_upper(int e, int& c1, int& c2) {
  int t = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (t * (t + 1) / 2 > e) --t;
  while ((t + 1) * (t + 2) / 2 <= e) ++t;
  c2 = t;
  c1 = e - t * (t + 1) / 2;
}

// =============================================================== reduce + Gram partials
// Gram partials: one per 32-row block (a cluster of kRGC CTAs sums its CTAs' 8-row Grams through
// distributed shared memory), so the consumers sum ceil(n / 32) partials, not ceil(n / 8).
__host__ __device__ constexpr int gram_blocks(int n) { return (n + kRGC * kRBr - 1) / (kRGC * kRBr); }

constexpr int kRT = 512;   // reduce_gram threads: (column c = tid / 8, partial slice h = tid % 8)

__global__ void __launch_bounds__(kRT) reduce_gram_kernel(const float* __restrict__ Ypart, int G, int ltot,
                                                         int n_rows, int n, int l,
                                                         const double* __restrict__ Qd,
                                                         const double* __restrict__ alpha, int power,
                                                         double* __restrict__ Y, double* __restrict__ gpart,
                                                         const int* __restrict__ stop, int gmode, int early) {
  // gmode 0: Y and the Gram partials; 1: Y only (a multi-GPU shard, before Y's all-reduce);
  // 2: the Gram partials of the (all-reduced) Y already in Y
  __shared__ double Ys[kRBr][kSL + 1];
  __shared__ double gps[kSL * (kSL + 1) / 2];   // this CTA's 8-row Gram (packed upper)
  // early: let the step kernel's CTAs launch now (onto the SMs this grid leaves free) so their
  // launch overlaps this reduction; they still wait for its completion in griddepcontrol.wait
  if (early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  sm100::pdl_wait();   // the power step's Y partials
  if (stop && *(volatile const int*)stop) return;   // Alg. B.1 stopped this mode (uniform over the grid)
  const int tid = threadIdx.x;
  const int i0 = blockIdx.x * kRBr;
  const int rows = min(kRBr, n - i0);
  const double a = power ? *alpha : 0.0;
  const int64_t gs = (int64_t)ltot * n_rows;
  static_assert(kRBr == 8 && kRT == 8 * kSL, "thread (column c, partial slice h) layout");
  // thread (c, h) sums the partials g = h, h+8, ... of its column's 8 rows (two 16-B loads per
  // partial, five partials in flight: ~150 KB of partials in flight per CTA); the 8 slices of a
  // column are 8 consecutive lanes and meet in a fixed xor tree (repeatable results).  The rows past n
  // are Ypart padding, masked below; n_rows is a multiple of 4, and a last group with only 4 rows
  // inside n_rows takes the scalar loop.
  const int c = tid >> 3, h = tid & 7;
  for (int ii = tid; ii < kRBr * (kSL + 1); ii += kRT) Ys[ii / (kSL + 1)][ii % (kSL + 1)] = 0.0;
  __syncthreads();
  if (gmode != 2) {
    double acc[kRBr];
#pragma unroll
    for (int ii = 0; ii < kRBr; ++ii) acc[ii] = 0.0;
    if (c < l && i0 + kRBr > n_rows) {
      const float* src = Ypart + (int64_t)c * n_rows + i0;
      for (int g = h; g < G; g += 8)
        for (int ii = 0; ii < n_rows - i0; ++ii) acc[ii] += (double)__ldcg(src + (int64_t)g * gs + ii);
    } else if (c < l) {
      const float* src = Ypart + (int64_t)c * n_rows + i0;
      int g = h;
      for (; g + 32 < G; g += 40) {
        float4 v[10];
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          const float4* p = reinterpret_cast<const float4*>(src + (int64_t)(g + 8 * u) * gs);
          v[2 * u] = __ldcg(p);
          v[2 * u + 1] = __ldcg(p + 1);
        }
#pragma unroll
        for (int u = 0; u < 5; ++u) {
          acc[0] += (double)v[2 * u].x; acc[1] += (double)v[2 * u].y;
          acc[2] += (double)v[2 * u].z; acc[3] += (double)v[2 * u].w;
          acc[4] += (double)v[2 * u + 1].x; acc[5] += (double)v[2 * u + 1].y;
          acc[6] += (double)v[2 * u + 1].z; acc[7] += (double)v[2 * u + 1].w;
        }
      }
      for (; g < G; g += 8) {
        const float4* p = reinterpret_cast<const float4*>(src + (int64_t)g * gs);
        const float4 x = __ldcg(p), y = __ldcg(p + 1);
        acc[0] += (double)x.x; acc[1] += (double)x.y; acc[2] += (double)x.z; acc[3] += (double)x.w;
        acc[4] += (double)y.x; acc[5] += (double)y.y; acc[6] += (double)y.z; acc[7] += (double)y.w;
      }
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1)
#pragma unroll
      for (int ii = 0; ii < kRBr; ++ii) acc[ii] += __shfl_xor_sync(0xffffffffu, acc[ii], o);
    // lane h of the column group finishes row h: Y = sum - alpha Q
    double sh = 0.0;
#pragma unroll
    for (int ii = 0; ii < kRBr; ++ii) sh = (ii == h) ? acc[ii] : sh;
    if (c < l && h < rows) {
      const int i = i0 + h;
      if (power) sh -= a * Qd[(int64_t)c * n + i];
      Y[(int64_t)c * n + i] = sh;
      Ys[h][c] = sh;
    }
  } else if (c < l && h < rows) {
    Ys[h][c] = Y[(int64_t)c * n + i0 + h];
  }
  if (gmode == 1) return;   // uniform over the grid: before any cluster barrier
  __syncthreads();
  const int np = l * (l + 1) / 2;
  for (int e = tid; e < np; e += kRT) {
    int c1, c2;
    unpack_upper(e, c1, c2);
    double s = 0.0;
#pragma unroll
    for (int ii = 0; ii < kRBr; ++ii) s += Ys[ii][c1] * Ys[ii][c2];
    gps[e] = s;
  }
  // the cluster's 32-row partial: CTA r sums its share of the entries over the kRGC CTAs' Grams
  // (CTA order), read through distributed shared memory
  cg::cluster_group cluster = cg::this_cluster();
  cluster.sync();
  const int r = (int)cluster.block_rank();
  double* gp = gpart + (int64_t)(blockIdx.x / kRGC) * np;
  const int e0 = r * np / kRGC, e1 = (r + 1) * np / kRGC;
  for (int e = e0 + tid; e < e1; e += kRT) {
    double v[kRGC];
#pragma unroll
    for (int q = 0; q < kRGC; ++q) v[q] = cluster.map_shared_rank(gps, q)[e];
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < kRGC; ++q) s += v[q];
    gp[e] = s;
  }
  cluster.sync();   // peers' shared memory stays live until every CTA has read it
}

// =============================================================== l x l building blocks
// (all called by the whole CTA, 256 threads; matrices in shared memory with ld kLD)

// Fast fp64 1/sqrt(x) (x > 0) and 1/x (x != 0), finite normal operands: the fp64 MUFU
// approximations (rsqrt/rcp.approx.ftz.f64, ~2^-22 relative) refined by two Newton steps to
// ~1e-16 relative -- no fp32 conversions, ~3x shorter dependent chains than DSQRT / DDIV.
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x * y, y, 1.5);
  y = y * fma(-0.5 * x * y, y, 1.5);
  return y;
}
// one Newton step (~2^-45 relative): the Cholesky pivots' 1/sqrt sits on the factorisation's serial
// pivot chain; R and R^{-1} at ~1e-13 relative leave Q^T Q - I at that level, far below the fp32 stream
__device__ __forceinline__ double rsqrt_1nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y * fma(-0.5 * x * y, y, 1.5);
}
__device__ __forceinline__ double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

// Blocked Cholesky A = R^T R of the symmetric l x l A (upper triangle read), R upper (zero below
// the diagonal, identity beyond l), with 4 x 4 blocks on a 16 x 16 thread grid: thread (I, J)
// keeps block A_IJ in registers.  Block step K: every thread (K, J >= K) factors the staged A_KK =
// R_KK^T R_KK itself (identical inputs, identical R_KK) and forms R_KJ = R_KK^{-T} A_KJ with the
// pivots' 1/sqrt, publishing row block K to R; then every (I, J > K) applies A_IJ -= R_KI^T R_KJ
// and thread (K+1, K+1) stages A_{K+1,K+1}.  Two barriers per 4 columns, no serial diagonal-block
// phase.  Returns false (uniformly) on a pivot <= 1e-13 * max(diag) or a non-finite pivot.
// flag: 32 doubles of scratch ([0] breakdown flag, [16..31] the staged diagonal block).
__device__ __noinline__ bool chol_upper(const double* A, double* R, double* flag, int l) {
  const int tid = threadIdx.x, bi = tid >> 4, bj = tid & 15;
  double a[4][4];
  double dmax = 0.0;
  for (int k = 0; k < l; ++k) dmax = fmax(dmax, A[k * kLD + k]);
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int row = 4 * bi + i, col = 4 * bj + j;
      a[i][j] = (row < l && col < l) ? A[min(row, col) * kLD + max(row, col)] : (row == col ? 1.0 : 0.0);
      if (row > col) R[row * kLD + col] = 0.0;
    }
  const double tol = 1e-13 * dmax;
  double* akk = flag + 16;
  if (tid == 0) {
    flag[0] = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) akk[4 * i + j] = a[i][j];
  }
  __syncthreads();
  const int nb = (l + 3) >> 2;
  for (int K = 0; K < nb; ++K) {
    if (bi == K && bj >= K) {
      double r[4][4], rs[4];
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) r[i][j] = akk[4 * i + j];
#pragma unroll
      for (int k = 0; k < 4; ++k) {   // 4 x 4 Cholesky in registers: r -> R_KK (upper)
        const double piv = r[k][k];
        if (!(piv > tol) || !(piv < DBL_MAX)) bad = true;
        rs[k] = bad ? 0.0 : rsqrt_fast(piv);
#pragma unroll
        for (int j = 0; j < 4; ++j) r[k][j] = j < k ? 0.0 : r[k][j] * rs[k];
#pragma unroll
        for (int i = k + 1; i < 4; ++i)
#pragma unroll
          for (int j = i; j < 4; ++j) r[i][j] = fma(-r[k][i], r[k][j], r[i][j]);
      }
      if (bj == K) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) R[(4 * K + i) * kLD + 4 * K + j] = r[i][j];
        if (bad) flag[0] = 1.0;
      } else {   // R_KJ = R_KK^{-T} A_KJ (forward substitution, 1 / R_KK(k, k) = rs[k])
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double v = a[k][j];
#pragma unroll
            for (int m = 0; m < k; ++m) v = fma(-r[m][k], a[m][j], v);
            a[k][j] = v * rs[k];
          }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) R[(4 * K + i) * kLD + 4 * bj + j] = a[i][j];
      }
    }
    __syncthreads();
    if (flag[0] != 0.0) return false;
    if (bi > K && bj >= bi) {   // trailing update (upper blocks only)
      double rki[4][4], rkj[4][4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
#pragma unroll
        for (int i = 0; i < 4; ++i) rki[m][i] = R[(4 * K + m) * kLD + 4 * bi + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) rkj[m][j] = R[(4 * K + m) * kLD + 4 * bj + j];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double v = a[i][j];
#pragma unroll
          for (int m = 0; m < 4; ++m) v = fma(-rki[m][i], rkj[m][j], v);
          a[i][j] = v;
        }
      if (bi == K + 1 && bj == K + 1) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) akk[4 * i + j] = a[i][j];
      }
    }
    __syncthreads();
  }
  for (int idx = tid; idx < (kSL - l) * kSL; idx += kST) {   // identity padding rows l..63
    const int k = l + idx / kSL, j = idx % kSL;
    R[k * kLD + j] = (k == j) ? 1.0 : 0.0;
  }
  for (int idx = tid; idx < l * (kSL - l); idx += kST) {     // zero padding columns of rows < l
    const int k = idx / (kSL - l), j = l + idx % (kSL - l);
    R[k * kLD + j] = 0.0;
  }
  __syncthreads();
  return true;
}

// T = R^{-1} for the upper triangular R (kSL x kSL, identity beyond l), as a 2 x 2 block inverse
// with 32 x 32 blocks: T11 = R11^{-1} and T22 = R22^{-1} by column back substitution (thread c of
// warps 0 / 1 owns column c of its block, in registers: T(i, c) = -(sum_{m>i} R(i, m) T(m, c)) /
// R(i, i), i descending; row i of R is a broadcast; the terms with m > c vanish as T(m, c) = 0),
// then X = R12 T22 and T12 = -T11 X on all threads (every block of T written: T11, T22 by the
// substitution, T12 by the product, the lower-left block zeroed).  rinv: kSL doubles of scratch.
// T has leading dimension kMLD.  (Measured in the step kernel: 28k cycles against 39k for a 4 x 4
// block-diagonal sweep; a recursive 8 -> 64 block version was no faster there.)
__device__ __noinline__ void tri_inv_upper(const double* R, double* T, int l, double* rinv) {
  // R is the identity beyond l, so is T; for l <= 32 the off-diagonal products vanish
  const int tid = threadIdx.x;
  constexpr int H = kSL / 2;
  static_assert(kST >= 4 * H && kST % H == 0, "thread layout");
  if (tid < kSL) rinv[tid] = 1.0 / R[tid * kLD + tid];
  __syncthreads();
  if (tid < kSL) {   // diagonal blocks: warp 0 -> T11, warp 1 -> T22; column in registers, unrolled
    const int lane = tid % H, lo = (tid / H) * H;
    const double* Rb = R + lo * kLD + lo;
    double t[H];
#pragma unroll
    for (int i = H - 1; i >= 0; --i) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;   // m = i+1 .. H-1 in 4 interleaved partial sums
#pragma unroll
      for (int m = i + 1; m < H; ++m) {
        switch ((m - i - 1) & 3) {
          case 0: s0 = fma(Rb[i * kLD + m], t[m], s0); break;
          case 1: s1 = fma(Rb[i * kLD + m], t[m], s1); break;
          case 2: s2 = fma(Rb[i * kLD + m], t[m], s2); break;
          default: s3 = fma(Rb[i * kLD + m], t[m], s3); break;
        }
      }
      const double ri = rinv[lo + i];
      t[i] = (lane > i) ? -((s0 + s1) + (s2 + s3)) * ri : (lane == i ? ri : 0.0);
    }
#pragma unroll
    for (int i = 0; i < H; ++i) T[(lo + i) * kMLD + lo + lane] = t[i];
  }
  __syncthreads();
  if (l <= H) {   // R12 = 0 and R22 = I (R is the identity beyond l): T12 = 0, T22 = I (done above)
    for (int idx = tid; idx < H * H; idx += kST) {
      T[(idx / H) * kMLD + H + idx % H] = 0.0;
      T[(H + idx / H) * kMLD + idx % H] = 0.0;
    }
    __syncthreads();
    return;
  }
  // X = R12 T22 (rows i < H, columns c >= H) staged in the lower-left block: X(i, c) at T(H + i, c - H)
  const int cc = tid % H, g = tid / H, rows = H / (kST / H);   // thread: column H + cc, rows g*rows ..
  {
    double x[H / (kST / H)];
#pragma unroll
    for (int k = 0; k < rows; ++k) x[k] = 0.0;
    for (int m = H; m < kSL; ++m) {
      const double t = T[m * kMLD + H + cc];
#pragma unroll
      for (int k = 0; k < rows; ++k) x[k] = fma(R[(g * rows + k) * kLD + m], t, x[k]);
    }
#pragma unroll
    for (int k = 0; k < rows; ++k) T[(H + g * rows + k) * kMLD + cc] = x[k];
  }
  __syncthreads();
  {   // T12 = -T11 X
    double y[H / (kST / H)];
#pragma unroll
    for (int k = 0; k < rows; ++k) y[k] = 0.0;
    for (int m = g * rows; m < H; ++m) {
      const double xv = T[(H + m) * kMLD + cc];
#pragma unroll
      for (int k = 0; k < rows; ++k) y[k] = fma(T[(g * rows + k) * kMLD + m], xv, y[k]);
    }
#pragma unroll
    for (int k = 0; k < rows; ++k) T[(g * rows + k) * kMLD + H + cc] = -y[k];
  }
  __syncthreads();
  for (int idx = tid; idx < H * H; idx += kST) T[(H + idx / H) * kMLD + idx % H] = 0.0;
  __syncthreads();
}

// Blocked Cholesky G = R^T R together with T = R^{-1} (l <= 64), 8 x 8 blocks, nb = ceil(l / 8)
// block steps.  R (ld kLD) and T (ld kMLD) come out as chol_upper / tri_inv_upper leave them: upper
// triangular, zero below the diagonal, the identity beyond l.  Block step K: thread 0 factors the
// updated diagonal block in registers -- R_KK and its inverse T_KK (1 / R_KK(k, k) is the pivot's
// rsqrt) -- then one thread per panel column forms R_KJ = T_KK^T A_KJ, and all threads apply the
// trailing update A_IJ -= R_KI^T R_KJ: three barriers per 8 columns against two per 4 columns plus
// a separate substitution inverse, and a small rolled code body (the 18k-instruction step kernel
// is fetched cold after every streaming pass, which evicts it from L2).  The off-diagonal blocks of
// T follow along block anti-diagonals d = J - I: T_IJ = -T_II sum_{K = I+1..J} R_IK T_KJ.  Returns
// false (uniformly) on a pivot <= 1e-13 max(diag G) or a non-finite pivot, the chol_upper rule.
// flag: 32 doubles of scratch.
__device__ unsigned long long g_chol_prof[8];   // phase cycles of chol_inv (RTK_CHOL=2, diagnostics)
__device__ __noinline__ bool chol_inv(const double* A, double* R, double* T, double* flag, int l, int prof) {
  const int tid = threadIdx.x;
  long long c0 = clock64(), c1;
#define CPROF(slot)                                                                     \
  if (prof && tid == 0 && blockIdx.x == 0) {                                           \
    c1 = clock64();                                                                     \
    atomicAdd(&g_chol_prof[slot], (unsigned long long)(c1 - c0));                       \
    c0 = c1;                                                                            \
  }
  const int nb = (l + 7) >> 3, L8 = 8 * nb;
  double dmax = 0.0;
  for (int k = 0; k < l; ++k) dmax = fmax(dmax, A[k * kLD + k]);
  const double tol = 1e-13 * dmax;
  for (int idx = tid; idx < kSL * kSL; idx += kST) {
    const int i = idx / kSL, j = idx % kSL;
    R[i * kLD + j] = (i < l && j < l) ? (j >= i ? A[i * kLD + j] : 0.0) : (i == j ? 1.0 : 0.0);
    T[i * kMLD + j] = (i == j) ? 1.0 : 0.0;
  }
  if (tid == 0) flag[0] = 0.0;
  __syncthreads();
  CPROF(0);
  for (int K = 0; K < nb; ++K) {
    const int b = 8 * K;
    if (tid == 0) {   // diagonal block: R_KK and T_KK in registers
      double a[8][8], t[8][8], rs[8];
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[i][j] = j >= i ? R[(b + i) * kLD + b + j] : 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double piv = a[k][k];
        if (!(piv > tol) || !(piv < DBL_MAX)) bad = true;
        rs[k] = bad ? 0.0 : rsqrt_1nr(piv);
        a[k][k] = piv * rs[k];
#pragma unroll
        for (int j = k + 1; j < 8; ++j) a[k][j] *= rs[k];
#pragma unroll
        for (int i = k + 1; i < 8; ++i)
#pragma unroll
          for (int j = i; j < 8; ++j) a[i][j] = fma(-a[k][i], a[k][j], a[i][j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        t[j][j] = rs[j];
#pragma unroll
        for (int i = j - 1; i >= 0; --i) {
          double sm = 0.0;
#pragma unroll
          for (int m = i + 1; m <= j; ++m) sm = fma(a[i][m], t[m][j], sm);
          t[i][j] = -sm * rs[i];
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = i; j < 8; ++j) {
          R[(b + i) * kLD + b + j] = a[i][j];
          T[(b + i) * kMLD + b + j] = t[i][j];
        }
      if (bad) flag[0] = 1.0;
    }
    __syncthreads();
    CPROF(1);
    if (flag[0] != 0.0) return false;
    const int S = L8 - b - 8;   // trailing columns
    if (tid < S) {   // panel column c: R_KJ(:, c) = T_KK^T A_KJ(:, c)
      const int c = b + 8 + tid;
      double x[8];
#pragma unroll
      for (int m = 0; m < 8; ++m) x[m] = R[(b + m) * kLD + c];
#pragma unroll
      for (int i = 7; i >= 0; --i) {
        double y = 0.0;
#pragma unroll
        for (int m = 0; m <= i; ++m) y = fma(T[(b + m) * kMLD + b + i], x[m], y);
        R[(b + i) * kLD + c] = y;
      }
    }
    __syncthreads();
    CPROF(2);
    {   // trailing update of the upper triangle, one 4 x 4 block per thread (16 independent chains)
      const int S4 = S >> 2;
      const int bi = tid / 14, bj = tid % 14;   // S4 <= 14
      if (bi < S4 && bj < S4 && bj >= bi) {
        const int r0 = b + 8 + 4 * bi, c0 = b + 8 + 4 * bj;
        double v[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) v[i][j] = R[(r0 + i) * kLD + c0 + j];
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          double x[4], y[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) { x[i] = R[(b + m) * kLD + r0 + i]; y[i] = R[(b + m) * kLD + c0 + i]; }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) v[i][j] = fma(-x[i], y[j], v[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (bj > bi || j >= i) R[(r0 + i) * kLD + c0 + j] = v[i][j];
      }
    }
    __syncthreads();
    CPROF(3);
  }
  for (int d = 1; d < nb; ++d) {   // T_IJ, J = I + d: one thread per block column
    const int p = tid >> 3, j = tid & 7;
    if (p < nb - d) {
      const int I = p, J = p + d;
      double P[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) P[i] = 0.0;
      for (int K = I + 1; K <= J; ++K)
#pragma unroll
        for (int m = 0; m < 8; ++m) {
          const double t = T[(8 * K + m) * kMLD + 8 * J + j];
#pragma unroll
          for (int i = 0; i < 8; ++i) P[i] = fma(R[(8 * I + i) * kLD + 8 * K + m], t, P[i]);
        }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double y = 0.0;
#pragma unroll
        for (int m = i; m < 8; ++m) y = fma(T[(8 * I + i) * kMLD + 8 * I + m], P[m], y);
        T[(8 * I + i) * kMLD + 8 * J + j] = -y;
      }
    }
    __syncthreads();
  }
  CPROF(4);
#undef CPROF
  return true;
}

// Householder tridiagonalisation H^T A H = tridiag(d, e) of the symmetric l x l A (read only).
// Thread (i = tid/4, part = tid%4) keeps A(i, part + 4jj), jj < 16, in registers.  Step k: the warp
// holding row k publishes it (Hv row k, entries j >= k+2; x0 = A(k, k+1), d_k = A(k, k) and
// ss = sum_{j>=k+2} A(k, j)^2 in scal), and after one barrier EVERY thread builds reflector k from
// those three scalars (identical inputs and operations, so no serial one-quad phase and no second
// barrier for it): v_k on rows k+1..l-1 with v_k(k+1) = x0 - alpha, beta_k = 2 / |v_k|^2 in hb[k].
// Then p = beta A v, K = beta/2 p^T v, A -= v p^T + (p - 2K v) v^T.  Two barriers per reflector.
// Hv rows are zero outside k+1..l-1 (so the reflector reads need no index tests).
// ACC: also accumulate QH = H_0 H_1 ... H_{l-3} (thread (i, part) keeps row i's columns part + 4jj in
// registers, the same layout as A) and write it to QH (ld kLD) at the end: the eigenvectors of A are
// then QH Z for those Z of the tridiagonal, one dense product instead of l - 2 reflector sweeps.
// (scripts/micro/trd_bench.cu: 136k cycles at l = 60 against 192k for the one-quad reflector.)
template <bool ACC>
__device__ __noinline__ void tridiag_t(const double* A, int l, double* Hv, double* hb, double* d, double* e, double* pbuf,
                                  double* pvbuf, double* scal, double* QH) {
  const int tid = threadIdx.x, i = tid >> 2, part = tid & 3;
  double w[16];
  double qh[ACC ? 16 : 1];
  if (ACC) {
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) qh[jj] = (i < l && part + 4 * jj == i) ? 1.0 : 0.0;
  }
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const int j = part + 4 * jj;
    w[jj] = (i < l && j < l) ? A[min(i, j) * kLD + max(i, j)] : 0.0;
  }
  // Hv row k holds v_k: entries j >= k+2 are A(k, j) as published by quad k, entry k+1 is v0 (every
  // thread writes the same value before reading), entries j <= k and j >= l stay zero -- so the
  // reflector reads need no index tests.  x0 = A(k, k+1), d_k = A(k, k), ss_k = sum_{j>=k+2} A(k, j)^2
  // go to scal[4 (k & 1) + 0..2].
  for (int idx = tid; idx < kSL * kSL; idx += kST) Hv[(idx >> 6) * kLD + (idx & 63)] = 0.0;
  auto publish = [&](int k) {   // the warp holding row k (warp-uniform branch, full-warp shuffles)
    if ((tid >> 5) != (k >> 3)) return;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = part + 4 * jj;
      if (j >= k + 2 && j < l) s4[jj & 3] = fma(w[jj], w[jj], s4[jj & 3]);
    }
    double ss = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    ss += __shfl_xor_sync(0xffffffffu, ss, 1);
    ss += __shfl_xor_sync(0xffffffffu, ss, 2);
    if (i == k) {
      double* sc = scal + 4 * (k & 1);
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = part + 4 * jj;
        if (j >= k + 2 && j < l) Hv[k * kLD + j] = w[jj];
        if (j == k + 1) sc[0] = w[jj];
        if (j == k) sc[1] = w[jj];
      }
      if (part == 0) sc[2] = ss;
    }
  };
  __syncthreads();
  publish(0);
  for (int k = 0; k + 2 < l; ++k) {
    __syncthreads();   // row k and ss_k published
    double* hk = Hv + k * kLD;
    const double* sc = scal + 4 * (k & 1);
    const double x0 = sc[0], dk = sc[1], ss = sc[2];
    double beta = 0.0, alph = x0, v0 = 0.0;
    if (ss > 0.0) {   // every thread builds reflector k (same inputs, same operations)
      const double t = ss + x0 * x0;
      const double nrm = t * rsqrt_fast(t);
      alph = x0 > 0.0 ? -nrm : nrm;
      v0 = x0 - alph;
      beta = 2.0 * rcp_fast(ss + v0 * v0);
    }
    if (tid == 0) {
      d[k] = dk;
      e[k] = alph;
      hb[k] = beta;
    }
    if (beta != 0.0) {
      hk[k + 1] = v0;   // identical value from every thread
      double vj[16];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) vj[jj] = hk[part + 4 * jj];
      const double vi = hk[i];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int jj = 0; jj < 16; jj += 4) {
        s0 = fma(w[jj], vj[jj], s0);
        s1 = fma(w[jj + 1], vj[jj + 1], s1);
        s2 = fma(w[jj + 2], vj[jj + 2], s2);
        s3 = fma(w[jj + 3], vj[jj + 3], s3);
      }
      double s = (s0 + s1) + (s2 + s3);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      double uq = 0.0;
      if (ACC) {
        double u4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) u4[jj & 3] = fma(qh[jj], vj[jj], u4[jj & 3]);
        uq = (u4[0] + u4[1]) + (u4[2] + u4[3]);
        uq += __shfl_xor_sync(0xffffffffu, uq, 1);
        uq += __shfl_xor_sync(0xffffffffu, uq, 2);
      }
      if (part == 0) {
        const bool act = i > k && i < l;
        pbuf[i] = act ? beta * s : 0.0;
        pvbuf[i] = act ? beta * s * vi : 0.0;
      }
      __syncthreads();
      const int lane = tid & 31;
      double t0 = pvbuf[lane] + pvbuf[lane + 32];
#pragma unroll
      for (int o = 16; o; o >>= 1) t0 += __shfl_xor_sync(0xffffffffu, t0, o);
      const double K = 0.5 * beta * t0;
      if (ACC) {
        const double bu = beta * uq;
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) qh[jj] = fma(-bu, vj[jj], qh[jj]);
      }
      if (i > k && i < l) {   // A -= v w^T + w v^T with w = p - K v:  A_ij -= v_i p_j + (p_i - 2K v_i) v_j
        const double bi = fma(-2.0 * K, vi, pbuf[i]);
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) w[jj] = fma(-bi, vj[jj], fma(-vi, pbuf[part + 4 * jj], w[jj]));
      }
    }
    publish(k + 1);
  }
  __syncthreads();
  if (l >= 2) {
    if (i == l - 2) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = part + 4 * jj;
        if (j == l - 2) d[l - 2] = w[jj];
        if (j == l - 1) e[l - 2] = w[jj];
      }
    }
    if (i == l - 1) {
#pragma unroll
      for (int jj = 0; jj < 16; ++jj)
        if (part + 4 * jj == l - 1) d[l - 1] = w[jj];
    }
  } else if (i == 0 && part == 0) {
    d[0] = w[0];
  }
  if (ACC && i < l) {
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      const int j = part + 4 * jj;
      if (j < l) QH[i * kLD + j] = qh[jj];
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void tridiag(const double* A, int l, double* Hv, double* hb, double* d, double* e,
                                        double* pbuf, double* pvbuf, double* scal) {
  tridiag_t<false>(A, l, Hv, hb, d, e, pbuf, pvbuf, scal, nullptr);
}

// Out(i, c) = sum_j QH(i, j) Z(j, c), i, c < l (QH, Out: ld kLD; Z: ld kMLD, 16-byte rows).
// Thread (rg = tid/16, cg = tid%16) computes the 4 x 4 block rows 4rg.., columns 4cg.. in registers:
// per j 4 broadcast loads of QH, 2 double2 loads of Z -- the two halves in an order alternating
// with bit 2 of cg, so a quarter warp's eight 16-byte loads fall in eight distinct bank groups.
__device__ __noinline__ void qh_times_z(const double* QH, const double* Z, int l, double* Out) {
  const int tid = threadIdx.x, rg = tid >> 4, cg = tid & 15;
  const int h0 = (cg >> 2) & 1;
  double acc[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) acc[r][cc] = 0.0;
#pragma unroll 2
  for (int j = 0; j < l; ++j) {
    double q[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) q[r] = QH[(4 * rg + r) * kLD + j];
    const double2* zr = reinterpret_cast<const double2*>(Z + j * kMLD + 4 * cg);
    const double2 za = zr[h0], zb = zr[h0 ^ 1];
    const double2 z01 = h0 ? zb : za, z23 = h0 ? za : zb;
    const double z[4] = {z01.x, z01.y, z23.x, z23.y};
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) acc[r][cc] = fma(q[r], z[cc], acc[r][cc]);
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
      if (4 * rg + r < l && 4 * cg + cc < l) Out[(4 * rg + r) * kLD + 4 * cg + cc] = acc[r][cc];
  __syncthreads();
}

// Number of eigenvalues < mu of the symmetric tridiagonal (d, e2 = e^2): sign changes of the
// Sturm sequence p_0 = 1, p_1 = d_0 - mu, p_k = (d_{k-1} - mu) p_{k-1} - e2_{k-2} p_{k-2},
// rescaled by exact powers of two every 4 terms (|p| grows by at most ~||T||^4 in between);
// an exact zero takes the sign opposite to its predecessor.
__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int l, double mu) {
  double pp = 1.0, p = d[0] - mu;
  if (p == 0.0) p = -1e-300;
  int cnt = (p < 0.0);
  auto step = [&](double dk, double ek) {
    double pn = fma(dk - mu, p, -ek * pp);
    if (pn == 0.0) pn = (p < 0.0) ? 1e-300 : -1e-300;
    cnt += ((pn < 0.0) != (p < 0.0));
    pp = p;
    p = pn;
  };
  int k = 1;
  for (; k + 3 < l; k += 4) {   // terms k..k+3 (k = 1 mod 4): loads first, rescale after term k+3
    double dk[4], ek[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { dk[u] = d[k + u]; ek[u] = e2[k - 1 + u]; }
#pragma unroll
    for (int u = 0; u < 4; ++u) step(dk[u], ek[u]);
    const int ex = max((int)((__double_as_longlong(p) >> 52) & 0x7ff), (int)((__double_as_longlong(pp) >> 52) & 0x7ff));
    const double sc = __longlong_as_double((long long)(2046 - ex) << 52);   // 2^(1023-ex)
    p *= sc;
    pp *= sc;
  }
  for (; k < l; ++k) step(d[k], e2[k - 1]);   // fewer than 4 terms left: no rescale point
  return cnt;
}

// lambda_min of the tridiagonal by 256-point multisection: one log-spaced round over
// [hi 2^-64, hi] (hi = min d_i >= lambda_min), then linear rounds to 1e-14 relative.
__device__ __noinline__ double lambda_min_ms(const double* d, const double* e2, int l, int* ibuf, double* dbuf) {
  const int tid = threadIdx.x;
  if (tid == 0) {
    double hi = d[0];
    for (int k = 1; k < l; ++k) hi = fmin(hi, d[k]);
    dbuf[0] = 0.0;
    dbuf[1] = hi;
  }
  __syncthreads();
  const double hi0 = dbuf[1];
  if (!(hi0 > 0.0)) return 0.0;
  for (int round = 0; round < 8; ++round) {
    const double lo = dbuf[0], hi = dbuf[1];
    if (round > 0 && hi - lo <= 1e-14 * hi) break;
    auto point = [&](int t) -> double {   // t in [0, kST]: grid point t (t = kST -> hi)
      if (round == 0) return t == 0 ? 0.0 : hi0 * exp2(-64.0 * (1.0 - (double)t / kST));
      return lo + (hi - lo) * (double)t / kST;
    };
    if (tid == 0) ibuf[0] = kST;
    __syncthreads();
    if (sturm_count(d, e2, l, point(tid + 1)) > 0) atomicMin(ibuf, tid);
    __syncthreads();
    if (tid == 0) {
      const int j = ibuf[0];   // smallest grid index whose point exceeds lambda_min
      if (j < kST) {
        dbuf[0] = point(j);
        dbuf[1] = point(j + 1);
      } else {
        dbuf[0] = hi;          // lambda_min == hi (within rounding)
        dbuf[1] = hi;
      }
    }
    __syncthreads();
  }
  return 0.5 * (dbuf[0] + dbuf[1]);
}

// All l eigenvalues (ascending, lam[c] = c-th smallest) by Sturm bisection: one 256-point
// log-spaced scan over the Gershgorin range, then 4 threads per eigenvalue, 5-section rounds.
__device__ __noinline__ void all_eigs(const double* d, const double* e, const double* e2, int l, double* lam, double* blo,
                         double* bhi, int* cnt) {
  const int tid = threadIdx.x;
  __shared__ double s_gl, s_gu;
  if (tid == 0) {
    double gl = DBL_MAX, gu = -DBL_MAX;
    for (int k = 0; k < l; ++k) {
      const double r = (k > 0 ? fabs(e[k - 1]) : 0.0) + (k + 1 < l ? fabs(e[k]) : 0.0);
      gl = fmin(gl, d[k] - r);
      gu = fmax(gu, d[k] + r);
    }
    const double nrm = fmax(fabs(gl), fabs(gu));
    s_gl = gl - 1e-14 * nrm - 1e-300;
    s_gu = gu + 1e-14 * nrm + 1e-300;
  }
  __syncthreads();
  const double gl = s_gl, gu = s_gu;
  // scan: point t = gu * 2^{-64 (1 - (t+1)/256)}, counts in cnt[t]
  const double pt = gu * exp2(-64.0 * (1.0 - (double)(tid + 1) / kST));
  cnt[tid] = (gu > 0.0) ? sturm_count(d, e2, l, pt) : l;
  __syncthreads();
  if (tid < l) {
    // smallest scan point with count > c
    int t = 0;
    while (t < kST && cnt[t] <= tid) ++t;
    double lo = (t == 0) ? gl : gu * exp2(-64.0 * (1.0 - (double)t / kST));
    double hi = (t < kST) ? gu * exp2(-64.0 * (1.0 - (double)(t + 1) / kST)) : gu;
    if (t == 0) lo = fmin(gl, 0.0);
    blo[tid] = lo;
    bhi[tid] = hi;
  }
  __syncthreads();
  const int c = tid >> 2, part = tid & 3;
  for (int round = 0; round < 40; ++round) {
    double mu = 0.0;
    int k = 0;
    if (c < l) {
      const double lo = blo[c], hi = bhi[c];
      mu = lo + (hi - lo) * (0.2 * (double)(part + 1));   // same expression as the update below
      k = sturm_count(d, e2, l, mu);
    }
    cnt[tid] = k;
    __syncthreads();
    int done = 1;
    if (c < l && part == 0) {
      double lo = blo[c], hi = bhi[c];
      const double base = lo;
      const double w = hi - lo;
      for (int s = 0; s < 4; ++s) {
        const double m = base + w * (0.2 * (double)(s + 1));
        if (cnt[4 * c + s] <= c) lo = fmax(lo, m);
        else hi = fmin(hi, m);
      }
      blo[c] = lo;
      bhi[c] = hi;
      // converged: 1e-15 relative, or the 4 eps ||T|| absolute accuracy a Sturm count can resolve
      // at all (without it tiny eigenvalues ran the full 40 rounds)
      done = (hi - lo) <= fmax(1e-15 * fmax(fabs(lo), fabs(hi)), 4.0 * DBL_EPSILON * fmax(fabs(gl), fabs(gu))) + 1e-300;
    }
    if (__syncthreads_and(done)) break;
  }
  if (tid < l) lam[tid] = 0.5 * (blo[tid] + bhi[tid]);
  __syncthreads();
}

// All l eigenvalues of the tridiagonal, split over the C CTAs of the step cluster: CTA `rank` owns
// eigenvalues c = rank, rank + C, ... (at most ceil(l / C)) and refines each with P = kST / owned
// threads by P-point multisection (P + 1 sub-intervals per round, ~log2(P) bits instead of the 2.3
// of the 4-thread 5-section in all_eigs), same convergence rule as all_eigs; each eigenvalue is
// computed by exactly one CTA (deterministic) and published to lamx, then every CTA reads all l
// after a cluster barrier.  lam[c] = c-th smallest.  cnt: kST ints, blo / bhi: kSL doubles.
// The step kernel's CTAs exchange data only through global memory (L2, ld.global.cg) and need a
// barrier with release / acquire ordering between them: a cluster barrier, or (gbar != nullptr) a
// self-resetting grid barrier in global memory -- a plain 16-CTA grid launches faster than a 16-CTA
// cluster (non-portable size).  gbar[0] counts arrivals, gbar[1] is the generation; both start at
// zero (memset per mode) and the count returns to zero after every barrier.  The CTAs are co-resident
// in practice (<= 16 CTAs; waiting CTAs only wait for the stream predecessor's CTAs to drain).
struct StepSync {
  unsigned int* gbar;
  __device__ void sync() const {
    if (!gbar) {
      cg::this_cluster().sync();
      return;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      volatile unsigned int* vgen = gbar + 1;
      const unsigned int gen = *vgen;   // before arriving: the last arrival bumps it
      __threadfence();                  // release this CTA's global writes
      if (atomicAdd(gbar, 1u) == gridDim.x - 1) {
        *(volatile unsigned int*)gbar = 0u;
        __threadfence();
        atomicAdd(gbar + 1, 1u);
      } else {
        while (*vgen == gen) { }
      }
      __threadfence();                  // acquire the other CTAs' writes
    }
    __syncthreads();
  }
};

__device__ __noinline__ void all_eigs_cluster(const double* d, const double* e, const double* e2, int l, double* lam,
                                 double* blo, double* bhi, int* cnt, double* lamx, int rank, int C,
                                 const StepSync& cluster) {
  const int tid = threadIdx.x;
  __shared__ double s_gl, s_gu;
  if (tid == 0) {
    double gl = DBL_MAX, gu = -DBL_MAX;
    for (int k = 0; k < l; ++k) {
      const double r = (k > 0 ? fabs(e[k - 1]) : 0.0) + (k + 1 < l ? fabs(e[k]) : 0.0);
      gl = fmin(gl, d[k] - r);
      gu = fmax(gu, d[k] + r);
    }
    const double nrm = fmax(fabs(gl), fabs(gu));
    s_gl = gl - 1e-14 * nrm - 1e-300;
    s_gu = gu + 1e-14 * nrm + 1e-300;
  }
  const int ne = (l > rank) ? (l - rank + C - 1) / C : 0;   // eigenvalues this CTA owns
  const int P = ne > 0 ? kST / ne : kST;                     // threads per eigenvalue
  const int u = tid / P, s = tid % P;                        // owned eigenvalue u, multisection point s
  const int c = rank + C * u;                                // its index (ascending)
  const bool act = u < ne && c < l;
  if (act && s == 0) { blo[u] = 0.0; bhi[u] = 0.0; }
  __syncthreads();
  const double gl = s_gl, gu = s_gu;
  const double floor_abs = 4.0 * DBL_EPSILON * fmax(fabs(gl), fabs(gu));
  if (act && s == 0) { blo[u] = gl; bhi[u] = gu; }
  __syncthreads();
  int* first = cnt;   // first[u]: smallest multisection point of eigenvalue u whose count exceeds u's index
  if (act && s == 0) first[u] = P;
  __syncthreads();
  for (int round = 0; round < 24; ++round) {
    double lo = 0.0, hi = 0.0;
    if (act) {
      lo = blo[u];
      hi = bhi[u];
      const double mu = lo + (hi - lo) * ((double)(s + 1) / (double)(P + 1));
      if (sturm_count(d, e2, l, mu) > c) atomicMin(first + u, s);
    }
    __syncthreads();
    int done = 1;
    if (act && s == 0) {
      // the first point whose count exceeds c bounds the eigenvalue from above
      const int j = first[u];
      first[u] = P;   // reset for the next round (read again only after the barrier below)
      const double w = hi - lo;
      const double nlo = (j == 0) ? lo : lo + w * ((double)j / (double)(P + 1));
      const double nhi = (j == P) ? hi : lo + w * ((double)(j + 1) / (double)(P + 1));
      blo[u] = fmax(lo, nlo);
      bhi[u] = fmin(hi, nhi);
      done = (bhi[u] - blo[u]) <= fmax(1e-15 * fmax(fabs(blo[u]), fabs(bhi[u])), floor_abs) + 1e-300;
    }
    if (__syncthreads_and(done)) break;
  }
  if (act && s == 0) lamx[c] = 0.5 * (blo[u] + bhi[u]);
  cluster.sync();
  for (int i = tid; i < l; i += kST) lam[i] = __ldcg(lamx + i);
  __syncthreads();
}

// Eigenvectors of the tridiagonal by inverse iteration (thread c < l: eigenvalue lam[c]); two
// solves of (T - lam I) x = b with LU without pivoting (tiny pivots replaced by eps ||T||), a
// deterministic start vector, normalised.  Z(i, c) = x_i at Z[i * ldz + c].  LU pivots kept in Lu(i, c).
__device__ __noinline__ void tri_eigvecs(const double* __restrict__ d, const double* __restrict__ e,
                                         const double* __restrict__ lam, int l, double* __restrict__ Z,
                                         double* __restrict__ Lu, int ldz) {
  const int c = threadIdx.x;
  if (c < l) {
    double tn = 0.0;
    for (int k = 0; k < l; ++k)
      tn = fmax(tn, fabs(d[k]) + (k > 0 ? fabs(e[k - 1]) : 0.0) + (k + 1 < l ? fabs(e[k]) : 0.0));
    const double tiny = DBL_EPSILON * tn + 1e-300;
    const double lm = lam[c];
    for (int i = 0; i < l; ++i) {   // start vector: deterministic, no special structure
      const uint32_t h = (uint32_t)(i * 0x9E3779B1u) ^ (uint32_t)(c * 0x85EBCA77u) ^ 0x2545F491u;
      Z[i * ldz + c] = 0.5 + (double)((h >> 8) & 0xffff) * (1.0 / 65536.0);
    }
    for (int it = 0; it < 2; ++it) {
      // forward: u_i = d_i - lam - m_i e_{i-1},  m_i = e_{i-1}/u_{i-1};  y_i = x_i - m_i y_{i-1}
      // (Lu keeps 1/u_i: one reciprocal on the forward chain, none on the backward one; rcp_fast is
      // within an ulp, which inverse iteration does not notice).  The factorisation is the same in
      // the second iteration: it reuses Lu and runs only the y recurrence.
      double y = Z[c];
      if (it == 0) {
        double u = d[0] - lm;
        if (fabs(u) < tiny) u = u < 0.0 ? -tiny : tiny;
        double ru = rcp_fast(u);
        Lu[c] = ru;
        for (int i = 1; i < l; ++i) {
          const double m = e[i - 1] * ru;
          u = d[i] - lm - m * e[i - 1];
          if (fabs(u) < tiny) u = u < 0.0 ? -tiny : tiny;
          ru = rcp_fast(u);
          Lu[i * kLD + c] = ru;
          y = Z[i * ldz + c] - m * y;
          Z[i * ldz + c] = y;
        }
      } else {
        for (int i = 1; i < l; ++i) {
          const double m = e[i - 1] * Lu[(i - 1) * kLD + c];
          y = Z[i * ldz + c] - m * y;
          Z[i * ldz + c] = y;
        }
      }
      // back: x_{l-1} = y_{l-1}/u_{l-1};  x_i = (y_i - e_i x_{i+1}) / u_i
      double x = Z[(l - 1) * ldz + c] * Lu[(l - 1) * kLD + c];
      Z[(l - 1) * ldz + c] = x;
      double mx = fabs(x);
      for (int i = l - 2; i >= 0; --i) {
        x = (Z[i * ldz + c] - e[i] * x) * Lu[i * kLD + c];
        Z[i * ldz + c] = x;
        mx = fmax(mx, fabs(x));
      }
      // scale, then normalise
      const double inv = mx > 0.0 ? 1.0 / mx : 1.0;
      double s = 0.0;
      for (int i = 0; i < l; ++i) {
        const double v = Z[i * ldz + c] * inv;
        Z[i * ldz + c] = v;
        s += v * v;
      }
      const double rn = 1.0 / sqrt(s);
      for (int i = 0; i < l; ++i) Z[i * ldz + c] *= rn;
    }
  }
  __syncthreads();
}

// Z <- H_0 H_1 ... H_{l-3} Z  (H_k = I - beta_k v_k v_k^T on rows k+1..l-1), column-private quads.
__device__ __noinline__ void back_transform(const double* Hv, const double* hb, int l, double* Z) {
  const int tid = threadIdx.x, c = tid >> 2, part = tid & 3;
  if (c < kSL) {
    for (int k = l - 3; k >= 0; --k) {
      const double b = hb[k];
      double s = 0.0;
      if (c < l && b != 0.0)
        for (int j = k + 1 + part; j < l; j += 4) s += Hv[k * kLD + j] * Z[j * kLD + c];
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (c < l && b != 0.0) {
        const double f = b * s;
        for (int j = k + 1 + part; j < l; j += 4) Z[j * kLD + c] -= f * Hv[k * kLD + j];
      }
    }
  }
  __syncthreads();
}

// ============================================================== step kernel (cluster)
struct StepArgs {
  int n, l, r, step, q;
  int shift, final_step;
  int nblk;                 // Gram partial blocks of Y (reduce_gram_kernel)
  const double* gpart;      // [nblk][np]
  const double* Y;          // [l][n]
  double* Q1;               // [l][n] scratch (two-pass)
  double* g2part;           // [C][np]
  double* gsum;             // [np] summed Gram of Y
  double* amax;             // [C][2*64] (|value|, index) per column, final step
  double* Qd;               // [l][n]
  float* Qs;                // [l][n]
  float* planes;            // [2 pN][pld] 3xTF32 planes of Q for the next op1 (nullptr: none)
  int pN, pld;
  int planes16;             // planes are the fp16 engine's: __half [2 pN][pld], Q scaled by 2^15
  int chol_old;             // RTK_CHOL=0: the 4 x 4 Cholesky + substitution inverse (A/B only)
  unsigned int* gbar;       // grid barrier (nullptr: a thread-block cluster, RTK_STEP_GBAR=0)
  int chol_prof;            // RTK_CHOL=2: phase clocks of chol_inv into g_chol_prof
  double* alpha;
  double* trace;            // [q]
  double* sigma;            // [128]
  int* status;              // [0] numeric, [1] fallback count, [2] q_used, [3] B.1 stopped
  float* U;                 // n x r (final step)
  uint64_t seed;
  uint32_t mode1;
  double* dbg;              // optional phase clocks [mode][step][16]
  int defer_alpha;          // non-final steps: the shift update runs in alpha_kernel (side stream)
  double pve_tol;           // > 0: Alg. B.1 stopping rule on power steps
  double* sighat;           // [kSL] B.1 sigma-hat of the previous power step (zero at mode start)
  int pin_q;                // Alg. A.2: U = sign-pinned Q (all l columns) and Qd pinned in place
  double* lamx;             // [kSL] eigenvalue exchange across the cluster (global scratch)
};

struct StepSmem {
  double G[kSL * kLD];      // Gram (later second-pass Gram); eigen path: Z aliases it
  double R[kSL * kLD];      // Cholesky factor; eigen path: LU pivots
  double T[kSL * kMLD];     // transform applied to the rows (ld kMLD)
  double H[kSL * kMLD];     // Householder vectors (ld kLD); product-chunk staging and the
                            // tridiagonal's eigenvectors (ld kMLD) alias it
  double d[kSL], e[kSL], e2[kSL], hb[kSL], lam[kSL], blo[kSL], bhi[kSL];
  double xrow[kSL], pbuf[kSL], rowbuf[2 * kSL], scal[32], dbuf[4];
  double colscale[kSL];
  double shat[kSL];         // B.1 sigma-hat, read before the first cluster barrier
  int valid[kSL];
  int cnt[kST];
  int ibuf[4];
  int flags[4];
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// out(i, c) = sum_k X(i, k) M(k, c) for the nrow (<= 64) rows staged in Xs and c < l; thread
// (rg = tid/16, cg = tid%16) computes rows 4rg.., columns 4cg.. in acc.  upper: M upper triangular.
__device__ __forceinline__ void chunk_product(const double* Xs, const double* M, int l, bool upper,
                                              double (&acc)[4][4]) {
  const int tid = threadIdx.x, rg = tid >> 4, cgp = tid & 15;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int kend = upper ? min(l, 4 * cgp + 4) : l;
#pragma unroll 2
  for (int k = 0; k < kend; ++k) {
    double x[4], m[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) x[i] = Xs[(4 * rg + i) * kLD + k];
    const double2 m01 = *reinterpret_cast<const double2*>(M + k * kMLD + 4 * cgp);
    const double2 m23 = *reinterpret_cast<const double2*>(M + k * kMLD + 4 * cgp + 2);
    m[0] = m01.x; m[1] = m01.y; m[2] = m23.x; m[3] = m23.y;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(x[i], m[j], acc[i][j]);
  }
}

// Stage rows [i0, i0+nr) of the column-major X ([c][n]) into Xs (zero padded), via L2.
__device__ void stage_rows(const double* X, int n, int l, int i0, int nr, double* Xs) {
  constexpr int kPer = kChunk * kSL / kST;   // 16 loads per thread, all issued before use
  double v[kPer];
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int idx = threadIdx.x + u * kST;
    const int c = idx / kChunk, ii = idx % kChunk;
    v[u] = (ii < nr && c < l) ? ldcg(X + (int64_t)c * n + i0 + ii) : 0.0;
  }
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int idx = threadIdx.x + u * kST;
    const int c = idx / kChunk, ii = idx % kChunk;
    Xs[ii * kLD + c] = v[u];
  }
  __syncthreads();
}

// Q rows [i0, i0+nr) staged in Xs -> fp64 master and either the 3xTF32 B planes of the next op1
// (hi = round-to-nearest tf32, lo = exact remainder; the tcgen05 paths) or the fp32 shadow the FFMA
// tiles read, rows fastest.
__device__ void write_outputs(const double* Xs, int nr, int i0, int n, int l, double* Qd, float* Qs,
                              float* planes, int pN, int pld, int p16) {
  const int cols = planes ? pN : l;
  for (int idx = threadIdx.x; idx < cols * kChunk; idx += kST) {
    const int c = idx / kChunk, row = idx % kChunk;
    if (row < nr) {
      const double v = c < l ? Xs[row * kLD + c] : 0.0;
      const int64_t o = (int64_t)c * n + i0 + row;
      const float f = (float)v;
      if (c < l) {
        Qd[o] = v;
        if (!planes) Qs[o] = f;
      }
      if (planes && p16) {   // fp16 engine (rtk_fused2.cu): 2^15 q = hi + lo, |q| <= 1
        const double x = v * 32768.0;
        const __half hi = __float2half_rn((float)x);
        const __half lo = __float2half_rn((float)(x - (double)__half2float(hi)));
        reinterpret_cast<__half*>(planes)[(int64_t)c * pld + i0 + row] = hi;
        reinterpret_cast<__half*>(planes)[(int64_t)(pN + c) * pld + i0 + row] = lo;
      } else if (planes) {
        const float hi = sm100::tf32_rna(f);
        planes[(int64_t)c * pld + i0 + row] = hi;
        planes[(int64_t)(pN + c) * pld + i0 + row] = (float)(v - (double)hi);
      }
    }
  }
}

// Fill G (symmetric, full) from packed upper entries in global memory (sum of `parts` arrays, in
// part order).  parts == 1: all of a thread's loads are issued before the first store.
__device__ void load_packed_sum(const double* src, int parts, int64_t stride, int l, double* G) {
  const int np = l * (l + 1) / 2;
  if (parts == 1) {
    constexpr int kPer = (kSL * (kSL + 1) / 2 + kST - 1) / kST;   // 9 entries per thread at most
    double v[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = threadIdx.x + u * kST;
      v[u] = e < np ? ldcg(src + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int e = threadIdx.x + u * kST;
      if (e < np) {
        int c1, c2;
        unpack_upper(e, c1, c2);
        G[c1 * kLD + c2] = v[u];
        G[c2 * kLD + c1] = v[u];
      }
    }
    __syncthreads();
    return;
  }
  for (int e = threadIdx.x; e < np; e += kST) {
    int c1, c2;
    unpack_upper(e, c1, c2);
    double s = 0.0;
    for (int b = 0; b < parts; ++b) s += ldcg(src + (int64_t)b * stride + e);
    G[c1 * kLD + c2] = s;
    G[c2 * kLD + c1] = s;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kST, 1) step_kernel(const StepArgs a) {
  extern __shared__ __align__(16) uint8_t smraw[];
  StepSmem& S = *reinterpret_cast<StepSmem*>(smraw);
  const StepSync cluster{a.gbar};
  const int C = a.gbar ? (int)gridDim.x : (int)cg::this_cluster().num_blocks();
  const int rank = a.gbar ? (int)blockIdx.x : (int)cg::this_cluster().block_rank();
  const int tid = threadIdx.x;
  const int n = a.n, l = a.l;
  const int np = l * (l + 1) / 2;
  const int r0 = (int)((int64_t)rank * n / C), r1 = (int)((int64_t)(rank + 1) * n / C);
  sm100::pdl_wait();   // the reduction's Y and Gram partials
  const double alpha0 = (a.step > 0) ? *a.alpha : 0.0;   // read before any cluster barrier
  const bool pve = a.pve_tol > 0.0 && a.step > 0;
  // Alg. B.1 stopped this mode at an earlier power step: the remaining launches are no-ops
  if (pve && *(volatile const int*)(a.status + 3)) return;
  if (pve)
    for (int i = tid; i < kSL; i += kST) S.shat[i] = i < l ? a.sighat[i] : 0.0;
  long long tck[16];
  int ntck = 0;
  tck[ntck++] = clock64();

  // ---- 1. G = sum of the Gram partials (entries split across the cluster, fixed b order -- the
  // order alpha_kernel uses, so both see the same G)
  {
    const int e0 = (int)((int64_t)rank * np / C), e1 = (int)((int64_t)(rank + 1) * np / C);
    for (int e = e0 + tid; e < e1; e += kST) {
      double s = 0.0;
      int b = 0;
      for (; b + 16 <= a.nblk; b += 16) {   // 16 independent loads in flight, summed in b order
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = ldcg(a.gpart + (int64_t)(b + u) * np + e);
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
      }
      for (; b < a.nblk; ++b) s += ldcg(a.gpart + (int64_t)b * np + e);
      a.gsum[e] = s;
    }
  }
  tck[ntck++] = clock64();
  cluster.sync();
  load_packed_sum(a.gsum, 1, 0, l, S.G);
  // a non-finite iterate (non-finite input, or fp32 overflow of Y = M M^T Q) shows on the Gram's
  // diagonal: report RTK_ERR_NUMERIC (the step still runs, its outputs are unreliable)
  if (rank == 0 && tid < l && !isfinite(S.G[tid * kLD + tid])) a.status[0] = 6;
  tck[ntck++] = clock64();

  // ---- 2a. Alg. B.1 lines 9-12: all eigenvalues of G = Y^T Y give
  // Sigma = sqrt(lambda) (descending); sigma = Sigma + alpha; stop when
  // max_{i<=r} |sigma_i - sigmahat_i| <= tol * sigma_{r+1}.  Identical in every CTA.
  bool stop = false, have_eigs = false;
  double lam_min = 0.0, s1 = 0.0;
  if (pve) {
    tridiag(S.G, l, S.H, S.hb, S.d, S.e, S.pbuf, S.xrow, S.scal);
    for (int k = tid; k + 1 < l; k += kST) S.e2[k] = S.e[k] * S.e[k];
    __syncthreads();
    all_eigs_cluster(S.d, S.e, S.e2, l, S.lam, S.blo, S.bhi, S.cnt, a.lamx, rank, C, cluster);
    if (tid == 0) {
      double dmax = 0.0;
      for (int i = 0; i < a.r; ++i)
        dmax = fmax(dmax, fabs(sqrt(fmax(S.lam[l - 1 - i], 0.0)) + alpha0 - S.shat[i]));
      const double sr = sqrt(fmax(S.lam[l - 1 - a.r], 0.0)) + alpha0;
      S.flags[2] = (dmax <= a.pve_tol * sr) ? 1 : 0;
    }
    __syncthreads();
    stop = S.flags[2] != 0;
    have_eigs = true;
    lam_min = fmax(S.lam[0], 0.0);
    s1 = sqrt(fmax(S.lam[l - 1], 0.0));
    // line 15: sigmahat = sigma (every CTA copied sigmahat before the first cluster barrier)
    if (!stop && rank == 0)
      for (int i = tid; i < l; i += kST) a.sighat[i] = sqrt(fmax(S.lam[l - 1 - i], 0.0)) + alpha0;
  }

  // ---- 2. the l x l factorisation (redundant in every CTA)
  bool eig = a.final_step != 0 || stop;
  bool two_pass = false;
  if (!eig) {
    const bool ok = a.chol_old ? chol_upper(S.G, S.R, S.rowbuf, l) : chol_inv(S.G, S.R, S.T, S.rowbuf, l, a.chol_prof);
    tck[ntck++] = clock64();
    if (!ok) {
      eig = true;
    } else {
      if (a.chol_old) tri_inv_upper(S.R, S.T, l, S.rowbuf);
      tck[ntck++] = clock64();
      // kappa_F(R) = ||R||_F ||R^{-1}||_F >= kappa_2(Y); one CholQR pass leaves
      // ||Q^T Q - I|| ~ eps kappa^2
      {   // all threads: (i, j) = (idx / kSL, idx % kSL) over the upper triangle, then warp + block sums
        double rf = 0.0, tf = 0.0;
        for (int idx = tid; idx < kSL * kSL; idx += kST) {
          const int i = idx / kSL, j = idx % kSL;
          if (j >= i && j < l) {
            rf = fma(S.R[i * kLD + j], S.R[i * kLD + j], rf);
            tf = fma(S.T[i * kMLD + j], S.T[i * kMLD + j], tf);
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          rf += __shfl_xor_sync(0xffffffffu, rf, o);
          tf += __shfl_xor_sync(0xffffffffu, tf, o);
        }
        if ((tid & 31) == 0) { S.scal[tid >> 5] = rf; S.scal[kST / 32 + (tid >> 5)] = tf; }
        __syncthreads();
        if (tid == 0) {
          double r2 = 0.0, t2 = 0.0;
          for (int w = 0; w < kST / 32; ++w) { r2 += S.scal[w]; t2 += S.scal[kST / 32 + w]; }
          S.flags[0] = (DBL_EPSILON * r2 * t2 > 1e-7) ? 1 : 0;
        }
      }
      __syncthreads();
      two_pass = S.flags[0] != 0;
      tck[ntck++] = clock64();
      if (a.step > 0 && !a.defer_alpha && !have_eigs) {
        tridiag(S.G, l, S.H, S.hb, S.d, S.e, S.pbuf, S.xrow, S.scal);
        tck[ntck++] = clock64();
        for (int k = tid; k + 1 < l; k += kST) S.e2[k] = S.e[k] * S.e[k];
        __syncthreads();
        lam_min = lambda_min_ms(S.d, S.e2, l, S.ibuf, S.dbuf);
        if (tid == 0) {
          double gmax = 0.0;   // sigma_1^2 >= max_i G_ii
          for (int k = 0; k < l; ++k) gmax = fmax(gmax, S.G[k * kLD + k]);
          S.dbuf[2] = sqrt(gmax);
        }
        __syncthreads();
        s1 = S.dbuf[2];
      }
    }
  }
  if (eig) {
    tck[ntck++] = clock64();
    double* Z = S.G;    // G no longer needed
    if (!have_eigs) {
      // tridiagonalise with the accumulated reflector product QH (into T: free until the rows)
      tridiag_t<true>(S.G, l, S.H, S.hb, S.d, S.e, S.pbuf, S.xrow, S.scal, S.T);
      for (int k = tid; k + 1 < l; k += kST) S.e2[k] = S.e[k] * S.e[k];
      __syncthreads();
      tck[ntck++] = clock64();
      all_eigs_cluster(S.d, S.e, S.e2, l, S.lam, S.blo, S.bhi, S.cnt, a.lamx, rank, C, cluster);
      tck[ntck++] = clock64();
      tri_eigvecs(S.d, S.e, S.lam, l, S.H, S.R, kMLD);   // tridiagonal's eigenvectors (Householder rows done)
      tck[ntck++] = clock64();
      qh_times_z(S.T, S.H, l, Z);                  // A's eigenvectors = QH Z
    } else {            // tridiag / all_eigs results are still intact when B.1 computed them
      tck[ntck++] = clock64();
      tri_eigvecs(S.d, S.e, S.lam, l, Z, S.R, kLD);
      tck[ntck++] = clock64();
      back_transform(S.H, S.hb, l, Z);
    }
    // T(:, cc) = V(:, l-1-cc) / sqrt(lambda): descending order; null columns flagged
    const double sg1 = sqrt(fmax(S.lam[l - 1], 0.0));
    if (tid == 0) S.flags[1] = 0;
    __syncthreads();
    for (int cc = tid; cc < l; cc += kST) {
      const double sg = sqrt(fmax(S.lam[l - 1 - cc], 0.0));
      // Gram eigenvalues below l eps lambda_max are zero to working accuracy (the Gram squares
      // the condition of Y, whose fp32-accumulated entries carry ~1e-7 relative noise anyway);
      // their inverse-iteration vectors are not orthogonal: those columns are completed instead
      const int ok = (S.lam[l - 1 - cc] > kSL * DBL_EPSILON * S.lam[l - 1] && sg > 1e-200) ? 1 : 0;
      S.valid[cc] = ok;
      S.colscale[cc] = ok ? 1.0 / sg : 0.0;
      if (!ok) atomicOr(&S.flags[1], 1);
    }
    __syncthreads();
    for (int idx = tid; idx < kSL * kSL; idx += kST) {
      const int k = idx / kSL, cc = idx % kSL;
      S.T[k * kMLD + cc] = (k < l && cc < l) ? Z[k * kLD + (l - 1 - cc)] * S.colscale[cc] : 0.0;
    }
    // second CholQR pass when one pass cannot leave ||Q^T Q - I|| <~ 1e-7 (C20): completed null
    // columns, eps kappa(Y)^2 = eps lambda_max / lambda_min > 1e-7, or eigenvalues so close
    // (relative gap < 1e-8) that inverse iteration may return non-orthogonal vectors
    if (tid == 0) {
      bool tp = S.flags[1] != 0 || !(DBL_EPSILON * S.lam[l - 1] <= 1e-7 * S.lam[0]);
      for (int k = 0; k + 1 < l && !tp; ++k)
        if (S.lam[k + 1] - S.lam[k] < 1e-8 * S.lam[l - 1]) tp = true;
      S.flags[3] = tp ? 1 : 0;
    }
    __syncthreads();
    two_pass = S.flags[3] != 0;
    lam_min = fmax(S.lam[0], 0.0);
    s1 = sg1;
  }

  tck[ntck++] = clock64();
  // ---- shift update (Alg. 3/4 lines 8-9) and reports: one writer
  if (rank == 0 && tid == 0) {
    const double sl = sqrt(fmax(lam_min, 0.0));
    double a1 = alpha0;
    if (a.step > 0 && a.shift && sl > alpha0 && !(sl < 1e-14 * s1)) a1 = 0.5 * (sl + alpha0);
    if (stop) a1 = alpha0;   // B.1 line 11: break before the shift update
    if (a.step > 0 && !(a.defer_alpha && !a.final_step)) {
      *a.alpha = a1;
      a.trace[a.step - 1] = a1;
      a.status[2] = a.step;
    }
    if (stop) a.status[3] = 1;
    if (eig) {
      int nf = 0;
      for (int cc = 0; cc < l; ++cc) nf += S.valid[cc] ? 0 : 1;
      a.status[1] += nf;
    }
    if (!(a.defer_alpha && !a.final_step)) a.sigma[126] = sl;
  }
  if (eig && (a.final_step || stop) && rank == 0)
    for (int cc = tid; cc < l; cc += kST) a.sigma[cc] = sqrt(fmax(S.lam[l - 1 - cc], 0.0)) + alpha0;

  // ---- 3. rows of this CTA: Q = Y T (one pass) or Q1 = Y T, Gram2, Q = Q1 T2
  double* Xs = S.H;   // staging (Householder vectors no longer needed)
  const bool upperT = !eig;
  double g2[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) g2[i][j] = 0.0;
  const int rg = tid >> 4, cgp = tid & 15;
  for (int i0 = r0; i0 < r1; i0 += kChunk) {
    const int nr = min(kChunk, r1 - i0);
    stage_rows(a.Y, n, l, i0, nr, Xs);
    if (i0 == r0) tck[ntck++] = clock64();
    double acc[4][4];
    chunk_product(Xs, S.T, l, upperT, acc);
    __syncthreads();   // everyone done reading Xs
    if (i0 == r0) tck[ntck++] = clock64();
#pragma unroll
    for (int ii = 0; ii < 4; ++ii) {
      const int row = 4 * rg + ii;
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const int c = 4 * cgp + jj;
        double v = acc[ii][jj];
        if (row >= nr || c >= l) v = 0.0;
        Xs[row * kLD + c] = v;
      }
    }
    __syncthreads();
    if (i0 == r0) tck[ntck++] = clock64();
    if (eig && S.flags[1]) {
      // rank-deficient columns (flagged invalid): deterministic Philox completion, which the
      // second CholQR pass orthonormalises against the valid ones
      for (int idx = tid; idx < nr * l; idx += kST) {
        const int row = idx / l, c = idx % l;
        if (!S.valid[c]) {
          const uint4 x = omega_bits(a.seed ^ 0x5eed5eed5eed5eedull, 0x40000000u | (a.mode1 << 8) | (uint32_t)a.step,
                                     (uint64_t)(i0 + row), (uint32_t)c);
          const double v = (double)box_muller(x.x, x.y).x;
          Xs[row * kLD + c] = v;
          a.Q1[(int64_t)c * n + i0 + row] = v;
        }
      }
      __syncthreads();
    }
    if (two_pass) {
      for (int idx = tid; idx < l * kChunk; idx += kST) {   // coalesced: rows fastest
        const int c = idx / kChunk, row = idx % kChunk;
        if (row < nr) a.Q1[(int64_t)c * n + i0 + row] = Xs[row * kLD + c];
      }
    } else {
      write_outputs(Xs, nr, i0, n, l, a.Qd, a.Qs, a.planes, a.pN, a.pld, a.planes16);
    }
    if (two_pass) {
      // Gram2 partial (upper 4 x 4 blocks) of the Q1 rows now in Xs
      if (cgp >= rg) {
        for (int row = 0; row < nr; ++row) {
          double x[4], y[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) { x[i] = Xs[row * kLD + 4 * rg + i]; y[i] = Xs[row * kLD + 4 * cgp + i]; }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) g2[i][j] = fma(x[i], y[j], g2[i][j]);
        }
      }
      __syncthreads();
    }
  }
  tck[ntck++] = clock64();
  if (two_pass) {
    // publish this CTA's Gram2 partial (packed upper), sum over the cluster
    double* gp = a.g2part + (int64_t)rank * np;
    if (cgp >= rg) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c1 = 4 * rg + i, c2 = 4 * cgp + j;
          if (c1 <= c2 && c2 < l) gp[c2 * (c2 + 1) / 2 + c1] = g2[i][j];
        }
    }
    cluster.sync();
    load_packed_sum(a.g2part, C, np, l, S.G);
    const bool ok2 = a.chol_old ? chol_upper(S.G, S.R, S.rowbuf, l) : chol_inv(S.G, S.R, S.T, S.rowbuf, l, a.chol_prof);
    if (!ok2) {
      if (rank == 0 && tid == 0) a.status[0] = 6;   // RTK_ERR_NUMERIC
      for (int idx = tid; idx < kSL * kSL; idx += kST) {
        const int k = idx / kSL, c = idx % kSL;
        S.T[k * kMLD + c] = (k == c) ? 1.0 : 0.0;
      }
      __syncthreads();
    } else if (a.chol_old) {
      tri_inv_upper(S.R, S.T, l, S.rowbuf);
    }
    for (int i0 = r0; i0 < r1; i0 += kChunk) {
      const int nr = min(kChunk, r1 - i0);
      stage_rows(a.Q1, n, l, i0, nr, Xs);
      double acc[4][4];
      chunk_product(Xs, S.T, l, true, acc);
      __syncthreads();
#pragma unroll
      for (int ii = 0; ii < 4; ++ii) {
        const int row = 4 * rg + ii;
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int c = 4 * cgp + jj;
          Xs[row * kLD + c] = (row < nr && c < l) ? acc[ii][jj] : 0.0;
        }
      }
      __syncthreads();
      write_outputs(Xs, nr, i0, n, l, a.Qd, a.Qs, a.planes, a.pN, a.pld, a.planes16);
      __syncthreads();
    }
  }
  tck[ntck++] = clock64();
  if (rank == 0 && tid == 0 && a.dbg && a.step < 8 && a.mode1 <= 8) {
    double* o = a.dbg + 16 * (a.mode1 - 1) * 8 + 16 * a.step;
    o[0] = (double)ntck;
    o[1] = eig ? 1.0 : 0.0;
    o[2] = two_pass ? 1.0 : 0.0;
    for (int z = 1; z < ntck && z < 14; ++z) o[2 + z] = (double)(tck[z] - tck[z - 1]);
  }
  // plane padding rows n..pld-1 (zero) -- the last CTA
  if (a.planes && rank == C - 1) {
    for (int idx = tid; idx < 2 * a.pN * (a.pld - n); idx += kST) {
      const int c = idx / (a.pld - n), i = n + idx % (a.pld - n);
      if (a.planes16) reinterpret_cast<__half*>(a.planes)[(int64_t)c * a.pld + i] = __float2half_rn(0.f);
      else a.planes[(int64_t)c * a.pld + i] = 0.f;
    }
  }

  // ---- 4. final step: U_k = Q(:, 1:r) with the sign pin (largest |entry| positive, lowest
  // row index on ties), cluster-wide argmax
  if (a.final_step || stop) {
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (int c = warp; c < a.r; c += kST / 32) {
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = r0 + lane; i < r1; i += 32) {
        const double v = fabs(a.Qd[(int64_t)c * n + i]);
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        a.amax[(int64_t)rank * 2 * kSL + 2 * c] = best;
        a.amax[(int64_t)rank * 2 * kSL + 2 * c + 1] = (double)bi;
      }
    }
    cluster.sync();
    // ties: |entries| within kPinTie of the column maximum count as tied (reading C6): the pivot is
    // the lowest such row over the cluster (second reduction, indices in amax + kMaxC * 2 * kSL)
    double* amax2 = a.amax + (int64_t)kMaxC * 2 * kSL;
    for (int c = warp; c < a.r; c += kST / 32) {
      double best = -1.0;
      for (int b = 0; b < C; ++b) best = fmax(best, ldcg(a.amax + (int64_t)b * 2 * kSL + 2 * c));
      const double thr = (1.0 - kPinTie) * best;
      int bi = 0x7fffffff;
      for (int i = r0 + lane; i < r1; i += 32)
        if (fabs(a.Qd[(int64_t)c * n + i]) >= thr) { bi = i; break; }
#pragma unroll
      for (int o = 16; o; o >>= 1) bi = min(bi, __shfl_xor_sync(0xffffffffu, bi, o));
      if (lane == 0) amax2[(int64_t)rank * kSL + c] = (double)bi;
    }
    cluster.sync();
    for (int c = warp; c < a.r; c += kST / 32) {
      int bi = 0x7fffffff;
      for (int b = 0; b < C; ++b) bi = min(bi, (int)ldcg(amax2 + (int64_t)b * kSL + c));
      if (bi < 0 || bi >= n) bi = 0;   // non-finite column (no maximum found): the numeric flag reports it
      const double sgn = ldcg(a.Qd + (int64_t)c * n + bi) < 0.0 ? -1.0 : 1.0;
      if (lane == 0) S.colscale[c] = sgn;
      for (int i = r0 + lane; i < r1; i += 32) a.U[(int64_t)c * n + i] = (float)(sgn * a.Qd[(int64_t)c * n + i]);
    }
    if (a.pin_q) {   // Alg. A.2: the fp64 basis takes the same signs (after every CTA read its pivot)
      __syncthreads();
      cluster.sync();
      for (int c = warp; c < a.r; c += kST / 32)
        for (int i = r0 + lane; i < r1; i += 32) a.Qd[(int64_t)c * n + i] *= S.colscale[c];
    }
  }
}

// ============================================================== deferred shift update
// Alg. 3/4 lines 8-9 for a non-final power step, off the critical path: the next power step's
// streaming kernels need only Q, so this one-CTA kernel runs on a side stream concurrently with
// them and is joined before the next reduce (which subtracts alpha Q).
struct AlphaSmem {
  double G[kSL * kLD];
  double H[kSL * kLD];
  double d[kSL], e[kSL], e2[kSL], hb[kSL], pbuf[kSL], pvbuf[kSL], scal[32], dbuf[4];
  int ibuf[4];
};

__global__ void __launch_bounds__(kST, 1) alpha_kernel(const double* __restrict__ gpart, int nblk, int l, int step,
                                                      int shift,
                                                      double* __restrict__ alpha, double* __restrict__ trace,
                                                      int* __restrict__ status, double* __restrict__ sigma) {
  extern __shared__ __align__(16) uint8_t smraw[];
  AlphaSmem& S = *reinterpret_cast<AlphaSmem*>(smraw);
  const int tid = threadIdx.x;
  const double alpha0 = *alpha;
  {   // G = sum_b Gram_b in the same fixed b order as step_kernel (identical G, identical alpha)
    const int np = l * (l + 1) / 2;
    for (int e = tid; e < np; e += kST) {
      double sum = 0.0;
      int b = 0;
      for (; b + 16 <= nblk; b += 16) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldcg(gpart + (int64_t)(b + u) * np + e);
#pragma unroll
        for (int u = 0; u < 16; ++u) sum += v[u];
      }
      for (; b < nblk; ++b) sum += __ldcg(gpart + (int64_t)b * np + e);
      int c1, c2;
      unpack_upper(e, c1, c2);
      S.G[c1 * kLD + c2] = sum;
      S.G[c2 * kLD + c1] = sum;
    }
    __syncthreads();
  }
  tridiag(S.G, l, S.H, S.hb, S.d, S.e, S.pbuf, S.pvbuf, S.scal);
  for (int k = tid; k + 1 < l; k += kST) S.e2[k] = S.e[k] * S.e[k];
  __syncthreads();
  const double lam_min = lambda_min_ms(S.d, S.e2, l, S.ibuf, S.dbuf);
  if (tid == 0) {
    double gmax = 0.0;   // sigma_1^2 >= max_i G_ii
    for (int k = 0; k < l; ++k) gmax = fmax(gmax, S.G[k * kLD + k]);
    const double s1 = sqrt(gmax);
    const double sl = sqrt(fmax(lam_min, 0.0));
    double a1 = alpha0;
    if (shift && sl > alpha0 && !(sl < 1e-14 * s1)) a1 = 0.5 * (sl + alpha0);
    *alpha = a1;
    trace[step - 1] = a1;
    status[2] = step;
    sigma[126] = sl;
  }
}

cudaError_t launch_alpha(const ModeBufs& B, int step, bool shift, cudaStream_t st) {
  const size_t smem = sizeof(AlphaSmem);
  cudaError_t e = cudaFuncSetAttribute(alpha_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  alpha_kernel<<<1, kST, smem, st>>>(B.gpart, gram_blocks(B.n), B.l, step, shift ? 1 : 0, B.alpha, B.trace,
                                     B.status, B.sigma);
  return cudaGetLastError();
}

// ============================================================== Alg. A.2 lines 14-15
// Deterministic ST-HOSVD (Alg. 1, ST branch) of the small l_1 x ... x l_d tensor B that the
// holistic mode loop leaves, and U_k = Q_k V_k.  fp64 throughout;
// every reduction has a fixed order.  The tensor is column-major; around mode k its extents are
// (P, c, S): element (a, i, b) at a + P (i + c b).

// gram(i, j) = sum_{a,b} T(a, i, b) T(a, j, b): one CTA per packed upper entry (i <= j)
__global__ void __launch_bounds__(kST) a2_gram_kernel(const double* __restrict__ T, int64_t P, int c, int64_t S,
                                                      double* __restrict__ gram) {
  __shared__ double red[kST / 32];
  int i, j;
  unpack_upper((int)blockIdx.x, i, j);
  double s = 0.0;
  const int64_t tot = P * S;
  for (int64_t t = threadIdx.x; t < tot; t += kST) {
    const int64_t a = t % P, b = t / P;
    s = fma(T[a + P * (i + (int64_t)c * b)], T[a + P * (j + (int64_t)c * b)], s);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kST / 32; ++w) t += red[w];
    gram[i * c + j] = t;
    gram[j * c + i] = t;
  }
}

struct A2Smem {
  double G[kSL * kLD], R[kSL * kLD], H[kSL * kMLD];
  double d[kSL], e[kSL], e2[kSL], hb[kSL], lam[kSL], blo[kSL], bhi[kSL], pbuf[kSL], xrow[kSL];
  double scal[32], dbuf[4], dots[kSL];
  int cnt[kST];
  int ibuf[4];
};

// V = the r leading eigenvectors of the c x c Gram (descending eigenvalues) = the leading left
// singular vectors of T_(k): tridiagonalisation, Sturm bisection, inverse iteration and back-
// transformation (the step kernel's eigen path), then two classical Gram-Schmidt passes in
// descending order so that clustered eigenvalues still give an orthonormal V.
__global__ void __launch_bounds__(kST, 1) a2_eig_kernel(const double* __restrict__ gram, int c, int r,
                                                       double* __restrict__ V) {
  extern __shared__ __align__(16) uint8_t smraw[];
  A2Smem& S = *reinterpret_cast<A2Smem*>(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int idx = tid; idx < c * c; idx += kST) S.G[(idx / c) * kLD + idx % c] = gram[idx];
  __syncthreads();
  tridiag_t<true>(S.G, c, S.H, S.hb, S.d, S.e, S.pbuf, S.xrow, S.scal, S.R);   // QH -> R
  for (int k = tid; k + 1 < c; k += kST) S.e2[k] = S.e[k] * S.e[k];
  __syncthreads();
  all_eigs(S.d, S.e, S.e2, c, S.lam, S.blo, S.bhi, S.cnt);
  double* Z = S.G;
  tri_eigvecs(S.d, S.e, S.lam, c, S.H, S.G, kMLD);   // tridiagonal's eigenvectors into H (G is scratch)
  qh_times_z(S.R, S.H, c, Z);                  // eigenvectors of the Gram = QH Z
  // descending order into R: R(i, cc) = Z(i, c-1-cc)
  for (int idx = tid; idx < c * r; idx += kST) {
    const int i = idx % c, cc = idx / c;
    S.R[i * kLD + cc] = Z[i * kLD + (c - 1 - cc)];
  }
  // Gram-Schmidt only where inverse iteration may not return orthonormal vectors: a null eigenvalue
  // among the r kept (below c eps lambda_max) or two kept eigenvalues closer than 1e-8 lambda_max
  // (as the step kernel's second-pass rule, C20); otherwise QH Z is orthonormal to rounding
  __shared__ int s_cgs;
  if (tid == 0) {
    const double lmax = S.lam[c - 1];
    bool need = !(lmax > 0.0);
    for (int cc = 0; cc < r && !need; ++cc) {
      const double lk = S.lam[c - 1 - cc];
      if (!(lk > c * DBL_EPSILON * lmax)) need = true;
      if (cc + 1 < r && S.lam[c - 1 - cc] - S.lam[c - 2 - cc] < 1e-8 * lmax) need = true;
    }
    s_cgs = need ? 1 : 0;
  }
  __syncthreads();
  for (int cc = 0; cc < r && s_cgs; ++cc) {
    // the eigenvector first; if Gram-Schmidt leaves (almost) nothing of it -- a duplicate from a
    // degenerate cluster, e.g. the null space when r_k exceeds the rank of the l-core's unfolding --
    // complete with the first unit vector e_i that keeps a quarter of its norm
    for (int attempt = 0; attempt <= c; ++attempt) {
      if (attempt > 0) {
        if (tid < c) S.R[tid * kLD + cc] = (tid == attempt - 1) ? 1.0 : 0.0;
        __syncthreads();
      }
      for (int pass = 0; pass < 2; ++pass) {
        for (int jj = warp; jj < cc; jj += kST / 32) {   // dots with the finished columns
          double t = 0.0;
          for (int i = lane; i < c; i += 32) t = fma(S.R[i * kLD + jj], S.R[i * kLD + cc], t);
#pragma unroll
          for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
          if (lane == 0) S.dots[jj] = t;
        }
        __syncthreads();
        if (tid < c) {
          double x = S.R[tid * kLD + cc];
          for (int jj = 0; jj < cc; ++jj) x = fma(-S.dots[jj], S.R[tid * kLD + jj], x);
          S.R[tid * kLD + cc] = x;
        }
        __syncthreads();
      }
      if (warp == 0) {
        double t = 0.0;
        for (int i = lane; i < c; i += 32) t = fma(S.R[i * kLD + cc], S.R[i * kLD + cc], t);
#pragma unroll
        for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0) { S.dbuf[1] = t; S.dbuf[0] = t > 0.0 ? 1.0 / sqrt(t) : 0.0; }
      }
      __syncthreads();
      if (S.dbuf[1] >= (attempt == 0 ? 1e-4 : 0.25)) break;
    }
    if (tid < c) S.R[tid * kLD + cc] *= S.dbuf[0];
    __syncthreads();
  }
  for (int idx = tid; idx < c * r; idx += kST) V[idx] = S.R[(idx % c) * kLD + idx / c];
}

// U(:, cc) = s Q_k V(:, cc) with the sign pin s (largest |entry| positive, lowest row on ties,
// SPEC.md:232); V(:, cc) *= s so that the core keeps G = A x_k U_k^T.  One CTA per column.
// u_i = sum_j Q(i, j) V(j, cc) for this thread's rows i = tid + t kST, t < kUR, in registers: the
// loads of one j for all rows are independent (the sum itself runs in j order, as in the scalar form)
constexpr int kUR = 8;
__device__ __forceinline__ void a2_u_rows(const double* __restrict__ Q, int n, int l, const double* vs,
                                          double (&u)[kUR]) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int t = 0; t < kUR; ++t) u[t] = 0.0;
#pragma unroll 4
  for (int j = 0; j < l; ++j) {
    const double v = vs[j];
#pragma unroll
    for (int t = 0; t < kUR; ++t) {
      const int i = tid + t * kST;
      if (i < n) u[t] = fma(Q[i + (int64_t)n * j], v, u[t]);
    }
  }
}

// U(:, cc) = Q V(:, cc) with the sign pin (C6, tie-tolerant pivot), V's column takes the same sign.
// n <= kUR kST rows: each row's u is formed once in registers; larger n recompute it per pass.
__global__ void __launch_bounds__(kST) a2_u_kernel(const double* __restrict__ Q, int n, int l,
                                                   double* __restrict__ V, int r, float* __restrict__ U) {
  __shared__ double vs[kSL];
  __shared__ double bv[kST / 32];
  __shared__ int bi[kST / 32];
  const int cc = blockIdx.x, tid = threadIdx.x;
  if (tid < l) vs[tid] = V[tid + (int64_t)l * cc];
  __syncthreads();
  const bool reg = n <= kUR * kST;
  double ur[kUR];
  if (reg) a2_u_rows(Q, n, l, vs, ur);
  auto urow = [&](int i) -> double {   // large-n mode: recompute
    double u = 0.0;
    for (int j = 0; j < l; ++j) u = fma(Q[i + (int64_t)n * j], vs[j], u);
    return u;
  };
  // visit every row of this thread in ascending order with its u (registers, or recomputed)
  auto rows = [&](auto&& f) {
    if (reg) {
#pragma unroll
      for (int t = 0; t < kUR; ++t)
        if (tid + t * kST < n && !f(tid + t * kST, ur[t])) return;
    } else {
      for (int i = tid; i < n; i += kST)
        if (!f(i, urow(i))) return;
    }
  };
  double best = -1.0, bval = 0.0;
  int bidx = 0x7fffffff;
  rows([&](int i, double u) {
    if (fabs(u) > best) { best = fabs(u); bidx = i; bval = u; }
    return true;
  });
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    const double ov = __shfl_xor_sync(0xffffffffu, bval, o);
    if (ob > best || (ob == best && oi < bidx)) { best = ob; bidx = oi; bval = ov; }
  }
  if ((tid & 31) == 0) { bv[tid >> 5] = (bval < 0.0) ? -best : best; bi[tid >> 5] = bidx; }
  __syncthreads();
  __shared__ double sgn_s, thr_s;
  __shared__ int piv_s;
  if (tid == 0) {
    double b = -1.0;
    for (int w = 0; w < kST / 32; ++w) b = fmax(b, fabs(bv[w]));
    thr_s = (1.0 - kPinTie) * b;   // ties within kPinTie of the maximum (reading C6)
    piv_s = 0x7fffffff;
  }
  __syncthreads();
  rows([&](int i, double u) {   // lowest row whose |u_i| reaches the tie threshold
    if (fabs(u) >= thr_s) { atomicMin(&piv_s, i); return false; }
    return true;
  });
  __syncthreads();
  if (tid == 0) {
    double u = 0.0;
    const int i = piv_s == 0x7fffffff ? 0 : piv_s;
    for (int j = 0; j < l; ++j) u = fma(Q[i + (int64_t)n * j], vs[j], u);
    sgn_s = u < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  const double sgn = sgn_s;
  rows([&](int i, double u) {
    U[i + (int64_t)n * cc] = (float)(sgn * u);
    return true;
  });
  if (tid < l) V[tid + (int64_t)l * cc] = sgn * vs[tid];
}

// out(a, i', b) = sum_i V(i, i') T(a, i, b): extents (P, c, S) -> (P, r, S)
__global__ void __launch_bounds__(kST) a2_modeprod_kernel(const double* __restrict__ T, int64_t P, int c, int64_t S,
                                                          const double* __restrict__ V, int r, double* __restrict__ out) {
  const int64_t tot = P * r * S;
  for (int64_t idx = (int64_t)blockIdx.x * kST + threadIdx.x; idx < tot; idx += (int64_t)gridDim.x * kST) {
    const int64_t a = idx % P, tmp = idx / P;
    const int ip = (int)(tmp % r);
    const int64_t b = tmp / r;
    double s = 0.0;
    for (int i = 0; i < c; ++i) s = fma(V[i + (int64_t)c * ip], T[a + P * (i + (int64_t)c * b)], s);
    out[idx] = s;
  }
}

__global__ void a2_widen_kernel(const float* __restrict__ x, int64_t n, double* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (double)x[i];
}
__global__ void a2_narrow_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}

cudaError_t a2_finish(const float* B, int d, const int* l, const int* r, const int64_t* n, double* const* Qk,
                      double* g0, double* g1, double* gram, double* V, float* const* U, float* core, cudaStream_t st) {
  int64_t ext[8], tot = 1;
  for (int k = 0; k < d; ++k) { ext[k] = l[k]; tot *= l[k]; }
  const int gs = (int)std::min<int64_t>(4096, (tot + 255) / 256);
  a2_widen_kernel<<<gs, 256, 0, st>>>(B, tot, g0);
  const size_t smem = sizeof(A2Smem);
  cudaError_t e = cudaFuncSetAttribute(a2_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  for (int k = 0; k < d; ++k) {
    int64_t P = 1, S = 1;
    for (int j = 0; j < k; ++j) P *= ext[j];
    for (int j = k + 1; j < d; ++j) S *= ext[j];
    const int c = (int)ext[k];
    a2_gram_kernel<<<c * (c + 1) / 2, kST, 0, st>>>(g0, P, c, S, gram);
    a2_eig_kernel<<<1, kST, smem, st>>>(gram, c, r[k], V);
    a2_u_kernel<<<r[k], kST, 0, st>>>(Qk[k], (int)n[k], c, V, r[k], U[k]);
    const int64_t ot = P * r[k] * S;
    a2_modeprod_kernel<<<(int)std::min<int64_t>(4096, (ot + kST - 1) / kST), kST, 0, st>>>(g0, P, c, S, V, r[k], g1);
    std::swap(g0, g1);
    ext[k] = r[k];
  }
  int64_t rt = 1;
  for (int k = 0; k < d; ++k) rt *= r[k];
  a2_narrow_kernel<<<(int)std::min<int64_t>(4096, (rt + 255) / 256), 256, 0, st>>>(g0, rt, core);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- host side
double* g_step_dbg = nullptr;   // diagnostics: set by rtk_debug_clocks (not part of the product path)

// one 64-row chunk per CTA where the cluster can hold it: up to 8 CTAs (portable) or 16 when the
// device schedules a 16-CTA cluster of step_kernel (non-portable size; queried once per device).
// RTK_STEP_CLUSTER=8 caps it (A/B timing).
static int max_step_cluster() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 8;
  if (cached[dev]) return cached[dev];
  int best = 8;
  const char* ev = getenv("RTK_STEP_CLUSTER");
  const int cap = ev ? atoi(ev) : 16;
  if (cap >= 16 &&
      cudaFuncSetAttribute(step_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
      cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StepSmem)) ==
          cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16, 1, 1);
    cfg.blockDim = dim3(kST, 1, 1);
    cfg.dynamicSmemBytes = sizeof(StepSmem);
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, step_kernel, &cfg) == cudaSuccess && nc >= 1) best = 16;
  }
  cudaGetLastError();   // a refused query leaves no sticky error
  cached[dev] = best;
  return best;
}

int solve_cluster_size(int n) {
  const int C = (n + kChunk - 1) / kChunk;
  if (C <= 8) return std::max(1, C);
  // more than 8 CTAs run on the grid barrier (no cluster size limit) unless RTK_STEP_GBAR=0;
  // RTK_STEP_ROWS sets the rows per CTA there (A/B timing)
  const char* gb = getenv("RTK_STEP_GBAR");
  if (gb && gb[0] == '0') return std::min(C, max_step_cluster());
  const char* sr = getenv("RTK_STEP_ROWS");
  const int rows = sr ? std::max(16, atoi(sr)) : kChunk;
  return std::max(1, std::min(kMaxC, (n + rows - 1) / rows));
}

size_t solve_gpart_doubles(int n, int l) { return (size_t)gram_blocks(n) * l * (l + 1) / 2; }

// reduce_gram releases the step kernel at entry (its CTAs launch onto the SMs the reduction leaves
// free and wait in griddepcontrol.wait): C4 1.511 -> 1.473 ms, C3 1.460 -> 1.433, C5 unchanged
// (profiles/r2l_ab.txt).  RTK_RG_EARLY=0 keeps the implicit trigger at grid exit.
static bool rg_early() {
  const char* e = getenv("RTK_RG_EARLY");
  return !(e && e[0] == '0');
}

cudaError_t launch_reduce_gram2(const ModeBufs& B, bool power, cudaStream_t st, const int* stop, int gmode) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gram_blocks(B.n) * kRGC, 1, 1);   // CTAs past n contribute zero rows
  cfg.blockDim = dim3(kRT, 1, 1);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kRGC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (kRGC == 1) {   // no cluster: the PDL attribute alone
    attr[0] = attr[1];
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
  }
  cudaError_t e = cudaLaunchKernelEx(&cfg, reduce_gram_kernel, (const float*)B.Ypart, B.G, B.ltot, B.n_rows, B.n,
                                     B.l, (const double*)B.Qd, (const double*)B.alpha, power ? 1 : 0, B.Y, B.gpart,
                                     stop, gmode, rg_early() ? 1 : 0);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_step(const ModeBufs& B, int step, int q, bool shift, float* U, uint64_t seed, uint32_t mode1,
                        float* planes, int pN, int pld, bool defer_alpha, double pve_tol, cudaStream_t st,
                        bool pin_q, bool planes16) {
  StepArgs a;
  a.n = B.n; a.l = B.l; a.r = B.r; a.step = step; a.q = q;
  a.shift = shift ? 1 : 0; a.final_step = (step == q) ? 1 : 0;
  a.nblk = gram_blocks(B.n);
  a.gpart = B.gpart; a.Y = B.Y; a.Q1 = B.Q1; a.g2part = B.g2part; a.gsum = B.gsum; a.amax = B.amax;
  a.Qd = B.Qd; a.Qs = B.Qs; a.planes = planes; a.pN = pN; a.pld = pld; a.planes16 = planes16 ? 1 : 0;
  {
    const char* ce = getenv("RTK_CHOL");
    // the blocked 8 x 8 version wins for l <= 40 (C3 1.70 -> 1.68 ms, C4 1.91 -> 1.83), the 4 x 4 one
    // with the substitution inverse at l = 60 (C5 9.62 vs 9.69): its 15 short pivot blocks pipeline
    // better than 8 single-thread 8 x 8 factorisations on the fp64 latency chain
    a.chol_old = (ce && ce[0] == '0') || (!(ce && ce[0] >= '1') && B.l > 40) ? 1 : 0;
    a.chol_prof = (ce && ce[0] == '2') ? 1 : 0;
    static int calls = 0;
    if (a.chol_prof && calls++ > 0) {   // report the previous launch and reset
      unsigned long long h[8];
      cudaMemcpyFromSymbol(h, g_chol_prof, sizeof(h));
      fprintf(stderr, "[chol_inv prof, previous launch, CTA 0] init %llu diag %llu panel %llu trail %llu inverse %llu\n",
              h[0], h[1], h[2], h[3], h[4]);
      unsigned long long z[8] = {};
      cudaMemcpyToSymbol(g_chol_prof, z, sizeof(z));
    }
  }
  a.alpha = B.alpha; a.trace = B.trace; a.sigma = B.sigma; a.status = B.status;
  a.U = U; a.seed = seed; a.mode1 = mode1;
  a.dbg = g_step_dbg;
  a.defer_alpha = defer_alpha ? 1 : 0;
  a.pve_tol = pve_tol;
  a.sighat = B.sighat;
  a.pin_q = pin_q ? 1 : 0;
  a.lamx = B.lamx;
  const int C = solve_cluster_size(B.n);
  // the grid barrier for the non-portable 16-CTA size (C5: 9.39 -> 9.31 ms); up to 8 CTAs the cluster
  // barrier is cheaper (C4, 2 CTAs: 1.85 vs 1.90 ms).  RTK_STEP_GBAR=0 / 1 forces either.
  const char* gb = getenv("RTK_STEP_GBAR");
  const bool use_gbar = gb ? gb[0] != '0' : C > 8;
  a.gbar = (B.gbar && use_gbar) ? B.gbar : nullptr;
  const size_t smem = sizeof(StepSmem);
  cudaError_t e = cudaFuncSetAttribute(step_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(C, 1, 1);
  cfg.blockDim = dim3(kST, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  if (a.gbar) {   // plain grid, software barrier: the PDL attribute alone
    attr[0] = attr[1];
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
  }
  e = cudaLaunchKernelEx(&cfg, step_kernel, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace rtk
