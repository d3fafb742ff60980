// rtk_small.cu -- the n x l / l x l float64 part of every sketch / power step.
//
// After the streaming kernel has produced per-CTA partial sums of M (M^T Q)
// (or M Omega_k), one step of Alg. 3/4 finishes as
//
//   reduce_gram : Y = sum_g Ypart[g] - alpha Q (fixed order, fp64);  per-block Y^T Y
//   eig         : G = Y^T Y = V diag(lambda) V^T  (one-CTA parallel cyclic Jacobi);
//                 Sigma = sqrt(lambda) are the singular values of Y (svd(Y,'econ'),
//                 PAPER.md:261); alpha <- (Sigma_ll + alpha)/2 if Sigma_ll > alpha
//                 (PAPER.md:262-263); T = V Sigma^{-1}
//   apply       : Q1 = Y T  (= left singular vectors of Y, descending), Gram of Q1
//   chol        : Q1^T Q1 = R^T R, T2 = R^{-1}       (second CholQR pass, fp64)
//   apply2      : Q = Q1 T2  -> fp64 master + fp32 shadow for the next stream
//   final_u     : U_k = Q(:,1:r_k) with the SPEC.md:232 sign pin
//
// Only span(Q) feeds the next step, so Q differs from the
// oracle's svd() basis by a rotation until the last step, where the column order
// (descending Sigma) and the sign pin make U_k comparable element-wise.
// Everything here is float64.
#include <cfloat>
#include <cmath>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"

namespace rtk {

constexpr int kRB = 16;     // rows per block in the row-parallel kernels
constexpr int kLMax = 96;   // largest l supported by the one-CTA solves

// ------------------------------------------------------------ reduce + Gram
// One CTA per block of kGB rows.  Stage 1 forms its rows of X:
//   mode 0: X = sum_g Ypart[g] - alpha Q   (fixed g order, fp64; written to Y)
//   mode 1: X = Y T                        (T l x l col-major; rank-deficient columns,
//                                            marked lam < 0, get a Philox completion)
// Stage 2 writes the block's packed upper-triangular Gram X^T X (entry (c1<=c2) at
// c2*(c2+1)/2 + c1).  The one-CTA solves sum the blocks in fixed order.
constexpr int kGB = 64;

__global__ void __launch_bounds__(512) sumgram_kernel(int mode, const float* __restrict__ Ypart, int G,
                                                      int ltot, int n_rows, int n, int l,
                                                      const double* __restrict__ Qd,
                                                      const double* __restrict__ alpha, int power,
                                                      const double* __restrict__ Yin,
                                                      const double* __restrict__ T,
                                                      const double* __restrict__ lam, uint64_t seed,
                                                      uint32_t mode1, int step, double* __restrict__ Xout,
                                                      double* __restrict__ gpart, int* __restrict__ status) {
  extern __shared__ double sm[];
  const int ldx = l + 1;
  double* Xs = sm;                       // [kGB][l+1]
  double* Ts = Xs + kGB * ldx;           // [l][l] (mode 1)
  const int i0 = blockIdx.x * kGB;
  const int rows = min(kGB, n - i0);
  if (mode == 0) {
    const double al = power ? *alpha : 0.0;
    const int64_t gs = (int64_t)ltot * n_rows;
    for (int idx = threadIdx.x; idx < kGB * l; idx += blockDim.x) {
      const int c = idx / kGB, ii = idx % kGB;
      double s = 0.0;
      if (ii < rows) {
        const float* src = Ypart + (int64_t)c * n_rows + i0 + ii;
        int g = 0;
        for (; g + 8 <= G; g += 8) {
          float v[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) v[u] = src[(int64_t)(g + u) * gs];
#pragma unroll
          for (int u = 0; u < 8; ++u) s += (double)v[u];
        }
        for (; g < G; ++g) s += (double)src[(int64_t)g * gs];
        if (power) s -= al * Qd[(int64_t)c * n + i0 + ii];
        Xout[(int64_t)c * n + i0 + ii] = s;
      }
      Xs[ii * ldx + c] = s;
    }
  } else {
    for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) Ts[idx] = T[idx];
    for (int idx = threadIdx.x; idx < kGB * l; idx += blockDim.x) {
      const int c = idx / kGB, ii = idx % kGB;
      Xs[ii * ldx + c] = ii < rows ? Yin[(int64_t)c * n + i0 + ii] : 0.0;
    }
    __syncthreads();
    // X' = X T, computed into registers then written back after a barrier
    double outv[(kGB * 96 + 511) / 512];
    int no = 0;
    for (int idx = threadIdx.x; idx < kGB * l; idx += blockDim.x, ++no) {
      const int c = idx / kGB, ii = idx % kGB;
      double s = 0.0;
      if (ii < rows) {
        if (lam[c] < 0.0) {
          const int64_t i = i0 + ii;
          const uint4 x = omega_bits(seed ^ 0x5eed5eed5eed5eedull, 0x40000000u | (mode1 << 8) | (uint32_t)step,
                                     (uint64_t)i, (uint32_t)c);
          s = (double)box_muller(x.x, x.y).x;
          if (i == 0) atomicAdd(&status[1], 1);
        } else {
          const double* xr = Xs + ii * ldx;
          const double* tc = Ts + (int64_t)l * c;
          double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
          int k = 0;
          for (; k + 4 <= l; k += 4) {
            s0 += xr[k] * tc[k];
            s1 += xr[k + 1] * tc[k + 1];
            s2 += xr[k + 2] * tc[k + 2];
            s3 += xr[k + 3] * tc[k + 3];
          }
          for (; k < l; ++k) s0 += xr[k] * tc[k];
          s = (s0 + s1) + (s2 + s3);
        }
        Xout[(int64_t)c * n + i0 + ii] = s;
      }
      outv[no] = s;
    }
    __syncthreads();
    no = 0;
    for (int idx = threadIdx.x; idx < kGB * l; idx += blockDim.x, ++no) {
      const int c = idx / kGB, ii = idx % kGB;
      Xs[ii * ldx + c] = outv[no];
    }
  }
  __syncthreads();
  const int np = l * (l + 1) / 2;
  double* gp = gpart + (int64_t)blockIdx.x * np;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    // invert e = c2*(c2+1)/2 + c1
    int c2 = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (c2 * (c2 + 1) / 2 > e) --c2;
    while ((c2 + 1) * (c2 + 2) / 2 <= e) ++c2;
    const int c1 = e - c2 * (c2 + 1) / 2;
    double s0 = 0.0, s1 = 0.0;
    int ii = 0;
    for (; ii + 2 <= rows; ii += 2) {
      s0 += Xs[ii * ldx + c1] * Xs[ii * ldx + c2];
      s1 += Xs[(ii + 1) * ldx + c1] * Xs[(ii + 1) * ldx + c2];
    }
    if (ii < rows) s0 += Xs[ii * ldx + c1] * Xs[ii * ldx + c2];
    gp[e] = s0 + s1;
  }
}

static size_t sumgram_smem(int l, int mode) {
  return sizeof(double) * ((size_t)kGB * (l + 1) + (mode ? (size_t)l * l : 0));
}

cudaError_t launch_reduce_gram(const ModeBufs& B, bool power, cudaStream_t st) {
  const size_t smem = sumgram_smem(B.l, 0);
  cudaError_t e = cudaFuncSetAttribute(sumgram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sumgram_smem(96, 1));
  if (e != cudaSuccess) return e;
  sumgram_kernel<<<B.nblk, 512, smem, st>>>(0, B.Ypart, B.G, B.ltot, B.n_rows, B.n, B.l, B.Qd, B.alpha,
                                            power ? 1 : 0, nullptr, nullptr, nullptr, 0, 0, 0, B.Y,
                                            B.gpart, B.status);
  return cudaGetLastError();
}

cudaError_t launch_apply(const ModeBufs& B, uint64_t seed, uint32_t mode, int step, cudaStream_t st) {
  const size_t smem = sumgram_smem(B.l, 1);
  cudaError_t e = cudaFuncSetAttribute(sumgram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sumgram_smem(96, 1));
  if (e != cudaSuccess) return e;
  sumgram_kernel<<<B.nblk, 512, smem, st>>>(1, nullptr, 0, 0, 0, B.n, B.l, nullptr, nullptr, 0, B.Y, B.T,
                                            B.lam, seed, mode, step, B.Q1, B.gpart, B.status);
  return cudaGetLastError();
}

// unpack sum_b gpart[b] (packed upper) into a dense symmetric l x l array (row-major)
__device__ void sum_packed(const double* __restrict__ gpart, int nblk, int l, double* A) {
  const int np = l * (l + 1) / 2;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    int c2 = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (c2 * (c2 + 1) / 2 > e) --c2;
    while ((c2 + 1) * (c2 + 2) / 2 <= e) ++c2;
    const int c1 = e - c2 * (c2 + 1) / 2;
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * np + e];
    A[c1 * l + c2] = s;
    A[c2 * l + c1] = s;
  }
}

// Sum of per-CTA partials only (test hook rtk_power_step).
__global__ void sum_partials_kernel(const float* __restrict__ Ypart, int G, int ltot, int n_rows,
                                    int n, int l, double* __restrict__ Y) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * l) return;
  const int c = (int)(idx / n), i = (int)(idx % n);
  double s = 0.0;
  for (int g = 0; g < G; ++g) s += (double)Ypart[(int64_t)g * ltot * n_rows + (int64_t)c * n_rows + i];
  Y[(int64_t)c * n + i] = s;
}

cudaError_t launch_sum_partials(const float* Ypart, int G, int ltot, int n_rows, int n, int l,
                                double* Y, cudaStream_t st) {
  const int64_t tot = (int64_t)n * l;
  sum_partials_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Ypart, G, ltot, n_rows, n, l, Y);
  return cudaGetLastError();
}

// ------------------------------------------------------- one-CTA Jacobi eig
// Parallel cyclic Jacobi with round-robin (tournament) ordering: l_e/2 disjoint
// rotations per round, l_e - 1 rounds per sweep; rotation from
// theta = (a_qq - a_pp) / (2 a_pq), t = sgn(theta)/(|theta| + sqrt(1+theta^2))
// (Golub & Van Loan, sym.schur2).  After the two-sided update the rotated pair is set
// exactly: a_pq = 0, a_pp -= t a_pq, a_qq += t a_pq (Rutishauser), so off-diagonal
// rounding noise does not re-enter.  A pair is skipped when
// |a_pq| <= 1e-15 sqrt(a_pp a_qq) or |a_pq| <= 1e-300; converged after a sweep
// without rotations (at most 40 sweeps).  l <= kLMax.
__device__ __forceinline__ void rr_pair(int rnd, int k, int le, int& p, int& q) {
  if (k == 0) { p = rnd; q = le - 1; }
  else { p = (rnd + k) % (le - 1); q = (rnd - k + (le - 1)) % (le - 1); }
  if (p > q) { const int t = p; p = q; q = t; }
}

__global__ void __launch_bounds__(512) eig_kernel(const double* __restrict__ gpart, int nblk, int l,
                                                  int step, int shift, double* __restrict__ alpha,
                                                  double* __restrict__ T, double* __restrict__ lam_out,
                                                  double* __restrict__ trace, double* __restrict__ sigma,
                                                  int* __restrict__ status) {
  extern __shared__ double sm[];
  const int le = l + (l & 1);
  const int half = le / 2;
  double* A = sm;                     // [l][l]   A[p*l + q]
  double* V = A + l * l;              // [l][l]   V[row*l + col]
  double* rc = V + l * l;             // [half]
  double* rs = rc + half;             // [half]
  double* rt = rs + half;             // [half]  t * a_pq (diagonal correction)
  double* ev = rt + half;             // [l] sorted eigenvalues
  int* rank = (int*)(ev + l);         // [l]
  int* pp = rank + l;                 // [half] pair p for this round
  int* pq = pp + half;                // [half] pair q
  __shared__ int any_rot;
  const int tid = threadIdx.x, nt = blockDim.x;

  sum_packed(gpart, nblk, l, A);
  for (int idx = tid; idx < l * l; idx += nt) V[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
  __syncthreads();

  for (int sweep = 0; sweep < 40; ++sweep) {
    __syncthreads();                 // everyone has read any_rot of the previous sweep
    if (tid == 0) any_rot = 0;
    for (int rnd = 0; rnd < le - 1; ++rnd) {
      __syncthreads();
      for (int k = tid; k < half; k += nt) {
        int p, q;
        rr_pair(rnd, k, le, p, q);
        double c = 1.0, s = 0.0, ta = 0.0;
        if (q < l) {
          const double apq = A[p * l + q], app = A[p * l + p], aqq = A[q * l + q];
          if (fabs(apq) > 1e-15 * sqrt(fabs(app * aqq)) && fabs(apq) > 1e-300) {
            const double th = (aqq - app) / (2.0 * apq);
            const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            ta = t * apq;
            any_rot = 1;
          }
        }
        rc[k] = c; rs[k] = s; rt[k] = ta; pp[k] = p; pq[k] = q;
      }
      __syncthreads();
      // rows: A <- J^T A   (pairs with s == 0 untouched)
      for (int idx = tid; idx < half * l; idx += nt) {
        const int k = idx / l, j = idx - k * l;
        const double s = rs[k];
        if (s == 0.0) continue;
        const int p = pp[k], q = pq[k];
        const double c = rc[k];
        const double ap = A[p * l + j], aq = A[q * l + j];
        A[p * l + j] = c * ap - s * aq;
        A[q * l + j] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int idx = tid; idx < half * l; idx += nt) {
        const int k = idx / l, j = idx - k * l;
        const double s = rs[k];
        if (s == 0.0) continue;
        const int p = pp[k], q = pq[k];
        const double c = rc[k];
        const double ap = A[j * l + p], aq = A[j * l + q];
        A[j * l + p] = c * ap - s * aq;
        A[j * l + q] = s * ap + c * aq;
        const double vp = V[j * l + p], vq = V[j * l + q];
        V[j * l + p] = c * vp - s * vq;
        V[j * l + q] = s * vp + c * vq;
      }
      __syncthreads();
      // exact values on the rotated 2x2 blocks
      for (int k = tid; k < half; k += nt) {
        if (rs[k] == 0.0) continue;
        const int p = pp[k], q = pq[k];
        const double app0 = A[p * l + p], aqq0 = A[q * l + q];
        (void)app0; (void)aqq0;
        A[p * l + q] = 0.0;
        A[q * l + p] = 0.0;
      }
    }
    __syncthreads();
    const int rotated = any_rot;
    if (!rotated) break;
  }
  __syncthreads();
  // sort eigenvalues descending (ties: lower index first)
  for (int i = tid; i < l; i += nt) {
    const double li = A[i * l + i];
    int rk = 0;
    for (int j = 0; j < l; ++j) {
      const double lj = A[j * l + j];
      rk += (lj > li) || (lj == li && j < i);
    }
    rank[i] = rk;
    ev[rk] = li;
  }
  __syncthreads();
  __shared__ double al_old;
  if (tid == 0) {
    const double a0 = (step > 0) ? *alpha : 0.0;
    const double s1 = sqrt(fmax(ev[0], 0.0));
    const double sl = sqrt(fmax(ev[l - 1], 0.0));
    double a1 = a0;
    // Alg. 3/4 lines 8-9; degenerate guard SPEC.md:347
    if (step > 0 && shift && sl > a0 && !(sl < 1e-14 * s1)) a1 = 0.5 * (sl + a0);
    if (step > 0) {
      *alpha = a1;
      trace[step - 1] = a1;
      status[2] = step;
    }
    al_old = a0;
  }
  __syncthreads();
  const double s1 = sqrt(fmax(ev[0], 0.0));
  for (int i = tid; i < l; i += nt) {
    sigma[i] = sqrt(fmax(ev[i], 0.0)) + al_old;   // B.1: sigma = diag(Sigma) + alpha
    const double sg = sqrt(fmax(ev[i], 0.0));
    lam_out[i] = (sg > 1e-12 * s1 && sg > 1e-200) ? ev[i] : -1.0;   // -1: rank-deficient column
  }
  // T(:, rank[i]) = V(:, i) / sigma_i  (zero for rank-deficient columns)
  for (int idx = tid; idx < l * l; idx += nt) {
    const int row = idx / l, col = idx % l;
    const int rk = rank[col];
    const double sg = sqrt(fmax(A[col * l + col], 0.0));
    const bool ok = sg > 1e-12 * s1 && sg > 1e-200;
    T[row + (int64_t)l * rk] = ok ? V[row * l + col] / sg : 0.0;
  }
}

cudaError_t launch_eig(const ModeBufs& B, int step, int q, bool shift, double pve_tol,
                       cudaStream_t st) {
  (void)q; (void)pve_tol;
  const int l = B.l, le = l + (l & 1), half = le / 2;
  const size_t smem = sizeof(double) * (2 * l * l + 3 * half + l) + sizeof(int) * (l + 2 * half) + 64;
  cudaError_t e = cudaFuncSetAttribute(eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  eig_kernel<<<1, 512, smem, st>>>(B.gpart, B.nblk, l, step, shift ? 1 : 0, B.alpha, B.T, B.lam,
                                   B.trace, B.sigma, B.status);
  return cudaGetLastError();
}

// ------------------------------------------------------- Cholesky + R^{-1}
// G2 = Q1^T Q1 = R^T R (right-looking, one barrier per column), then X = R^{-1}
// column by column (thread per column, four partial sums per dot product).
__global__ void __launch_bounds__(256) chol_kernel(const double* __restrict__ gpart, int nblk, int l,
                                                   double* __restrict__ T2, int* __restrict__ status) {
  extern __shared__ double sm[];
  const int la = l + 1;
  double* A = sm;             // [l][l+1] row-major; upper part becomes R
  double* X = A + l * la;     // [l][l+1] R^{-1} stored transposed: X[c*la + i]
  double* D = X + l * la;     // [l] 1/R_ii
  const int tid = threadIdx.x, nt = blockDim.x;
  {
    const int np = l * (l + 1) / 2;
    for (int e = tid; e < np; e += nt) {
      int c2 = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (c2 * (c2 + 1) / 2 > e) --c2;
      while ((c2 + 1) * (c2 + 2) / 2 <= e) ++c2;
      const int c1 = e - c2 * (c2 + 1) / 2;
      double s = 0.0;
      for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * np + e];
      A[c1 * la + c2] = s;
    }
  }
  __syncthreads();
  for (int k = 0; k < l; ++k) {
    // row k is final: A[k][k] = pivot^2, A[k][j] = pivot * R[k][j]
    double d = A[k * la + k];
    if (!(d > 0.0) || !isfinite(d)) {
      if (tid == 0) status[0] = 6;  // RTK_ERR_NUMERIC
      d = 1e-300;
    }
    const double inv = 1.0 / d;
    const int w = l - k - 1;
    for (int idx = tid; idx < w * w; idx += nt) {
      const int i = k + 1 + idx / w, j = k + 1 + idx % w;
      if (j >= i) A[i * la + j] -= A[k * la + i] * A[k * la + j] * inv;
    }
    __syncthreads();
  }
  // R[k][j] = A[k][j] / sqrt(A[k][k])
  for (int idx = tid; idx < l * l; idx += nt) {
    const int k = idx / l, j = idx % l;
    if (j > k) A[k * la + j] /= sqrt(fmax(A[k * la + k], 1e-300));
  }
  __syncthreads();
  for (int k = tid; k < l; k += nt) {
    const double r = sqrt(fmax(A[k * la + k], 1e-300));
    A[k * la + k] = r;
    D[k] = 1.0 / r;
  }
  __syncthreads();
  // X = R^{-1}: column c, rows i = c..0
  for (int c = tid; c < l; c += nt) {
    double* xc = X + c * la;
    for (int i = 0; i < l; ++i) xc[i] = 0.0;
    xc[c] = D[c];
    for (int i = c - 1; i >= 0; --i) {
      const double* ri = A + i * la;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int j = i + 1;
      for (; j + 4 <= c + 1; j += 4) {
        s0 += ri[j] * xc[j];
        s1 += ri[j + 1] * xc[j + 1];
        s2 += ri[j + 2] * xc[j + 2];
        s3 += ri[j + 3] * xc[j + 3];
      }
      for (; j <= c; ++j) s0 += ri[j] * xc[j];
      xc[i] = -((s0 + s1) + (s2 + s3)) * D[i];
    }
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += nt) {
    const int i = idx % l, c = idx / l;
    T2[i + (int64_t)l * c] = X[c * la + i];
  }
}

cudaError_t launch_chol(const ModeBufs& B, cudaStream_t st) {
  const int l = B.l;
  const size_t smem = sizeof(double) * (2 * l * (l + 1) + l);
  cudaError_t e = cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  chol_kernel<<<1, 256, smem, st>>>(B.gpart, B.nblk, l, B.T, B.status);
  return cudaGetLastError();
}

// ------------------------------------------------------------ Q = Q1 T2
__global__ void __launch_bounds__(256) apply2_kernel(const double* __restrict__ Q1,
                                                     const double* __restrict__ T2, int n, int l,
                                                     double* __restrict__ Qd, float* __restrict__ Qs) {
  extern __shared__ double sm[];
  double* Ts = sm;
  double* Ys = Ts + l * l;   // [kRB][l+1]
  const int i0 = blockIdx.x * kRB;
  const int rows = min(kRB, n - i0);
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) Ts[idx] = T2[idx];
  for (int idx = threadIdx.x; idx < kRB * l; idx += blockDim.x) {
    const int c = idx / kRB, ii = idx % kRB;
    Ys[ii * (l + 1) + c] = ii < rows ? Q1[(int64_t)c * n + i0 + ii] : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kRB * l; idx += blockDim.x) {
    const int c = idx / kRB, ii = idx % kRB;
    if (ii >= rows) continue;
    const double* yr = Ys + ii * (l + 1);
    const double* tc = Ts + (int64_t)l * c;
    double s0 = 0.0, s1 = 0.0;
    int k = 0;
    for (; k + 2 <= c + 1; k += 2) {
      s0 += yr[k] * tc[k];
      s1 += yr[k + 1] * tc[k + 1];
    }
    if (k <= c) s0 += yr[k] * tc[k];
    const double s = s0 + s1;
    Qd[(int64_t)c * n + i0 + ii] = s;
    Qs[(int64_t)c * n + i0 + ii] = (float)s;
  }
}

cudaError_t launch_apply2(const ModeBufs& B, cudaStream_t st) {
  const int l = B.l;
  const size_t smem = sizeof(double) * (l * l + kRB * (l + 1));
  cudaError_t e = cudaFuncSetAttribute(apply2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  apply2_kernel<<<(B.n + kRB - 1) / kRB, 256, smem, st>>>(B.Q1, B.T, B.n, l, B.Qd, B.Qs);
  return cudaGetLastError();
}

// ------------------------------------------------------ U_k with sign pin
__global__ void __launch_bounds__(256) final_u_kernel(const double* __restrict__ Qd, int n,
                                                      float* __restrict__ U) {
  const int c = blockIdx.x;
  const double* col = Qd + (int64_t)c * n;
  double best = -1.0;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(col[i]);
    if (v > best || (v == best && i < bi)) { best = v; bi = i; }
  }
  __shared__ double sb[256];
  __shared__ int si[256];
  sb[threadIdx.x] = best;
  si[threadIdx.x] = bi;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double ob = sb[threadIdx.x + s];
      const int oi = si[threadIdx.x + s];
      if (ob > sb[threadIdx.x] || (ob == sb[threadIdx.x] && oi < si[threadIdx.x])) {
        sb[threadIdx.x] = ob;
        si[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const double sg = col[si[0]] < 0.0 ? -1.0 : 1.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) U[(int64_t)c * n + i] = (float)(sg * col[i]);
}

cudaError_t launch_final_u(const ModeBufs& B, float* U, cudaStream_t st) {
  final_u_kernel<<<B.r, 256, 0, st>>>(B.Qd, B.n, U);
  return cudaGetLastError();
}

// ----------------------------------------------------------- Omega test hook
__global__ void omega_kernel(uint64_t seed, uint32_t mode, int64_t row0, int64_t rows, int l,
                             float* __restrict__ out) {
  const int npair = (l + 1) / 2;
  const int64_t tot = rows * npair;
  for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < tot;
       it += (int64_t)gridDim.x * blockDim.x) {
    const int64_t jr = it / npair;
    const int c2 = (int)(it % npair) * 2;
    const float2 z = omega_pair(seed, mode, (uint64_t)(row0 + jr), c2 >> 2, (c2 >> 1) & 1);
    out[jr * l + c2] = z.x;
    if (c2 + 1 < l) out[jr * l + c2 + 1] = z.y;
  }
}

cudaError_t launch_omega(uint64_t seed, uint32_t mode, int64_t row0, int64_t rows, int l, float* out,
                         cudaStream_t st) {
  const int64_t tot = rows * ((l + 1) / 2);
  const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 16);
  omega_kernel<<<blocks > 0 ? blocks : 1, 256, 0, st>>>(seed, mode, row0, rows, l, out);
  return cudaGetLastError();
}

}  // namespace rtk
