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
__global__ void __launch_bounds__(256) reduce_gram_kernel(const float* __restrict__ Ypart, int G,
                                                          int ltot, int n_rows, int n, int l,
                                                          const double* __restrict__ Qd,
                                                          const double* __restrict__ alpha,
                                                          int power, double* __restrict__ Y,
                                                          double* __restrict__ gpart) {
  __shared__ double Ys[kRB][kLMax + 1];
  const int i0 = blockIdx.x * kRB;
  const int rows = min(kRB, n - i0);
  const double al = power ? *alpha : 0.0;
  const int64_t gs = (int64_t)ltot * n_rows;
  for (int idx = threadIdx.x; idx < kRB * l; idx += blockDim.x) {
    const int c = idx / kRB, ii = idx % kRB;
    double s = 0.0;
    if (ii < rows) {
      const float* src = Ypart + (int64_t)c * n_rows + i0 + ii;
      for (int g = 0; g < G; ++g) s += (double)src[(int64_t)g * gs];
      if (power) s -= al * Qd[(int64_t)c * n + i0 + ii];
      Y[(int64_t)c * n + i0 + ii] = s;
    }
    Ys[ii][c] = s;
  }
  __syncthreads();
  double* gp = gpart + (int64_t)blockIdx.x * l * l;
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int c1 = idx % l, c2 = idx / l;
    if (c1 > c2) continue;
    double s = 0.0;
    for (int ii = 0; ii < rows; ++ii) s += Ys[ii][c1] * Ys[ii][c2];
    gp[c1 + l * c2] = s;
    gp[c2 + l * c1] = s;
  }
}

cudaError_t launch_reduce_gram(const ModeBufs& B, bool power, cudaStream_t st) {
  reduce_gram_kernel<<<B.nblk, 256, 0, st>>>(B.Ypart, B.G, B.ltot, B.n_rows, B.n, B.l, B.Qd,
                                             B.alpha, power ? 1 : 0, B.Y, B.gpart);
  return cudaGetLastError();
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
// rotations per round, l_e - 1 rounds per sweep; rotation (c,s) from
// theta = (a_qq - a_pp) / (2 a_pq) (Golub & Van Loan, sym.schur2).  A rotation is
// skipped when |a_pq| <= 1e-17 sqrt(|a_pp a_qq|); converged when a whole sweep
// rotates nothing.  Sizes: l <= kLMax.
__global__ void __launch_bounds__(512) eig_kernel(const double* __restrict__ gpart, int nblk, int l,
                                                  int step, int q, int shift, double pve_tol,
                                                  double* __restrict__ alpha, double* __restrict__ T,
                                                  double* __restrict__ lam_out,
                                                  double* __restrict__ trace, double* __restrict__ sigma,
                                                  int* __restrict__ status, int r) {
  extern __shared__ double sm[];
  const int le = l + (l & 1);
  double* A = sm;                     // [l][l]   A[p*l + q]
  double* V = A + l * l;              // [l][l]   V[row*l + col]
  double* rc = V + l * l;             // [le/2]
  double* rs = rc + le / 2;           // [le/2]
  double* ev = rs + le / 2;           // [l] sorted eigenvalues
  int* rank = (int*)(ev + l);         // [l]
  __shared__ int any_rot;
  const int tid = threadIdx.x, nt = blockDim.x;

  for (int idx = tid; idx < l * l; idx += nt) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * l * l + idx];
    A[idx] = s;
    V[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
  }
  __syncthreads();

  const int half = le / 2;
  for (int sweep = 0; sweep < 60; ++sweep) {
    if (tid == 0) any_rot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < le - 1; ++rnd) {
      // pair k: (p_k, q_k) by the circle method; player le-1 fixed
      for (int k = tid; k < half; k += nt) {
        int p, qq;
        if (k == 0) { p = rnd; qq = le - 1; }
        else { p = (rnd + k) % (le - 1); qq = (rnd - k + (le - 1)) % (le - 1); }
        if (p > qq) { const int t = p; p = qq; qq = t; }
        double c = 1.0, s = 0.0;
        if (qq < l) {
          const double apq = A[p * l + qq], app = A[p * l + p], aqq = A[qq * l + qq];
          if (fabs(apq) > 1e-17 * sqrt(fabs(app * aqq)) && apq != 0.0) {
            const double th = (aqq - app) / (2.0 * apq);
            const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
            c = 1.0 / sqrt(1.0 + t * t);
            s = t * c;
            any_rot = 1;
          }
        }
        rc[k] = c;
        rs[k] = s;
      }
      __syncthreads();
      // rows: A <- J^T A
      for (int idx = tid; idx < half * l; idx += nt) {
        const int k = idx / l, j = idx % l;
        if (rs[k] == 0.0) continue;
        int p, qq;
        if (k == 0) { p = rnd; qq = le - 1; }
        else { p = (rnd + k) % (le - 1); qq = (rnd - k + (le - 1)) % (le - 1); }
        if (p > qq) { const int t = p; p = qq; qq = t; }
        const double c = rc[k], s = rs[k];
        const double ap = A[p * l + j], aq = A[qq * l + j];
        A[p * l + j] = c * ap - s * aq;
        A[qq * l + j] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: A <- A J ; V <- V J
      for (int idx = tid; idx < half * l; idx += nt) {
        const int k = idx / l, j = idx % l;
        if (rs[k] == 0.0) continue;
        int p, qq;
        if (k == 0) { p = rnd; qq = le - 1; }
        else { p = (rnd + k) % (le - 1); qq = (rnd - k + (le - 1)) % (le - 1); }
        if (p > qq) { const int t = p; p = qq; qq = t; }
        const double c = rc[k], s = rs[k];
        const double ap = A[j * l + p], aq = A[j * l + qq];
        A[j * l + p] = c * ap - s * aq;
        A[j * l + qq] = s * ap + c * aq;
        const double vp = V[j * l + p], vq = V[j * l + qq];
        V[j * l + p] = c * vp - s * vq;
        V[j * l + qq] = s * vp + c * vq;
      }
      __syncthreads();
    }
    if (!any_rot) break;
  }
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
  __shared__ double al_old, al_new;
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
    al_new = a1;
  }
  __syncthreads();
  const double s1 = sqrt(fmax(ev[0], 0.0));
  for (int i = tid; i < l; i += nt) {
    sigma[i] = sqrt(fmax(ev[i], 0.0)) + al_old;   // B.1 sigma = diag(Sigma)+alpha
    lam_out[i] = ev[i];
  }
  __syncthreads();
  // T(:, rank[i]) = V(:, i) / sigma_i ; invalid (rank-deficient) columns -> 0 with lam<0 marker
  for (int idx = tid; idx < l * l; idx += nt) {
    const int row = idx / l, col = idx % l;
    const int rk = rank[col];
    const double sg = sqrt(fmax(A[col * l + col], 0.0));
    const bool ok = sg > 1e-12 * s1 && sg > 1e-200;
    T[row + (int64_t)l * rk] = ok ? V[row * l + col] / sg : 0.0;
    if (row == 0 && !ok) lam_out[rk] = -1.0;
  }
  (void)al_new; (void)pve_tol; (void)q; (void)r;
}

cudaError_t launch_eig(const ModeBufs& B, int step, int q, bool shift, double pve_tol,
                       cudaStream_t st) {
  const int l = B.l, le = l + (l & 1);
  const size_t smem = sizeof(double) * (2 * l * l + le + l) + sizeof(int) * l + 64;
  cudaError_t e = cudaFuncSetAttribute(eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  eig_kernel<<<1, 512, smem, st>>>(B.gpart, B.nblk, l, step, q, shift ? 1 : 0, pve_tol, B.alpha,
                                   B.T, B.lam, B.trace, B.sigma, B.status, B.r);
  return cudaGetLastError();
}

// ------------------------------------------------------------- Q1 = Y T
__global__ void __launch_bounds__(256) apply_kernel(const double* __restrict__ Y,
                                                    const double* __restrict__ T,
                                                    const double* __restrict__ lam, int n, int l,
                                                    uint64_t seed, uint32_t mode, int step,
                                                    double* __restrict__ Q1,
                                                    double* __restrict__ gpart,
                                                    int* __restrict__ status) {
  extern __shared__ double sm[];
  double* Ts = sm;                       // [l][l] col-major
  double* Ys = Ts + l * l;               // [kRB][l+1]
  double* Qs = Ys + kRB * (l + 1);       // [kRB][l+1]
  const int i0 = blockIdx.x * kRB;
  const int rows = min(kRB, n - i0);
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) Ts[idx] = T[idx];
  for (int idx = threadIdx.x; idx < kRB * l; idx += blockDim.x) {
    const int c = idx / kRB, ii = idx % kRB;
    Ys[ii * (l + 1) + c] = ii < rows ? Y[(int64_t)c * n + i0 + ii] : 0.0;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < kRB * l; idx += blockDim.x) {
    const int c = idx / kRB, ii = idx % kRB;
    double s = 0.0;
    if (ii < rows) {
      if (lam[c] < 0.0) {
        // rank-deficient column: deterministic Gaussian completion (re-orthogonalised by CholQR)
        const int64_t i = i0 + ii;
        const uint4 x = omega_bits(seed ^ 0x5eed5eed5eed5eedull, 0x40000000u | (mode << 8) | (uint32_t)step,
                                   (uint64_t)i, (uint32_t)c);
        s = (double)box_muller(x.x, x.y).x;
        if (blockIdx.x == 0 && ii == 0) atomicAdd(&status[1], 1);
      } else {
        for (int k = 0; k < l; ++k) s += Ys[ii * (l + 1) + k] * Ts[k + l * c];
      }
      Q1[(int64_t)c * n + i0 + ii] = s;
    }
    Qs[ii * (l + 1) + c] = s;
  }
  __syncthreads();
  double* gp = gpart + (int64_t)blockIdx.x * l * l;
  for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) {
    const int c1 = idx % l, c2 = idx / l;
    if (c1 > c2) continue;
    double s = 0.0;
    for (int ii = 0; ii < rows; ++ii) s += Qs[ii * (l + 1) + c1] * Qs[ii * (l + 1) + c2];
    gp[c1 + l * c2] = s;
    gp[c2 + l * c1] = s;
  }
}

cudaError_t launch_apply(const ModeBufs& B, uint64_t seed, uint32_t mode, int step, cudaStream_t st) {
  const int l = B.l;
  const size_t smem = sizeof(double) * (l * l + 2 * kRB * (l + 1));
  cudaError_t e = cudaFuncSetAttribute(apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  apply_kernel<<<B.nblk, 256, smem, st>>>(B.Y, B.T, B.lam, B.n, l, seed, mode, step, B.Q1, B.gpart,
                                          B.status);
  return cudaGetLastError();
}

// ------------------------------------------------------- Cholesky + R^{-1}
__global__ void __launch_bounds__(256) chol_kernel(const double* __restrict__ gpart, int nblk, int l,
                                                   double* __restrict__ T2, int* __restrict__ status) {
  extern __shared__ double sm[];
  double* A = sm;            // [l][l] row-major, upper part used
  double* X = A + l * l;     // [l][l] R^{-1}
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int idx = tid; idx < l * l; idx += nt) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * l * l + idx];
    A[idx] = s;   // symmetric: row/col interchangeable
  }
  __syncthreads();
  // right-looking Cholesky, upper R with A = R^T R
  for (int k = 0; k < l; ++k) {
    __shared__ double piv;
    if (tid == 0) {
      double d = A[k * l + k];
      if (!(d > 0.0) || !isfinite(d)) {
        status[0] = 6;  // RTK_ERR_NUMERIC
        d = 1e-300;
      }
      piv = sqrt(d);
      A[k * l + k] = piv;
    }
    __syncthreads();
    for (int j = k + 1 + tid; j < l; j += nt) A[k * l + j] /= piv;
    __syncthreads();
    for (int idx = tid; idx < (l - k - 1) * (l - k - 1); idx += nt) {
      const int i = k + 1 + idx / (l - k - 1), j = k + 1 + idx % (l - k - 1);
      if (j >= i) A[i * l + j] -= A[k * l + i] * A[k * l + j];
    }
    __syncthreads();
  }
  // X = R^{-1}: column c solves R x = e_c by back substitution
  for (int c = tid; c < l; c += nt) {
    for (int i = l - 1; i >= 0; --i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int j = i + 1; j <= c; ++j) s -= A[i * l + j] * X[j * l + c];
      X[i * l + c] = (i <= c) ? s / A[i * l + i] : 0.0;
    }
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += nt) {
    const int i = idx % l, c = idx / l;
    T2[i + (int64_t)l * c] = X[i * l + c];
  }
}

cudaError_t launch_chol(const ModeBufs& B, cudaStream_t st) {
  const int l = B.l;
  const size_t smem = sizeof(double) * 2 * l * l;
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
    double s = 0.0;
    for (int k = 0; k <= c; ++k) s += Ys[ii * (l + 1) + k] * Ts[k + l * c];
    Qd[(int64_t)c * n + i0 + ii] = s;
    Qs[(int64_t)c * n + i0 + ii] = (float)s;
  }
}

cudaError_t launch_apply2(const ModeBufs& B, cudaStream_t st) {
  const int l = B.l;
  const size_t smem = sizeof(double) * (l * l + kRB * (l + 1));
  cudaError_t e = cudaFuncSetAttribute(apply2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  apply2_kernel<<<B.nblk, 256, smem, st>>>(B.Q1, B.T, B.n, l, B.Qd, B.Qs);
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
