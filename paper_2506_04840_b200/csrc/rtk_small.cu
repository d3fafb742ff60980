// rtk_small.cu -- the n x l / l x l float64 part of every sketch / power step.
//
// After the streaming kernel has produced per-CTA partial sums of M (M^T Q)
// (or M Omega_k), one step of Alg. 3/4 finishes as
//
//   reduce  : Y = sum_g Ypart[g] - alpha Q      (fixed g order, fp64; all SMs)
//   gram    : per 64-row block, packed upper Y^T Y
//   orth    : one CTA on G = Y^T Y (l x l):
//             * non-final steps: Cholesky G = R^T R, T = R^{-1} (CholQR, span only --
//               SURVEY.md 8(c) C4); the shift needs Sigma_ll = sqrt(lambda_min(G)):
//               single-warp Householder tridiagonalisation + block-wide Sturm
//               multisection;  alpha <- (Sigma_ll + alpha)/2 if Sigma_ll > alpha
//
//             * final step (and Cholesky breakdown): cyclic Jacobi G = V diag(lambda) V^T,
//               T = V Sigma^{-1} (left singular vectors of Y in descending order, which
//               U_k = Q(:,1:r_k) needs), completion of rank-deficient columns
//   gram(T) : Q1 = Y T, packed Q1^T Q1
//   chol    : second CholQR pass, T2 = R2^{-1}
//   apply2  : Q = Q1 T2 -> fp64 master + fp32 shadow for the next stream
//   final_u : U_k = Q(:,1:r_k) with the SPEC.md:232 sign pin
//
// Everything here is float64; reductions use fixed orders so
// repeated runs are bit-identical.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"

namespace rtk {

constexpr int kRB = 16;     // rows per block in apply2
constexpr int kGB = 64;     // rows per Gram block
constexpr int kOrthThreads = 1024;

// ------------------------------------------------------------------ reduce
// Y(c, i) = sum_g Ypart[g][c][i] (g ascending) - alpha Q(c, i); one thread per element.
__global__ void __launch_bounds__(256) reduce_kernel(const float* __restrict__ Ypart, int G, int ltot,
                                                     int n_rows, int n, int l,
                                                     const double* __restrict__ Qd,
                                                     const double* __restrict__ alpha, int power,
                                                     double* __restrict__ Y) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * l) return;
  const int c = (int)(idx / n), i = (int)(idx - (int64_t)c * n);
  const int64_t gs = (int64_t)ltot * n_rows;
  const float* src = Ypart + (int64_t)c * n_rows + i;
  double s = 0.0;
  int g = 0;
  for (; g + 8 <= G; g += 8) {
    float v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + (int64_t)(g + u) * gs);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += (double)v[u];
  }
  for (; g < G; ++g) s += (double)__ldg(src + (int64_t)g * gs);
  if (power) s -= (*alpha) * Qd[idx];
  Y[idx] = s;
}

// ------------------------------------------------------------------ gram
// One CTA per kGB-row block.  mode 0: X = Y.  mode 1: X = Y T (T l x l column-major);
// columns marked lam[c] < 0 (rank-deficient, Jacobi path) get a deterministic Philox
// Gaussian completion that the second CholQR pass orthonormalises.  mode 1 writes X to
// Xout and, when status[3] == 0 (single pass suffices), straight to Qd / Qs.
// Then the block's packed upper Gram X^T X (entry (c1<=c2) at c2(c2+1)/2 + c1).
__device__ __forceinline__ void unpack_index(int e, int& c1, int& c2) {
  int t = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (t * (t + 1) / 2 > e) --t;
  while ((t + 1) * (t + 2) / 2 <= e) ++t;
  c2 = t;
  c1 = e - t * (t + 1) / 2;
}

__global__ void __launch_bounds__(512) gram_kernel(int mode, int n, int l, const double* __restrict__ Yin,
                                                   const double* __restrict__ T, const double* __restrict__ lam,
                                                   uint64_t seed, uint32_t mode1, int step,
                                                   double* __restrict__ Xout, double* __restrict__ gpart,
                                                   int* __restrict__ status, double* __restrict__ Qo,
                                                   float* __restrict__ Qo32) {
  extern __shared__ double sm[];
  const int ldx = l + 1;
  double* Xs = sm;                       // [kGB][l+1]
  double* Ts = Xs + kGB * ldx;           // [l][l] (mode 1)
  const int i0 = blockIdx.x * kGB;
  const int rows = min(kGB, n - i0);
  const bool single = (mode == 1) && (status[3] == 0);
  if (mode == 1) {
    for (int idx = threadIdx.x; idx < l * l; idx += blockDim.x) Ts[idx] = T[idx];
  }
  for (int idx = threadIdx.x; idx < kGB * l; idx += blockDim.x) {
    const int c = idx / kGB, ii = idx % kGB;
    Xs[ii * ldx + c] = ii < rows ? Yin[(int64_t)c * n + i0 + ii] : 0.0;
  }
  __syncthreads();
  if (mode == 1) {
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
        const int64_t o = (int64_t)c * n + i0 + ii;
        Xout[o] = s;
        if (single) {
          Qo[o] = s;
          Qo32[o] = (float)s;
        }
      }
      outv[no] = s;
    }
    if (single) return;
    __syncthreads();
    no = 0;
    for (int idx = threadIdx.x; idx < kGB * l; idx += blockDim.x, ++no) {
      const int c = idx / kGB, ii = idx % kGB;
      Xs[ii * ldx + c] = outv[no];
    }
    __syncthreads();
  }
  const int np = l * (l + 1) / 2;
  double* gp = gpart + (int64_t)blockIdx.x * np;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    int c1, c2;
    unpack_index(e, c1, c2);
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

static size_t gram_smem(int l, int mode) {
  return sizeof(double) * ((size_t)kGB * (l + 1) + (mode ? (size_t)l * l : 0));
}

cudaError_t launch_reduce_gram(const ModeBufs& B, bool power, cudaStream_t st) {
  const int64_t tot = (int64_t)B.n * B.l;
  reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(B.Ypart, B.G, B.ltot, B.n_rows, B.n, B.l, B.Qd,
                                                               B.alpha, power ? 1 : 0, B.Y);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)gram_smem(96, 1));
  if (e != cudaSuccess) return e;
  gram_kernel<<<B.nblk, 512, gram_smem(B.l, 0), st>>>(0, B.n, B.l, B.Y, nullptr, nullptr, 0, 0, 0, nullptr,
                                                      B.gpart, B.status, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t launch_apply(const ModeBufs& B, uint64_t seed, uint32_t mode, int step, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)gram_smem(96, 1));
  if (e != cudaSuccess) return e;
  gram_kernel<<<B.nblk, 512, gram_smem(B.l, 1), st>>>(1, B.n, B.l, B.Y, B.T, B.lam, seed, mode, step, B.Q1,
                                                      B.gpart, B.status, B.Qd, B.Qs);
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

// ================================================================ one-CTA l x l solves
// unpack sum_b gpart[b] (packed upper) into a dense symmetric l x l array (ld = lda)
__device__ void sum_packed(const double* __restrict__ gpart, int nblk, int l, double* A, int lda) {
  const int np = l * (l + 1) / 2;
  for (int e = threadIdx.x; e < np; e += blockDim.x) {
    int c1, c2;
    unpack_index(e, c1, c2);
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * np + e];
    A[c1 * lda + c2] = s;
    A[c2 * lda + c1] = s;
  }
}

// Rotation (c, s) annihilating a_pq for the 2x2 block [[a_pp, a_pq], [a_pq, a_qq]]:
// t = 2 a_pq / (d + sgn(d) sqrt(d^2 + 4 a_pq^2)), d = a_qq - a_pp  (= sgn(theta)/(|theta| +
// sqrt(1+theta^2)) of sym.schur2).  t is evaluated in fp32 on exponent-scaled operands (an
// inexact angle only leaves a small residual that later sweeps remove); c = (1+t^2)^-1/2 is
// refined to fp64 by Newton steps so that (c, s = t c) is orthogonal to fp64 rounding.
__device__ __forceinline__ void rot_params(double apq, double d, double& c, double& s) {
  const double mx = fmax(fabs(d), fabs(apq));
  const int ex = (int)((__double_as_longlong(mx) >> 52) & 0x7ff) - 1023;
  const double sc = __longlong_as_double((long long)(1023 - ex) << 52);   // 2^-ex (exact)
  const float df = (float)(d * sc), af = (float)(apq * sc);
  const float den = df + copysignf(sqrtf(fmaf(df, df, 4.f * af * af)), df);
  const float tf = (den != 0.f) ? __fdividef(2.f * af, den) : 1.f;
  const double t = (double)tf;
  const double x = fma(t, t, 1.0);
  double y = (double)rsqrtf((float)x);
  y = y * fma(-0.5 * x * y, y, 1.5);
  y = y * fma(-0.5 * x * y, y, 1.5);
  c = y;
  s = t * y;
}

__device__ __forceinline__ void rr_pair(int rnd, int k, int le, int& p, int& q) {
  if (k == 0) { p = rnd; q = le - 1; }
  else { p = (rnd + k) % (le - 1); q = (rnd - k + (le - 1)) % (le - 1); }
  if (p > q) { const int t = p; p = q; q = t; }
}

// Parallel cyclic Jacobi on A (l x l, ld l) with V accumulated (V[row*l+col]); round-robin
// ordering, warp per pair-row: one lane per pair computes its rotation, then each lane of the
// warp of row-pair kr applies J^T A J to the 2x2 block (kr, kc) and V <- V J on pair kr's columns.
// A pair is skipped when |a_pq| <= 1e-15 sqrt(a_pp a_qq) or |a_pq| <= 1e-300; converged after
// a sweep without rotations (<= 40 sweeps).  Returns the sweep count.
__device__ int jacobi(double* A, double* V, int l, double* rc, double* rs, int2* tab) {
  __shared__ int any_rot;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int le = l + (l & 1), half = le / 2;
  for (int idx = tid; idx < l * l; idx += nt) V[idx] = (idx / l == idx % l) ? 1.0 : 0.0;
  for (int idx = tid; idx < (le - 1) * half; idx += nt) {
    int p, q;
    rr_pair(idx / half, idx % half, le, p, q);
    tab[idx] = make_int2(p, q);
  }
  int nsweep = 0;
  for (int sweep = 0; sweep < 40; ++sweep) {
    __syncthreads();
    if (tid == 0) any_rot = 0;
    for (int rnd = 0; rnd < le - 1; ++rnd) {
      const int2* tr = tab + rnd * half;
      for (int k = warp; k < half; k += nw) {
        if (lane == 0) {
          const int2 pq = tr[k];
          double c = 1.0, s = 0.0;
          if (pq.y < l) {
            const double apq = A[pq.x * l + pq.y], app = A[pq.x * l + pq.x], aqq = A[pq.y * l + pq.y];
            if (apq * apq > 1e-30 * fabs(app * aqq) && fabs(apq) > 1e-300) {
              rot_params(apq, aqq - app, c, s);
              any_rot = 1;
            }
          }
          rc[k] = c;
          rs[k] = s;
        }
      }
      __syncthreads();
      for (int kr = warp; kr < half; kr += nw) {
        const int2 rp = tr[kr];
        const double sr = rs[kr], cr = rc[kr];
        for (int kc = lane; kc < half; kc += 32) {
          const double sc = rs[kc];
          if (sr == 0.0 && sc == 0.0) continue;
          const double cc = rc[kc];
          const int2 cp = tr[kc];
          const int p = rp.x, q = rp.y, u = cp.x, w = cp.y;
          const bool hq = q < l, hw = w < l;      // (odd l: one dummy player)
          const double apu = A[p * l + u];
          const double apw = hw ? A[p * l + w] : 0.0;
          const double aqu = hq ? A[q * l + u] : 0.0;
          const double aqw = (hq && hw) ? A[q * l + w] : 0.0;
          const double bpu = cr * apu - sr * aqu, bqu = sr * apu + cr * aqu;
          const double bpw = cr * apw - sr * aqw, bqw = sr * apw + cr * aqw;
          A[p * l + u] = cc * bpu - sc * bpw;
          if (hw) A[p * l + w] = sc * bpu + cc * bpw;
          if (hq) A[q * l + u] = cc * bqu - sc * bqw;
          if (hq && hw) A[q * l + w] = sc * bqu + cc * bqw;
        }
        if (sr != 0.0 && rp.y < l) {
          for (int j = lane; j < l; j += 32) {
            const double vp = V[j * l + rp.x], vq = V[j * l + rp.y];
            V[j * l + rp.x] = cr * vp - sr * vq;
            V[j * l + rp.y] = sr * vp + cr * vq;
          }
        }
      }
      __syncthreads();
    }
    const int rotated = any_rot;
    nsweep = sweep + 1;
    if (!rotated) break;
  }
  __syncthreads();
  return nsweep;
}

// In-place Cholesky A = R^T R (upper R written over the upper triangle, lda), one barrier per
// column.  Returns false (uniformly) on a non-positive or relatively tiny pivot.
__device__ bool cholesky(double* A, int l, int lda) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double dmax = 0.0;
  for (int k = 0; k < l; ++k) dmax = fmax(dmax, A[k * lda + k]);
  for (int k = 0; k < l; ++k) {
    const double d = A[k * lda + k];
    if (!(d > 1e-13 * dmax) || !isfinite(d)) return false;
    const double inv = 1.0 / d;
    const int w = l - k - 1;
    for (int idx = tid; idx < w * w; idx += nt) {
      const int i = k + 1 + idx / w, j = k + 1 + idx % w;
      if (j >= i) A[i * lda + j] -= A[k * lda + i] * A[k * lda + j] * inv;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < l * l; idx += nt) {
    const int k = idx / l, j = idx % l;
    if (j > k) A[k * lda + j] /= sqrt(A[k * lda + k]);
  }
  __syncthreads();
  for (int k = tid; k < l; k += nt) A[k * lda + k] = sqrt(A[k * lda + k]);
  __syncthreads();
  return true;
}

// X = R^{-1} (upper), thread per column; X stored transposed: X[c*ldx + i].
__device__ void tri_inverse(const double* R, int l, int lda, double* X, int ldx) {
  __shared__ double rinv[128];
  for (int i = threadIdx.x; i < l; i += blockDim.x) rinv[i] = 1.0 / R[i * lda + i];
  __syncthreads();
  for (int c = threadIdx.x; c < l; c += blockDim.x) {
    double* xc = X + c * ldx;
    for (int i = 0; i < l; ++i) xc[i] = 0.0;
    xc[c] = rinv[c];
    for (int i = c - 1; i >= 0; --i) {
      const double* ri = R + i * lda;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int j = i + 1;
      for (; j + 4 <= c + 1; j += 4) {
        s0 += ri[j] * xc[j];
        s1 += ri[j + 1] * xc[j + 1];
        s2 += ri[j + 2] * xc[j + 2];
        s3 += ri[j + 3] * xc[j + 3];
      }
      for (; j <= c; ++j) s0 += ri[j] * xc[j];
      xc[i] = -((s0 + s1) + (s2 + s3)) * rinv[i];
    }
  }
  __syncthreads();
}

// Householder tridiagonalisation of the symmetric A (l x l, lda; destroyed) by the whole CTA:
// T = H^T A H with diagonal d[0..l) and off-diagonal e[0..l-1).  p: l scratch.
// Per reflection k: every warp recomputes the column norm (no barrier), warps form
// p = beta A_sub v row by row (barrier), every thread recomputes K = beta/2 p^T v and applies
// A_sub -= v w^T + w v^T with w = p - K v (barrier).  v is read from column k of A, which the
// trailing update never touches.
__device__ void tridiag_cta(double* A, int l, int lda, double* d, double* e, double* p) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int k = 0; k + 2 < l; ++k) {
    const int m = l - k - 1;
    const int b = k + 1;
    double s = 0.0;
    for (int i = lane + 1; i < m; i += 32) { const double x = A[(b + i) * lda + k]; s += x * x; }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double x0 = A[b * lda + k];
    if (tid == 0) d[k] = A[k * lda + k];
    if (s == 0.0) {             // column already reduced (uniform decision)
      if (tid == 0) e[k] = x0;
      __syncthreads();
      continue;
    }
    const double nrm = sqrt(s + x0 * x0);
    const double alph = x0 > 0.0 ? -nrm : nrm;
    const double v0 = x0 - alph;
    const double beta = 2.0 / (s + v0 * v0);
    // p_i = beta * sum_j A_sub(i, j) v_j  (warp per row)
    for (int i = warp; i < m; i += nw) {
      const double* ar = A + (b + i) * lda + b;
      double acc = 0.0;
      for (int j = lane; j < m; j += 32) acc += ar[j] * (j == 0 ? v0 : A[(b + j) * lda + k]);
#pragma unroll
      for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) p[i] = beta * acc;
    }
    if (tid == 0) e[k] = alph;
    __syncthreads();
    double dot = 0.0;
    for (int j = lane; j < m; j += 32) dot += p[j] * (j == 0 ? v0 : A[(b + j) * lda + k]);
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    const double K = 0.5 * beta * dot;
    for (int i = warp; i < m; i += nw) {
      const double vi = i == 0 ? v0 : A[(b + i) * lda + k];
      const double wi = p[i] - K * vi;
      double* ar = A + (b + i) * lda + b;
      for (int j = lane; j < m; j += 32) {
        const double vj = j == 0 ? v0 : A[(b + j) * lda + k];
        const double wj = p[j] - K * vj;
        ar[j] -= vi * wj + wi * vj;
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    d[l - 2] = A[(l - 2) * lda + (l - 2)];
    d[l - 1] = A[(l - 1) * lda + (l - 1)];
    e[l - 2] = A[(l - 1) * lda + (l - 2)];
  }
  __syncthreads();
}

// # eigenvalues of the tridiagonal (d, e) below mu (Sturm sequence / LDL^T inertia).  The
// division uses a fp32 reciprocal refined by two Newton steps (relative error ~1e-16): the
// count only needs the signs of the pivots.
__device__ __forceinline__ double fast_rcp(double x) {
  const float xf = (float)x;
  double y = (double)__frcp_rn(xf);
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

__device__ __forceinline__ int sturm_count(const double* d, const double* e2, int l, double mu) {
  int cnt = 0;
  double q = d[0] - mu;
  cnt += q < 0.0;
  for (int i = 1; i < l; ++i) {
    if (fabs(q) < 1e-280) q = q < 0.0 ? -1e-280 : 1e-280;
    q = (d[i] - mu) - e2[i - 1] * fast_rcp(q);
    cnt += q < 0.0;
  }
  return cnt;
}

// lambda_min of the tridiagonal by multisection on the first kMS threads: one log-spaced
// round over [hi 2^-60, hi] (hi = min_i d_i >= lambda_min) then linear rounds until the
// bracket is below 1e-13 relative.  Called by the whole CTA (barriers inside).
constexpr int kMS = 128;
__device__ double lambda_min_multisection(const double* d, const double* e2, int l) {
  __shared__ double lo_s, hi_s;
  __shared__ int best;
  const int tid = threadIdx.x;
  if (tid == 0) {
    double hi = d[0];
    for (int i = 1; i < l; ++i) hi = fmin(hi, d[i]);
    hi_s = hi;
    lo_s = 0.0;
  }
  __syncthreads();
  const double hi0 = hi_s;
  if (!(hi0 > 0.0) || sturm_count(d, e2, l, 0.0) > 0) return 0.0;
  const double lg = log2(hi0);
  for (int round = 0; round < 12; ++round) {
    const double lo = lo_s, hi = hi_s;
    if (hi - lo <= 1e-13 * hi) break;
    auto point = [&](int j) {   // j in [0, kMS]: the multisection grid (deterministic)
      if (round == 0) return j == 0 ? 0.0 : exp2(lg - 60.0 * (1.0 - (double)j / kMS));
      return lo + (hi - lo) * (double)j / kMS;
    };
    if (tid == 0) best = kMS;
    __syncthreads();
    if (tid < kMS && sturm_count(d, e2, l, point(tid + 1)) > 0) atomicMin(&best, tid);
    __syncthreads();
    if (tid == 0) {
      const int j = best;          // smallest grid index whose point exceeds lambda_min
      hi_s = j < kMS ? point(j + 1) : hi;
      lo_s = j < kMS ? point(j) : point(kMS);
      if (round == 0 && j == kMS) lo_s = hi;   // lambda_min == hi
    }
    __syncthreads();
  }
  return 0.5 * (lo_s + hi_s);
}

// One CTA: G = sum of packed partials; orthonormalising transform T (l x l, column-major) and,
// for power steps (step >= 1), the shift update from Sigma_ll = sqrt(lambda_min(G)).
__global__ void __launch_bounds__(kOrthThreads) orth_kernel(const double* __restrict__ gpart, int nblk, int l,
                                                            int step, int final_step, int shift,
                                                            double* __restrict__ alpha, double* __restrict__ T,
                                                            double* __restrict__ lam_out,
                                                            double* __restrict__ trace,
                                                            double* __restrict__ sigma, int* __restrict__ status) {
  extern __shared__ double sm[];
  const int le = l + (l & 1), half = le / 2;
  double* A = sm;                  // [l][l] Gram (kept for the fallback)
  double* W1 = A + l * l;          // [l][l] Cholesky factor / Jacobi V
  double* W2 = W1 + l * l;         // [l][l] R^{-1} (transposed) / tridiagonal work copy
  double* rc = W2 + l * l;         // [half]
  double* rs = rc + half;          // [half]
  double* ev = rs + half;          // [l]
  double* td = ev + l;             // [l] tridiagonal d
  double* te = td + l;             // [l] tridiagonal e, then e^2
  double* vw = te + l;             // [2l]
  int* rank = (int*)(vw + 2 * l);  // [l]
  int2* tab = (int2*)(rank + l + (l & 1));   // [le-1][half]
  __shared__ double al_old, lam_min_s;
  __shared__ int use_eig;
  const int tid = threadIdx.x, nt = blockDim.x;

  long long tclk[6];
  tclk[0] = clock64();
  sum_packed(gpart, nblk, l, A, l);
  if (tid == 0) use_eig = final_step;
  __syncthreads();
  tclk[1] = clock64();
  if (!use_eig) {
    for (int idx = tid; idx < l * l; idx += nt) W1[idx] = A[idx];
    __syncthreads();
    const bool ok = cholesky(W1, l, l);
    if (!ok && tid == 0) use_eig = 1;   // breakdown -> Jacobi basis with completion
    __syncthreads();
  }
  if (!use_eig) {
    // ---------------- CholQR path: T = R^{-1}; lambda_min for the shift
    tclk[2] = clock64();
    tri_inverse(W1, l, l, W2, l);
    for (int idx = tid; idx < l * l; idx += nt) {
      const int i = idx % l, c = idx / l;
      T[i + (int64_t)l * c] = W2[c * l + i];
    }
    for (int c = tid; c < l; c += nt) lam_out[c] = 1.0;    // every column valid
    if (tid == 0) status[3] = 1;                            // CholQR always takes the second pass
    double lmin = 0.0;
    if (step > 0) {
      __syncthreads();
      for (int idx = tid; idx < l * l; idx += nt) W2[idx] = A[idx];
      __syncthreads();
      tclk[3] = clock64();
      tridiag_cta(W2, l, l, td, te, vw);
      __syncthreads();
      for (int i = tid; i < l - 1; i += nt) te[i] = te[i] * te[i];
      __syncthreads();
      tclk[4] = clock64();
      lmin = lambda_min_multisection(td, te, l);
      tclk[5] = clock64();
      if (tid == 0) for (int z = 0; z < 5; ++z) sigma[110 + z] = (double)(tclk[z + 1] - tclk[z]);
    }
    if (tid == 0) lam_min_s = lmin;
  } else {
    // ---------------- Jacobi path: T = V Sigma^{-1} in descending order
    const int sw = jacobi(A, W1, l, rc, rs, tab);
    if (tid == 0) { sigma[127] = (double)sw; if (step < 24) sigma[100 + step] = (double)sw; }
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
    const double s1 = sqrt(fmax(ev[0], 0.0));
    for (int i = tid; i < l; i += nt) {
      const double sg = sqrt(fmax(ev[i], 0.0));
      lam_out[i] = (sg > 1e-12 * s1 && sg > 1e-200) ? ev[i] : -1.0;   // -1: rank-deficient column
    }
    if (tid == 0) {
      const bool ok = ev[l - 1] > 0.0 && ev[0] <= 1e6 * ev[l - 1] && sqrt(ev[l - 1]) > 1e-12 * s1;
      status[3] = ok ? 0 : 1;   // second CholQR pass only if Q1 can lose orthogonality
      lam_min_s = fmax(ev[l - 1], 0.0);
    }
    for (int idx = tid; idx < l * l; idx += nt) {
      const int row = idx / l, col = idx % l;
      const int rk = rank[col];
      const double sg = sqrt(fmax(A[col * l + col], 0.0));
      const bool ok = sg > 1e-12 * s1 && sg > 1e-200;
      T[row + (int64_t)l * rk] = ok ? W1[row * l + col] / sg : 0.0;
    }
  }
  __syncthreads();
  // ---------------- shift update (Alg. 3/4 lines 8-9; degenerate guard SPEC.md:347)
  if (tid == 0) {
    const double a0 = (step > 0) ? *alpha : 0.0;
    double s1 = 0.0;
    if (use_eig) {
      s1 = sqrt(fmax(ev[0], 0.0));
    } else {
      double gmax = 0.0;               // sigma_1^2 >= max_i G_ii
      for (int i = 0; i < l; ++i) gmax = fmax(gmax, A[i * l + i]);
      s1 = sqrt(gmax);
    }
    const double sl = sqrt(lam_min_s);
    double a1 = a0;
    if (step > 0 && shift && sl > a0 && !(sl < 1e-14 * s1)) a1 = 0.5 * (sl + a0);
    if (step > 0) {
      *alpha = a1;
      trace[step - 1] = a1;
      status[2] = step;
    }
    al_old = a0;
    sigma[126] = sl;
  }
  __syncthreads();
  if (use_eig) {
    for (int i = tid; i < l; i += nt) sigma[i] = sqrt(fmax(ev[i], 0.0)) + al_old;  // B.1 sigma
  }
}

static size_t orth_smem(int l) {
  const int le = l + (l & 1), half = le / 2;
  return sizeof(double) * (3 * (size_t)l * l + 2 * half + 5 * l) + sizeof(int) * (l + (l & 1)) +
         sizeof(int2) * (size_t)(le - 1) * half + 64;
}

cudaError_t launch_eig(const ModeBufs& B, int step, int q, bool shift, double pve_tol, cudaStream_t st) {
  (void)pve_tol;
  const size_t smem = orth_smem(B.l);
  cudaError_t e = cudaFuncSetAttribute(orth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  orth_kernel<<<1, kOrthThreads, smem, st>>>(B.gpart, B.nblk, B.l, step, step == q ? 1 : 0, shift ? 1 : 0,
                                             B.alpha, B.T, B.lam, B.trace, B.sigma, B.status);
  return cudaGetLastError();
}

// ------------------------------------------------------- second CholQR pass
// G2 = Q1^T Q1 = R^T R, T2 = R^{-1}  (no-op when the first pass already suffices)
__global__ void __launch_bounds__(1024) chol_kernel(const double* __restrict__ gpart, int nblk, int l,
                                                    double* __restrict__ T2, int* __restrict__ status) {
  if (!status[3]) return;
  extern __shared__ double sm[];
  double* A = sm;            // [l][l]
  double* X = A + l * l;     // [l][l] R^{-1} transposed
  const int tid = threadIdx.x, nt = blockDim.x;
  sum_packed(gpart, nblk, l, A, l);
  __syncthreads();
  if (!cholesky(A, l, l)) {
    if (tid == 0) status[0] = 6;   // RTK_ERR_NUMERIC: Q1 numerically rank deficient
    for (int idx = tid; idx < l * l; idx += nt) T2[idx] = (idx % l == idx / l) ? 1.0 : 0.0;
    return;
  }
  tri_inverse(A, l, l, X, l);
  for (int idx = tid; idx < l * l; idx += nt) {
    const int i = idx % l, c = idx / l;
    T2[i + (int64_t)l * c] = X[c * l + i];
  }
}

cudaError_t launch_chol(const ModeBufs& B, cudaStream_t st) {
  const size_t smem = sizeof(double) * 2 * B.l * B.l;
  cudaError_t e = cudaFuncSetAttribute(chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  chol_kernel<<<1, 1024, smem, st>>>(B.gpart, B.nblk, B.l, B.T, B.status);
  return cudaGetLastError();
}

// ------------------------------------------------------------ Q = Q1 T2
__global__ void __launch_bounds__(256) apply2_kernel(const double* __restrict__ Q1,
                                                     const double* __restrict__ T2, int n, int l,
                                                     double* __restrict__ Qd, float* __restrict__ Qs,
                                                     const int* __restrict__ status) {
  if (!status[3]) return;
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
  apply2_kernel<<<(B.n + kRB - 1) / kRB, 256, smem, st>>>(B.Q1, B.T, B.n, l, B.Qd, B.Qs, B.status);
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
  // ties: |entries| within 1e-5 of the maximum count as tied, lowest row wins (reading C6)
  const double thr = (1.0 - 1e-5) * sb[0];
  __shared__ int piv;
  if (threadIdx.x == 0) piv = 0x7fffffff;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (fabs(col[i]) >= thr) { atomicMin(&piv, i); break; }
  __syncthreads();
  const double sg = col[piv == 0x7fffffff ? 0 : piv] < 0.0 ? -1.0 : 1.0;
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
