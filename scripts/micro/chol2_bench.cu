// Candidate Cholesky for the step kernel, timed against rtk_solve.cu's blocked chol_upper on one CTA:
// right-looking by single columns on the tridiagonalisation's layout (thread (i = tid/4, part =
// tid%4) keeps A(i, part + 4jj) in registers), one barrier per column: the quad of row k+1 forms
// R's row k+1 right after its own update of step k and publishes it; every row then subtracts
// r_ki r_kj from its entries with broadcast loads of row k.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o chol2_bench chol2_bench.cu
#include "../../paper_2506_04840_b200/csrc/rtk_solve.cu"
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
namespace rtk { int num_sms() { return 148; } bool pdl_enabled() { return false; } }
using namespace rtk;

__device__ __noinline__ bool chol_cols(const double* A, double* R, double* flag, int l) {
  const int tid = threadIdx.x, i = tid >> 2, part = tid & 3;
  const int src = (tid & 31) & ~3;
  double a[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const int j = part + 4 * jj;
    a[jj] = (i < l && j < l) ? A[min(i, j) * kLD + max(i, j)] : (i == j ? 1.0 : 0.0);
  }
  double dmax = 0.0;
  for (int k = 0; k < l; ++k) dmax = fmax(dmax, A[k * kLD + k]);
  const double tol = 1e-13 * dmax;
  if (tid == 0) flag[0] = 0.0;
  // quad k forms and publishes row k of R (zero left of the diagonal), all 64 columns
  auto publish = [&](int k) {
    double piv = 0.0;
#pragma unroll
    for (int jj = 0; jj < 16; ++jj)
      if (part + 4 * jj == k) piv = a[jj];
    piv = __shfl_sync(0xffffffffu, piv, src | (k & 3));
    if (i == k) {
      const bool bad = !(piv > tol) || !(piv < DBL_MAX);
      const double rs = bad ? 0.0 : rsqrt_fast(piv);
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        const int j = part + 4 * jj;
        R[k * kLD + j] = j < k ? 0.0 : a[jj] * rs;
      }
      if (bad && part == 0) flag[0] = 1.0;
    }
  };
  if (i < 8) publish(0);
  for (int k = 0; k < l; ++k) {
    __syncthreads();   // row k of R published
    if (flag[0] != 0.0) return false;
    if (k + 1 == l) break;
    if (i > k && i < l) {
      const double rki = R[k * kLD + i];
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) a[jj] = fma(-rki, R[k * kLD + part + 4 * jj], a[jj]);
    }
    if ((i >> 3) == ((k + 1) >> 3)) publish(k + 1);   // the warp holding row k+1 (full-warp shuffle)
  }
  for (int idx = tid; idx < (kSL - l) * kSL; idx += kST) {   // identity rows l..63
    const int k = l + idx / kSL, j = idx % kSL;
    R[k * kLD + j] = (k == j) ? 1.0 : 0.0;
  }
  __syncthreads();
  return true;
}

template <int V>
__global__ void __launch_bounds__(256, 1) bench(const double* Gg, int l, long long* clk, double* out) {
  extern __shared__ __align__(16) uint8_t smraw[];
  StepSmem& S = *reinterpret_cast<StepSmem*>(smraw);
  const int tid = threadIdx.x;
  for (int i = tid; i < l * l; i += 256) S.G[(i / l) * kLD + i % l] = Gg[i];
  __syncthreads();
  long long t0 = clock64();
  const bool ok = V == 0 ? chol_upper(S.G, S.R, S.rowbuf, l) : chol_cols(S.G, S.R, S.rowbuf, l);
  long long t1 = clock64();
  if (tid == 0) { clk[0] = t1 - t0; out[0] = ok; }
  for (int i = tid; i < kSL * kSL; i += 256) out[1 + i] = S.R[(i / kSL) * kLD + i % kSL];
}

int main(int argc, char** argv) {
  const int l = argc > 1 ? atoi(argv[1]) : 60, n = 1000;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> Y((size_t)n * l), G(l * l);
  for (int c = 0; c < l; ++c)
    for (int i = 0; i < n; ++i) Y[(size_t)c * n + i] = nd(g) * std::pow(0.85, c);
  for (int a = 0; a < l; ++a)
    for (int b = 0; b < l; ++b) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += Y[(size_t)a * n + i] * Y[(size_t)b * n + i];
      G[a * l + b] = s;
    }
  double *dG, *dout;
  long long* dclk;
  const int no = 1 + kSL * kSL;
  cudaMalloc(&dG, l * l * 8);
  cudaMalloc(&dout, 2 * no * 8);
  cudaMalloc(&dclk, 64);
  cudaMemcpy(dG, G.data(), l * l * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StepSmem));
  cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StepSmem));
  long long c0 = 0, c1 = 0;
  for (int r = 0; r < 3; ++r) {
    bench<0><<<1, 256, sizeof(StepSmem)>>>(dG, l, dclk, dout);
    cudaMemcpy(&c0, dclk, 8, cudaMemcpyDeviceToHost);
    bench<1><<<1, 256, sizeof(StepSmem)>>>(dG, l, dclk + 1, dout + no);
    cudaMemcpy(&c1, dclk + 1, 8, cudaMemcpyDeviceToHost);
  }
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> o(2 * no);
  cudaMemcpy(o.data(), dout, 2 * no * 8, cudaMemcpyDeviceToHost);
  double dr = 0, rn = 0, res = 0, gn = 0;
  for (int i = 0; i < kSL * kSL; ++i) {
    dr = std::fmax(dr, std::fabs(o[1 + i] - o[no + 1 + i]));
    rn = std::fmax(rn, std::fabs(o[1 + i]));
  }
  const double* R = o.data() + no + 1;
  for (int a = 0; a < l; ++a)
    for (int b = 0; b < l; ++b) {
      double s = 0;
      for (int k = 0; k < l; ++k) s += R[k * kSL + a] * R[k * kSL + b];
      res = std::fmax(res, std::fabs(s - G[a * l + b]));
      gn = std::fmax(gn, std::fabs(G[a * l + b]));
    }
  int pad_ok = 1;   // identity / zero padding beyond l
  for (int a = 0; a < kSL; ++a)
    for (int b = 0; b < kSL; ++b)
      if (a >= l || b >= l) pad_ok &= (R[a * kSL + b] == (a == b ? 1.0 : 0.0)) || (a < b && a >= l && false);
  printf("l=%d %s blocked %lld cycles, columns %lld cycles | ok %g %g | max|R diff|/max|R| %.2e  |R'R-G|/|G| %.2e pad %d\n",
         l, cudaGetErrorString(e), c0, c1, o[0], o[no], dr / rn, res / gn, pad_ok);
  return 0;
}
