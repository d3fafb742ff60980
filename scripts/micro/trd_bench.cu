// Isolated timing (clock64, one CTA) of the Householder tridiagonalisation with the accumulated
// reflector product, rtk_solve.cu's tridiag_t<true> (every warp rebuilds reflector k from the
// published pivot row); checks QH^T G QH = tridiag(d, e).  (The one-quad-reflector version it
// replaced measured 192k cycles at l = 60; this one 136k.)
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o trd_bench trd_bench.cu
#include "../../paper_2506_04840_b200/csrc/rtk_solve.cu"
#include <cstdio>
#include <vector>
#include <random>
#include <cmath>
namespace rtk { int num_sms() { return 148; } bool pdl_enabled() { return false; } }
using namespace rtk;


template <int V>
__global__ void __launch_bounds__(256, 1) bench(const double* Gg, int l, long long* clk, double* out) {
  extern __shared__ __align__(16) uint8_t smraw[];
  StepSmem& S = *reinterpret_cast<StepSmem*>(smraw);
  const int tid = threadIdx.x;
  for (int i = tid; i < l * l; i += 256) S.G[(i / l) * kLD + i % l] = Gg[i];
  __syncthreads();
  long long t0 = clock64();
  tridiag_t<true>(S.G, l, S.H, S.hb, S.d, S.e, S.pbuf, S.xrow, S.scal, S.T);
  long long t1 = clock64();
  if (tid == 0) clk[0] = t1 - t0;
  for (int i = tid; i < l; i += 256) { out[i] = S.d[i]; out[l + i] = S.e[i]; }
  for (int i = tid; i < l * l; i += 256) out[2 * l + i] = S.T[(i / l) * kLD + i % l];
}

int main(int argc, char** argv) {
  const int l = argc > 1 ? atoi(argv[1]) : 60, n = 1000;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> Y((size_t)n * l), G(l * l);
  for (int c = 0; c < l; ++c)
    for (int i = 0; i < n; ++i) Y[(size_t)c * n + i] = nd(g) * std::pow(0.8, c);
  for (int a = 0; a < l; ++a)
    for (int b = 0; b < l; ++b) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += Y[(size_t)a * n + i] * Y[(size_t)b * n + i];
      G[a * l + b] = s;
    }
  double *dG, *dout;
  long long* dclk;
  const size_t no = 2 * l + l * l;
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
  double dd = 0, dq = 0, nrm = 0, res = 0;
  for (int i = 0; i < l; ++i) nrm = std::fmax(nrm, std::fabs(o[i]));
  for (int i = 0; i < 2 * l; ++i) dd = std::fmax(dd, std::fabs(o[i] - o[no + i]));
  for (int i = 0; i < l * l; ++i) dq = std::fmax(dq, std::fabs(o[2 * l + i] - o[no + 2 * l + i]));
  // residual of the candidate: QH^T G QH - tridiag(d, e)
  const double* Q = o.data() + no + 2 * l;
  for (int a = 0; a < l; ++a)
    for (int b = 0; b < l; ++b) {
      double s = 0;
      for (int x = 0; x < l; ++x)
        for (int y = 0; y < l; ++y) s += Q[x * l + a] * G[x * l + y] * Q[y * l + b];
      double t = a == b ? o[no + a] : (std::abs(a - b) == 1 ? o[no + l + std::min(a, b)] : 0.0);
      res = std::fmax(res, std::fabs(s - t));
    }
  printf("l=%d %s current %lld cycles, trd2 %lld cycles | max|d,e diff| %.2e max|QH diff| %.2e  |Q^T G Q - T|max %.2e (|d|max %.3e)\n",
         l, cudaGetErrorString(e), c0, c1, dd, dq, res, nrm);
  return 0;
}
