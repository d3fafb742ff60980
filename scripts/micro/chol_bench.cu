// Isolated timing (clock64) of the l x l building blocks of rtk_solve.cu on one CTA.
#include "../../paper_2506_04840_b200/csrc/rtk_solve.cu"
#include <cstdio>
#include <vector>
#include <random>
namespace rtk { int num_sms() { return 148; } bool pdl_enabled() { return false; } }
using namespace rtk;
__global__ void __launch_bounds__(256, 1) bench(const double* Gg, int l, long long* clk, double* out) {
  extern __shared__ __align__(16) uint8_t smraw[];
  StepSmem& S = *reinterpret_cast<StepSmem*>(smraw);
  const int tid = threadIdx.x;
  for (int i = tid; i < l * l; i += 256) S.G[(i / l) * kLD + i % l] = Gg[i];
  __syncthreads();
  long long t0 = clock64();
  bool ok = chol_upper(S.G, S.R, S.rowbuf, l);
  long long t1 = clock64();
  tri_inv_upper(S.R, S.T, l, S.rowbuf);
  long long t2 = clock64();
  tridiag(S.G, l, S.H, S.hb, S.d, S.e, S.pbuf, S.xrow, S.scal);
  long long t3 = clock64();
  for (int k = tid; k + 1 < l; k += kST) S.e2[k] = S.e[k] * S.e[k];
  __syncthreads();
  double lm = lambda_min_ms(S.d, S.e2, l, S.ibuf, S.dbuf);
  long long t4 = clock64();
  __syncthreads();
  long long t5 = clock64();
  __syncthreads();
  long long t6 = clock64();
  if (tid == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; clk[3] = t4 - t3; clk[4] = t6 - t5; out[0] = lm; out[1] = ok; }
  for (int i = tid; i < l * l; i += 256) { out[2 + i] = S.R[(i / l) * kLD + i % l]; out[2 + l * l + i] = S.T[(i / l) * kMLD + i % l]; }
}
int main(int argc, char** argv) {
  int l = argc > 1 ? atoi(argv[1]) : 60, n = 1000;
  std::mt19937_64 g(1); std::normal_distribution<double> nd;
  std::vector<double> Y((size_t)n * l), G(l * l);
  for (int c = 0; c < l; ++c) for (int i = 0; i < n; ++i) Y[(size_t)c * n + i] = nd(g) * (1.0 + 0.1 * c);
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) { double s = 0; for (int i = 0; i < n; ++i) s += Y[(size_t)a * n + i] * Y[(size_t)b * n + i]; G[a * l + b] = s; }
  double *dG, *dout; long long* dclk;
  cudaMalloc(&dG, l * l * 8); cudaMalloc(&dout, (2 + 2 * l * l) * 8); cudaMalloc(&dclk, 64);
  cudaMemcpy(dG, G.data(), l * l * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(StepSmem));
  for (int r = 0; r < 3; ++r) bench<<<1, 256, sizeof(StepSmem)>>>(dG, l, dclk, dout);
  cudaError_t e = cudaDeviceSynchronize();
  long long clk[5]; std::vector<double> out(2 + 2 * l * l);
  cudaMemcpy(clk, dclk, 40, cudaMemcpyDeviceToHost); cudaMemcpy(out.data(), dout, out.size() * 8, cudaMemcpyDeviceToHost);
  // check R^T R = G and R T = I
  double e1 = 0, e2 = 0, nG = 0;
  for (int a = 0; a < l; ++a) for (int b = 0; b < l; ++b) {
    double s = 0, t = 0;
    for (int k = 0; k < l; ++k) { s += out[2 + k * l + a] * out[2 + k * l + b]; t += out[2 + a * l + k] * out[2 + l * l + k * l + b]; }
    e1 += (s - G[a * l + b]) * (s - G[a * l + b]); nG += G[a * l + b] * G[a * l + b]; e2 += (t - (a == b)) * (t - (a == b));
  }
  printf("l=%d %s ok=%g chol %lld inv %lld tridiag %lld lammin %lld sync %lld cycles | |R'R-G|/|G| %.2e |RT-I| %.2e lam_min %.10g\n", l,
         cudaGetErrorString(e), out[1], clk[0], clk[1], clk[2], clk[3], clk[4], sqrt(e1 / nG), sqrt(e2), out[0]);
  return 0;
}
