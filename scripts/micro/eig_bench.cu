// Microbenchmark of the one-CTA Jacobi (rtk_small.cu eig_kernel) on a random SPD Gram.
#include "../../paper_2506_04840_b200/csrc/rtk_small.cu"
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
using namespace rtk;
int main(int argc, char** argv) {
  int l = argc > 1 ? atoi(argv[1]) : 60;
  int n = 1000;
  std::mt19937_64 g(1);
  std::normal_distribution<double> nd;
  std::vector<double> Y((size_t)n * l), P(l * (l + 1) / 2);
  for (int c = 0; c < l; ++c)
    for (int i = 0; i < n; ++i) Y[(size_t)c * n + i] = nd(g) * (1.0 + c);
  for (int c2 = 0; c2 < l; ++c2)
    for (int c1 = 0; c1 <= c2; ++c1) {
      double s = 0;
      for (int i = 0; i < n; ++i) s += Y[(size_t)c1 * n + i] * Y[(size_t)c2 * n + i];
      P[c2 * (c2 + 1) / 2 + c1] = s;
    }
  ModeBufs B;
  B.l = l; B.n = n; B.r = l - 10; B.nblk = 1;
  cudaMalloc(&B.gpart, P.size() * 8);
  cudaMemcpy(B.gpart, P.data(), P.size() * 8, cudaMemcpyHostToDevice);
  cudaMalloc(&B.T, l * l * 8); cudaMalloc(&B.lam, l * 8); cudaMalloc(&B.alpha, 8); cudaMemset(B.alpha, 0, 8);
  cudaMalloc(&B.trace, 64 * 8); cudaMalloc(&B.sigma, 128 * 8); cudaMalloc(&B.status, 16); cudaMemset(B.status, 0, 16);
  for (int i = 0; i < 3; ++i) launch_eig(B, argc > 2 ? atoi(argv[2]) : 1, 5, true, 0.0, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int i = 0; i < reps; ++i) launch_eig(B, argc > 2 ? atoi(argv[2]) : 1, 5, true, 0.0, 0);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double sig[128]; cudaMemcpy(sig, B.sigma, 128 * 8, cudaMemcpyDeviceToHost);
  printf("l=%d eig %.1f us/call, sweeps %.0f, err=%s  clk: sum %.0f chol %.0f inv %.0f tridiag %.0f ms %.0f\n", l, ms * 1e3 / reps, sig[127], cudaGetErrorString(cudaGetLastError()), sig[110], sig[111], sig[112], sig[113], sig[114]);
  return 0;
}
