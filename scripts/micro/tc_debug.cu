// Standalone checks of the tcgen05 op1 / op2 kernels (rtk_tc.cu) against a host fp64 reference.
#include "../../paper_2506_04840_b200/csrc/rtk_tc.cu"
#include <cstdio>
#include <random>
#include <vector>
namespace rtk { int num_sms() { return 148; } }
using namespace rtk;
int main(int argc, char** argv) {
  int n = argc > 1 ? atoi(argv[1]) : 128, m = argc > 2 ? atoi(argv[2]) : 256, l = argc > 3 ? atoi(argv[3]) : 16;
  int N = tc_npad(l);
  std::mt19937_64 g(1); std::normal_distribution<float> nd;
  std::vector<float> M((size_t)n * m), Q((size_t)n * l);
  for (auto& x : M) x = nd(g);
  for (auto& x : Q) x = nd(g);
  float *dM, *dQ, *dP, *dW, *dY; 
  cudaMalloc(&dM, M.size() * 4); cudaMalloc(&dQ, Q.size() * 4);
  int ldp = (n + 3) / 4 * 4; int64_t ldw = (m + 3) / 4 * 4; int nit = (n + 127) / 128; int G = 8;
  cudaMalloc(&dP, (size_t)2 * N * ldp * 4); cudaMalloc(&dW, (size_t)2 * N * ldw * 4); cudaMalloc(&dY, (size_t)G * N * nit * 128 * 4);
  cudaMemcpy(dM, M.data(), M.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dQ, Q.data(), Q.size() * 4, cudaMemcpyHostToDevice);
  View v; v.base = dM; v.n = n; v.P = 1; v.S = m; v.sp = 1; v.si = 1; v.ss = n;
  printf("supported %d\n", (int)tc_supported(v, l));
  cudaError_t e = tc_split(nullptr, dQ, n, l, dP, 0); printf("split %s\n", cudaGetErrorString(e));
  e = tc_op1(v, l, dP, dW, ldw, false, nullptr, 1, 1, 1, 0); printf("op1 launch %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize(); printf("op1 sync %s\n", cudaGetErrorString(e));
  std::vector<float> W((size_t)2 * N * ldw);
  cudaMemcpy(W.data(), dW, W.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  std::vector<double> Wref((size_t)m * l);
  for (int j = 0; j < m; ++j) for (int c = 0; c < l; ++c) {
    double s = 0; for (int i = 0; i < n; ++i) s += (double)M[(size_t)j * n + i] * Q[(size_t)c * n + i];
    Wref[(size_t)c * m + j] = s;
    double got = (double)W[(size_t)c * ldw + j] + (double)W[(size_t)(N + c) * ldw + j];
    err += (got - s) * (got - s); nrm += s * s;
  }
  printf("op1 rel err %.3e   W[0][0..3] = %g %g %g %g  ref %g %g\n", sqrt(err / nrm), W[0], W[1], W[2], W[3], Wref[0], Wref[1]);
  // op2 with the reference W planes from op1 output
  e = tc_op2(v, l, dW, ldw, false, 0, 0, dY, G, 0); printf("op2 launch %s\n", cudaGetErrorString(e));
  e = cudaDeviceSynchronize(); printf("op2 sync %s\n", cudaGetErrorString(e));
  std::vector<float> Yp((size_t)G * N * nit * 128);
  cudaMemcpy(Yp.data(), dY, Yp.size() * 4, cudaMemcpyDeviceToHost);
  err = 0; nrm = 0;
  for (int c = 0; c < l; ++c) for (int i = 0; i < n; ++i) {
    double s = 0; for (int j = 0; j < m; ++j) s += (double)M[(size_t)j * n + i] * ((double)W[(size_t)c * ldw + j] + W[(size_t)(N + c) * ldw + j]);
    double got = 0; for (int gg = 0; gg < G; ++gg) got += Yp[((size_t)gg * N + c) * nit * 128 + i];
    err += (got - s) * (got - s); nrm += s * s;
    if (c == 0 && i < 3) printf("  Y[%d][0] got %g ref %g\n", i, got, s);
  }
  printf("op2 rel err %.3e\n", sqrt(err / nrm));
  // sketch
  e = tc_op2(v, l, nullptr, 0, true, 1234, 1, dY, G, 0); cudaDeviceSynchronize(); printf("sketch %s\n", cudaGetErrorString(e));
  return 0;
}
