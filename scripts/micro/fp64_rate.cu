// Microbenchmark: FP64 DFMA and FP32 FFMA throughput per SM (B200 sanity check).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
    x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <typename T>
void run(const char* name) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * 4, threads = 256, iters = 1 << 14;
  T* out; cudaMalloc(&out, sizeof(T) * blocks * threads);
  fma_loop<T><<<blocks, threads>>>(out, 16, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fmas = (double)blocks * threads * iters * 8;
  printf("%s: %.2f TFLOP/s  (%.1f FMA/clk/SM at 1.965 GHz)\n", name, 2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(out);
}
int main() { run<float>("fp32 FFMA"); run<double>("fp64 DFMA"); return 0; }
