// Latency (cycles) of the Householder reflector's scalar chain (rsqrt_fast, rcp_fast as in
// rtk_solve.cu) on 1 warp vs 8 warps of one CTA, and of a fp64 SHFL.BFLY + DADD level.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-0.5 * x * y, y, 1.5);
  y = y * fma(-0.5 * x * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}
__global__ void k(double* out, long long* cyc, double a, int n) {
  double x = a + threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt_fast(x + 1.0);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = rcp_fast(x + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = x + __shfl_xor_sync(0xffffffffu, x, 1);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, 1e-3);
  long long t4 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 64);
  const int n = 1000;
  for (int th : {32, 256}) {
    k<<<1, th>>>(o, c, 0.5, n); k<<<1, th>>>(o, c, 0.5, n);
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("threads %d: rsqrt_fast %.1f  rcp_fast %.1f  shfl+dadd %.1f  dfma %.1f cycles\n", th, (double)h[0] / n,
           (double)h[1] / n, (double)h[2] / n, (double)h[3] / n);
  }
  return 0;
}
