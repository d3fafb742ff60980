// Dependent-chain latency of fp64 ops on one thread (cycles per op).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int n) {
  double x = a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  double y = a;
  for (int i = 0; i < n; ++i) y = b / y;
  long long t2 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = sqrt(z + b);
  long long t3 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = fmaf(f, (float)a, (float)b);
  long long t4 = clock64();
  double w = a;
  for (int i = 0; i < n; ++i) w = (double)(float)(w * b);
  long long t5 = clock64();
  out[0] = x + y + z + f + w;
  cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 40);
  int n = 4096;
  lat<<<1, 1>>>(o, c, 0.999, 1.0001, n);
  lat<<<1, 1>>>(o, c, 0.999, 1.0001, n);
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  printf("cycles/op: DFMA %.1f  DDIV %.1f  DSQRT %.1f  FFMA %.1f  D->F->D+DMUL %.1f\n", (double)h[0] / n,
         (double)h[1] / n, (double)h[2] / n, (double)h[3] / n, (double)h[4] / n);
  return 0;
}
