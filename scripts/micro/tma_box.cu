// TMA 2-D box streaming throughput over a column-major n x m fp32 matrix (n = 1000 rows, like a
// C5 unfolding): each CTA streams its own column blocks; box shapes of the fused kernel vs others.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tma_box tma_box.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

template <int ST>
__global__ void __launch_bounds__(64) box_kernel(const __grid_constant__ CUtensorMap tm, int n, int m, int bx, int by,
                                                 int bytes, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    bar_fence_init();
  }
  __syncthreads();
  // tiles: (row tile r, col tile c) for this CTA's column range
  const int nrt = (n + bx - 1) / bx, nct = m / by;
  const int c0 = (int)((long long)blockIdx.x * nct / gridDim.x), c1 = (int)((long long)(blockIdx.x + 1) * nct / gridDim.x);
  const long long total = (long long)(c1 - c0) * nrt;
  if (warp == 0 && lane == 0) {
    for (long long it = 0; it < total; ++it) {
      const int s = (int)(it % ST);
      bar_wait(&empty[s], (uint32_t)(((it / ST) & 1) ^ 1));
      bar_expect_tx(&full[s], bytes);
      const int ct = c0 + (int)(it / nrt), rt = (int)(it % nrt);
      tma_load_2d(sm + s * bytes, &tm, rt * bx, ct * by, &full[s]);
    }
  } else if (warp == 1) {
    unsigned long long acc = 0;
    for (long long it = 0; it < total; ++it) {
      const int s = (int)(it % ST);
      bar_wait(&full[s], (uint32_t)((it / ST) & 1));
      acc += *(const unsigned*)(sm + s * bytes + lane * 4);
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);
    }
    if (acc == 0x12345ull) sink[0] = acc;
  }
}

typedef CUresult (*PFN_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 1000, m = 1000000;
  float* A;
  cudaMalloc(&A, (size_t)n * m * 4);
  cudaMemset(A, 0, (size_t)n * m * 4);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
  PFN_t enc = (PFN_t)p;
  struct Cfg { int bx, by; CUtensorMapSwizzle sw; const char* name; };
  Cfg cfgs[] = {{32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "{32 rows,128 cols} SW128 (fused op1 A)"},
                {128, 32, CU_TENSOR_MAP_SWIZZLE_NONE, "{128 rows,32 cols} none (fused op2 A)"},
                {32, 64, CU_TENSOR_MAP_SWIZZLE_128B, "{32 rows,64 cols} SW128"},
                {256, 16, CU_TENSOR_MAP_SWIZZLE_NONE, "{256 rows,16 cols} none"},
                {128, 64, CU_TENSOR_MAP_SWIZZLE_NONE, "{128 rows,64 cols} none (32 KB)"}};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (const Cfg& c : cfgs) {
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
    cuuint64_t str[1] = {(cuuint64_t)n * 4};
    cuuint32_t box[2] = {(cuuint32_t)c.bx, (cuuint32_t)c.by};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, A, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int bytes = c.bx * c.by * 4;
    for (int st : {4, 8}) {
      const int smem = st * bytes + 1024;
      if (smem > 227 * 1024) continue;
      auto kern = st == 4 ? box_kernel<4> : box_kernel<8>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<148, 64, smem>>>(tm, n, m, c.bx, c.by, bytes, sink);
      cudaEventRecord(e0);
      kern<<<148, 64, smem>>>(tm, n, m, c.bx, c.by, bytes, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double moved = (double)((n + c.bx - 1) / c.bx) * c.bx * (double)(m / c.by) * c.by * 4;
      printf("%-42s stages %d: %.3f ms  %.0f GB/s  [%d %s]\n", c.name, st, ms, moved / ms / 1e6, (int)r,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
