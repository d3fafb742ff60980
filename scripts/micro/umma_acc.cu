// tcgen05.mma kind::tf32 issue throughput vs the number of independent accumulators the MMAs
// rotate over (not product code).  One warp per CTA issues 48 MMAs per iteration (fully unrolled),
// D = tb + (k % NACC) * N, A from SMEM ("ss") or TMEM ("ts"), B from SMEM; all 148 SMs busy.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o umma_acc umma_acc.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}

template <int N, int NACC, int TS>
__global__ void __launch_bounds__(128, 1) acc_kernel(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) char smraw[];
  char* sm = (char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  if (threadIdx.x == 0) { bar_init(&done, 1); bar_fence_init(); }
  if (warp == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t IDESC = idesc_tf32(128, N, 0, 0);
  if (warp == 0) {
    const uint64_t ad = sdesc_sw128(smem_addr(sm), 16, 1024), bd = sdesc_sw128(smem_addr(sm + 32768), 16, 1024);
    const uint32_t ta = tb + 448;   // A operand columns (ts)
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 48; ++k) {
        const uint32_t d = tb + (uint32_t)((k % NACC) * N);
        if (TS) umma_ts(d, ta + 8 * (k & 3), bd + 2 * (k & 3), IDESC, 1);
        else umma_tf32_e(d, ad + 2 * (k & 3), bd + 2 * (k & 3), IDESC, 1);
      }
    }
    umma_commit_e(&done);
    bar_wait(&done, 0);
    const long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[0] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

template <int N, int NACC, int TS>
void run(unsigned long long* dc) {
  auto k = acc_kernel<N, NACC, TS>;
  const int smem = 65536 + 1024, iters = 1000;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<148, 128, smem>>>(10, dc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, smem>>>(iters, dc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c;
  cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
  printf("N=%3d nacc=%d %s: %.2f cyc/mma  chip %.0f TFLOP/s tf32  [%s]\n", N, NACC, TS ? "ts" : "ss",
         (double)c / (iters * 48.0), 2.0 * 128 * N * 8 * 48.0 * iters * 148 / ms / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* dc;
  cudaMalloc(&dc, 64);
  run<64, 1, 0>(dc); run<64, 2, 0>(dc); run<64, 4, 0>(dc);
  run<64, 1, 1>(dc); run<64, 2, 1>(dc); run<64, 4, 1>(dc);
  run<128, 1, 0>(dc); run<128, 2, 0>(dc); run<128, 1, 1>(dc); run<128, 2, 1>(dc);
  run<256, 1, 1>(dc);
  run<32, 1, 1>(dc); run<32, 4, 1>(dc);
  return 0;
}
