// Microbenchmark (not product code): the fused power step's MMA stream with the uniform-register
// issue recipe (C++ elect branch, TMEM base literal 0): 4 K-steps x 3 tf32 products per stage,
// A (hi|lo) in TMEM from a 2-stage ring, B (hi|lo) planes in SMEM, optional commit per stage.
// Reports cycles per MMA; no producers / TMA, so it is the tensor pipe's own rate for the pattern.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o mma_clean mma_clean.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n@px mov.s32 %0, 1;\n}\n" : "+r"(pred));
  return pred;
}
template <uint32_t IDESC, bool COLL>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t bhi, uint64_t blo, uint32_t acc) {
  if (COLL)
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, p;\n"
        "tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
        "tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
        "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
  else
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, p;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %6, 1;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
        "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
}

template <int N, bool COLL, int MODE>   // MODE 0: no commits; 1: commit a ring barrier per stage + wait 2 back
__global__ void __launch_bounds__(128, 1) k(int stages, unsigned long long* out) {
  constexpr uint32_t IDESC = idesc_tf32(128, N, 0, 0);
  extern __shared__ __align__(1024) char smraw[];
  __shared__ __align__(8) uint64_t bars[3];
  __shared__ uint32_t tb;
  char* sm = smraw + ((1024u - (smem_addr(smraw) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < 4 * 2 * N * 128 / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i % 97);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) bar_init(&bars[i], 1);
    bar_fence_init();
  }
  if (threadIdx.x < 32) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x < 32) {
    const uint64_t b0 = sdesc_sw128(smem_addr(sm), 16, 1024);
    const long long t0 = clock64();
    uint32_t ph[2] = {0, 0};
    for (int s = 0; s < stages; ++s) {
      const int sa = s & 1;
      if (MODE == 1 && s >= 2) { bar_wait(&bars[sa], ph[sa]); ph[sa] ^= 1; }
      if (elect_one()) {
        const uint32_t d = (uint32_t)((s & 3) * N);
        const uint32_t ta = 320u + 64u * (uint32_t)sa;
        const uint64_t bs = b0 + (uint64_t)(((s & 3) * 2 * N * 128) >> 4);
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8)
          mma3<IDESC, COLL>(d, ta + 8 * k8, ta + 32 + 8 * k8, bs + (uint64_t)((k8 * 32) >> 4),
                            bs + (uint64_t)((N * 128 + k8 * 32) >> 4), (s | k8) != 0);
        if (MODE == 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&bars[sa]))
                       : "memory");
      }
      __syncwarp();
    }
    if (elect_one())
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(&bars[2]))
                   : "memory");
    __syncwarp();
    bar_wait(&bars[2], 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc<512>(0u);
}

template <int N, bool COLL, int MODE>
void run(int grid) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * grid);
  const int smem = 1024 + 4 * 2 * N * 128;
  cudaFuncSetAttribute(k<N, COLL, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 8000;
  k<N, COLL, MODE><<<grid, 128, smem>>>(stages, d);
  k<N, COLL, MODE><<<grid, 128, smem>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("N=%d collector=%d mode=%d grid=%d: %.1f cyc/MMA  %s\n", N, (int)COLL, MODE, grid, h / (stages * 12.0),
         cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<64, true, 0>(1);
  run<64, false, 0>(1);
  run<64, true, 1>(1);
  run<64, false, 1>(1);
  run<32, true, 1>(1);
  run<128, true, 1>(1);
  run<64, true, 1>(148);
  run<64, false, 1>(148);
  return 0;
}
