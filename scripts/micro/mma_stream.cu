// Microbenchmark (not product code): the fused power step's MMA stream in isolation.
// A (hi | lo planes) in TMEM, B (hi | lo planes) in SMEM, 3 tf32 MMAs per K-step of 8
// (A_lo B_hi, A_hi B_lo [collector fill], A_hi B_hi [lastuse]), 4 K-steps per stage, one commit
// per stage; no producers, no TMA -- operands are whatever TMEM / SMEM hold.  Reports cycles per
// MMA for cta_group::1 (M = 128) and cta_group::2 (M = 256 over a CTA pair).
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o mma_stream mma_stream.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n@px mov.s32 %0, 1;\n}\n"
      : "+r"(pred));
  return pred;
}

template <int CG, uint32_t IDESC>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t bhi, uint64_t blo, uint32_t acc,
                                     int variant) {
  if (variant == 0) {
    if (CG == 1)
      asm volatile(
          "{\n.reg .pred p, e;\nsetp.ne.b32 p, %5, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, p;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
          "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
    else
      asm volatile(
          "{\n.reg .pred p, e;\nsetp.ne.b32 p, %5, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%2], %3, %6, p;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
          "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
  } else if (variant == 1) {
    if (CG == 1)
      asm volatile(
          "{\n.reg .pred p, e;\nsetp.ne.b32 p, %5, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, p;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %6, 1;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
          "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
    else
      asm volatile(
          "{\n.reg .pred p, e;\nsetp.ne.b32 p, %5, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%2], %3, %6, p;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %4, %6, 1;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
          "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
  } else if (variant == 3) {   // CUTLASS style: C++-level elect branch, plain asm
    if (elect_one()) {
      if (CG == 1)
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, p;\n"
            "tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
            "tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
            "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
      else
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%2], %3, %6, p;\n"
            "tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
            "tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
            "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
    }
    __syncwarp();
  } else if (variant == 4 || variant == 5 || variant == 6) {
    // 4: v0 with acc = 1; 5: three single-MMA blocks (umma_ts style); 6: v5 with acc = 1
    const uint32_t ac = (variant == 5) ? acc : 1u;
    if (variant == 4) {
      mma3<CG, IDESC>(d, ahi, alo, bhi, blo, 1u, 0);
    } else if (CG == 1) {
      asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %3, 0;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %4, p;\n}\n" ::"r"(d), "r"(alo), "l"(bhi),
                   "r"(ac), "n"(IDESC));
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(d), "r"(ahi), "l"(blo),
                   "n"(IDESC));
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(d), "r"(ahi), "l"(bhi),
                   "n"(IDESC));
    } else {
      asm volatile("{\n.reg .pred p, e;\nsetp.ne.b32 p, %3, 0;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %4, p;\n}\n" ::"r"(d), "r"(alo), "l"(bhi),
                   "r"(ac), "n"(IDESC));
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(d), "r"(ahi), "l"(blo),
                   "n"(IDESC));
      asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                   "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(d), "r"(ahi), "l"(bhi),
                   "n"(IDESC));
    }
  } else {   // one product per K-step (baseline rate)
    if (CG == 1)
      asm volatile(
          "{\n.reg .pred p, e;\nsetp.ne.b32 p, %5, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %6, p;\n}\n" ::"r"(d),
          "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
    else
      asm volatile(
          "{\n.reg .pred p, e;\nsetp.ne.b32 p, %5, 0;\nelect.sync _|e, 0xffffffff;\n"
          "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %3, %6, p;\n}\n" ::"r"(d),
          "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
  }
}

template <int CG>
__device__ __forceinline__ void commit(uint64_t* b) {
  if (CG == 1)
    asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
                     smem_addr(b))
                 : "memory");
  else
    asm volatile(
        "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
            smem_addr(b)),
        "h"((uint16_t)3)
        : "memory");
}

// stages: number of 32-K stages; ntile: D tiles cycled per stage (1 = op1-like, 4 = op2-like);
// commits: 1 = commit an mbarrier per stage (and wait on it 2 stages later, like the ring)
template <int CG, int N, bool TB0>
__global__ void __launch_bounds__(128, 1) stream_kernel(int stages, int ntile, int commits, int variant,
                                                        unsigned long long* out) {
  constexpr uint32_t IDESC = idesc_tf32(128 * CG, N, 0, 0);
  constexpr int NB = CG == 1 ? N : N / 2;   // B rows in this CTA
  extern __shared__ __align__(1024) char smraw[];
  char* sm = (char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bars[4];
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5;
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 4 * NB * 128 / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i % 97);
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) bar_init(&bars[i], 1);
    bar_fence_init();
  }
  if (warp == 0) {
    if (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tb)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tb)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  tc_fence_after();
  // TB0: a full 512-column allocation always starts at TMEM address 0; using the literal keeps
  // every operand address warp-uniform (uniform registers, no R2UR per MMA)
  const uint32_t tbase = TB0 ? 0u : tb;
  if (warp == 1 && rank == 0) {
    const uint64_t b0 = sdesc_sw128(smem_addr(sm), 16, 1024);
    const long long t0 = clock64();
    uint32_t dcur = tbase, ta = tbase + 256;
    const uint32_t dend = tbase + (uint32_t)(ntile * N);
    for (int s = 0; s < stages; ++s) {
      const int sa = s & 1;
      if (commits && s >= 2) bar_wait(&bars[sa], (uint32_t)(((s - 2) >> 1) & 1));
      const uint32_t d = dcur;
      dcur += N;
      if (dcur == dend) dcur = tbase;
      ta ^= 64u;
#pragma unroll
      for (int k8 = 0; k8 < 4; ++k8) {
        const uint64_t bhi = b0 + (uint64_t)((k8 * 32) >> 4), blo = b0 + (uint64_t)((NB * 128 + k8 * 32) >> 4);
        mma3<CG, IDESC>(d, ta + 8 * k8, ta + 32 + 8 * k8, bhi, blo, (s | k8) != 0, variant);
      }
      if (commits) commit<CG>(&bars[sa]);
    }
    commit<CG>(&bars[2]);
    bar_wait(&bars[2], 0);
    const long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  if (CG == 2 && rank == 1 && warp == 1) {   // the peer's bars[2] also receives the multicast
    bar_wait(&bars[2], 0);
  }
  tc_fence_before();
  __syncthreads();
  if (CG == 2) asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
    else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
  }
}

template <int CG, int N, bool TB0 = false>
void run(int grid, int stages, int ntile, int commits, int variant) {
  unsigned long long* d;
  cudaMalloc(&d, sizeof(unsigned long long) * grid);
  const size_t smem = 1024 + 4 * (CG == 1 ? N : N / 2) * 128;
  cudaFuncSetAttribute(stream_kernel<CG, N, TB0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, stream_kernel<CG, N, TB0>, stages, ntile, commits, variant, d);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, stream_kernel<CG, N, TB0>, stages, ntile, commits, variant, d);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const int per_k = variant == 2 ? 1 : 3;   // variant 3: 3 products
  const double mmas = (double)stages * 4 * per_k;
  printf("tb0=%d cg%d N=%d grid=%d stages=%d ntile=%d commits=%d variant=%d: %.1f cyc/MMA (%.1f cyc/stage)  %.3f ms  %s\n",
         (int)TB0, CG, N, grid, stages, ntile, commits, variant, h / mmas, (double)h / stages, ms, cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  for (int v = 4; v <= 6; ++v)
    for (int c = 0; c < 2; ++c) {
      run<1, 64, true>(1, 4000, 4, c, v);
      run<2, 64, true>(2, 4000, 4, c, v);
      run<1, 64, false>(1, 4000, 1, c, v);
    }
  return 0;
  for (int v = 0; v < 3; ++v)
    for (int c = 0; c < 2; ++c) {
      run<1, 64, true>(1, 4000, 4, c, v);
      run<2, 64, true>(2, 4000, 4, c, v);
    }
  run<2, 64, true>(148, 4000, 4, 1, 0);
  for (int v = 0; v < 3; ++v)
    for (int nt = 1; nt <= 4; nt += 3)
      for (int c = 0; c < 2; ++c) {
        run<1, 64>(1, 4000, nt, c, v);
        run<2, 64>(2, 4000, nt, c, v);
      }
  run<1, 64>(148, 4000, 4, 1, 0);
  run<2, 64>(148, 4000, 4, 1, 0);
  run<1, 32>(1, 4000, 4, 1, 0);
  run<2, 32>(2, 4000, 4, 1, 0);
  return 0;
}
