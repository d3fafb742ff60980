// Microbenchmarks that decide the fused power-step design (not product code):
//  (1) bulk-copy (TMA 1-D) streaming rate: HBM stream, and HBM stream + immediate L2 re-read
//      of the same chunk window (the "second pass through L2" of a fused op1/op2 kernel);
//  (2) tcgen05.mma kind::tf32 SS throughput (cycles per instruction) for M=128 and several N,
//      alone and with 4 warps hammering shared memory (the A_lo split traffic).
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o l2_umma l2_umma.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

// Each CTA owns a contiguous region of `per_cta` bytes, processed in windows of `win` bytes;
// every window is read `passes` times (pass 0 from HBM, later passes hit L2) in 16 KB chunks.
constexpr int CH = 16384, ST = 8;
__global__ void __launch_bounds__(64) stream_kernel(const char* base, size_t per_cta, size_t win, int passes,
                                                    unsigned long long* sink) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t full[ST], empty[ST];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    bar_fence_init();
  }
  __syncthreads();
  const char* my = base + (size_t)blockIdx.x * per_cta;
  const size_t nwin = per_cta / win, nch = win / CH;
  const size_t total = nwin * passes * nch;
  if (warp == 0 && lane == 0) {
    size_t it = 0;
    for (size_t w = 0; w < nwin; ++w)
      for (int p = 0; p < passes; ++p)
        for (size_t c = 0; c < nch; ++c, ++it) {
          const int s = (int)(it % ST);
          bar_wait(&empty[s], (uint32_t)(((it / ST) & 1) ^ 1));
          bar_expect_tx(&full[s], CH);
          bulk_g2s(sm + s * CH, my + w * win + c * CH, CH, &full[s]);
        }
  } else if (warp == 1) {
    unsigned long long acc = 0;
    for (size_t it = 0; it < total; ++it) {
      const int s = (int)(it % ST);
      bar_wait(&full[s], (uint32_t)((it / ST) & 1));
      acc += *(const unsigned*)(sm + s * CH + lane * 4);
      __syncwarp();
      if (lane == 0) bar_arrive(&empty[s]);
    }
    if (acc == 0x123456789ull) sink[0] = acc;
  }
}

__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void umma_tf32_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p, e;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// UMMA throughput: one thread issues `iters` x (nmma) tf32 MMAs M=128 xN, K=8 on fixed smem tiles.
template <int N>
__global__ void __launch_bounds__(192, 1) umma_kernel(int iters, int nmma, int hammer, unsigned long long* out,
                                                      int nacc, int astride) {
  extern __shared__ __align__(1024) char smraw[];
  char* sm = (char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tb;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((float*)sm)[i] = 1.0f;
  if (threadIdx.x == 0) { bar_init(&done, 1); bar_fence_init(); stop = 0; }
  if (warp == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t IDESC = idesc_tf32(128, N, 0, 0);
  if (warp == 1) {
    const uint32_t a = smem_addr(sm), b = smem_addr(sm + 32768);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (nacc == 1) {
        const uint64_t ad0 = sdesc_sw128(a, 16, 1024), bd0 = sdesc_sw128(b, 16, 1024);
#pragma unroll
        for (int k = 0; k < 12; ++k) umma_tf32_elect(tb, ad0 + (k & 3) * 2, bd0 + (k & 3) * 2, IDESC, 1);
      } else {
#pragma unroll 1
      for (int k = 0; k < nmma; ++k) {
        const uint64_t ad = sdesc_sw128(a + (k & 3) * 32 + ((k >> 2) & 1) * astride, 16, 1024);
        const uint64_t bd = sdesc_sw128(b + (k & 3) * 32, 16, 1024);
        umma_tf32_elect(tb + (uint32_t)((k % nacc) * N), ad, bd, IDESC, 1);
      }
      }
    }
    if (elect_one()) umma_commit(&done);
    __syncwarp();
    bar_wait(&done, 0);
    long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) { out[blockIdx.x] = (unsigned long long)(t1 - t0); stop = 1; }
  } else if (warp >= 2 && hammer) {
    // lo-split-like traffic on a disjoint 16 KB region: read float4, write float4
    float4* src = (float4*)(sm + 49152);
    float4* dst = (float4*)(sm + 49152 + 8192);
    const int t = threadIdx.x - 64;
    unsigned long long n = 0;
    while (!stop) {
#pragma unroll 4
      for (int r = 0; r < 4; ++r) {
        float4 v = src[(t + 128 * r) & 511];
        v.x += 1.f;
        dst[(t + 128 * r) & 511] = v;
      }
      ++n;
    }
    if (t == 0) out[gridDim.x + blockIdx.x] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

int main() {
  int dev = 0;
  cudaSetDevice(dev);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int G = 148;
  const size_t per = 24ull << 20;   // 24 MB per CTA -> 3.5 GB total
  char* buf;
  cudaMalloc(&buf, per * G);
  cudaMemset(buf, 1, per * G);
  unsigned long long* sink;
  cudaMalloc(&sink, 4096 * 8);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CH * ST);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const size_t wins[] = {65536, 262144, 524288, 1048576};
  for (int passes = 1; passes <= 0; ++passes) {
    for (size_t win : wins) {
      if (passes == 1 && win != 65536) continue;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        stream_kernel<<<G, 64, CH * ST>>>(buf, per, win, passes, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep)
          printf("stream passes=%d win=%zuKB: %.3f ms, HBM-bytes rate %.0f GB/s, smem-fill rate %.0f GB/s\n", passes,
                 win >> 10, ms, per * G / ms / 1e6, per * G * passes / ms / 1e6);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  unsigned long long* dout;
  cudaMalloc(&dout, 2 * G * 8);
  unsigned long long h[2 * 148];
  auto run = [&](auto kern, int N, int nmma, int hammer, int nacc = 1, int astride = 0) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 + 1024);
    const int iters = 2000;
    kern<<<G, 192, 65536 + 1024>>>(iters, nmma, hammer, dout, nacc, astride);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<G, 192, 65536 + 1024>>>(iters, nmma, hammer, dout, nacc, astride);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, dout, 2 * G * 8, cudaMemcpyDeviceToHost);
    printf("umma N=%d nacc=%d hammer=%d: %.2f cyc/mma (CTA0 clock64), %.3f ms, chip %.1f TFLOP/s tf32, hammer iters %llu  [%s]\n",
           N, nacc, hammer, (double)h[0] / (iters * nmma), ms, 2.0 * 128 * 8 * N * iters * nmma * G / ms / 1e9,
           hammer ? h[G] : 0ull, cudaGetErrorString(cudaGetLastError()));
  };
  for (int nacc : {1}) {
    run(umma_kernel<16>, 16, 12, 0, nacc);
    run(umma_kernel<32>, 32, 12, 0, nacc);
    run(umma_kernel<64>, 64, 12, 0, nacc);
    run(umma_kernel<128>, 128, 12, 0, nacc);
  }
  run(umma_kernel<256>, 256, 12, 0, 1);
  run(umma_kernel<256>, 256, 12, 0, 2);
  run(umma_kernel<64>, 64, 12, 1, 4);
  run(umma_kernel<64>, 64, 12, 0, 4, 16384);
  run(umma_kernel<64>, 64, 12, 0, 1, 16384);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}
