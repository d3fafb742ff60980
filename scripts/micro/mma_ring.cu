// Microbenchmark (not product code): the fused power step's TMEM A-ring handshake in isolation.
// Producer warps (2 groups x 4 lane quadrants) write each stage's A hi/lo planes to TMEM
// (tcgen05.st 32x32b.x32 twice, wait::st) and arrive on a_full[ts]; the MMA warp waits a_full,
// issues 12 tf32 MMAs (uniform-register issue) and commits a_empty[ts].  SA TMEM stages.
// Optional: producers load the stage from a fixed 16 KB shared-memory tile first (LDS),
// which is the real kernel's shared-memory -> register -> TMEM path.
// nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o mma_ring mma_ring.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n@px mov.s32 %0, 1;\n}\n" : "+r"(pred));
  return pred;
}
template <uint32_t IDESC>
__device__ __forceinline__ void mma3(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t bhi, uint64_t blo, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %6, p;\n"
      "tcgen05.mma.cta_group::1.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
      "tcgen05.mma.cta_group::1.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
      "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
}
__device__ __forceinline__ void commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

// SA TMEM A stages at columns 320.. (64 each; 3 stages max with D at 0..255 and W at 256)
template <int SA, bool LDS, int NG>
__global__ void __launch_bounds__(32 * (2 + 4 * NG), 1) k(int stages, unsigned long long* out) {
  constexpr uint32_t IDESC = idesc_tf32(128, 64, 0, 0);
  constexpr uint32_t TA0 = 512 - 64 * SA;
  extern __shared__ __align__(1024) char smraw[];
  __shared__ __align__(8) uint64_t a_full[SA], a_empty[SA], done;
  __shared__ uint32_t tb;
  char* sm = smraw + ((1024u - (smem_addr(smraw) & 1023u)) & 1023u);
  for (int i = threadIdx.x; i < (32768 + 16384) / 4; i += blockDim.x) ((float*)sm)[i] = 0.001f * (i % 97);
  if (threadIdx.x == 0) {
    for (int i = 0; i < SA; ++i) { bar_init(&a_full[i], 4); bar_init(&a_empty[i], 1); }
    bar_init(&done, 1);
    bar_fence_init();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) {   // MMA issuer
    const uint64_t b0 = sdesc_sw128(smem_addr(sm), 16, 1024);
    const long long t0 = clock64();
    int sa = 0;
    uint32_t ph = 0;
    for (int s = 0; s < stages; ++s) {
      bar_wait(&a_full[sa], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t d = (uint32_t)((s & 3) * 64);
        const uint32_t ta = TA0 + 64u * (uint32_t)sa;
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8)
          mma3<IDESC>(d, ta + 8 * k8, ta + 32 + 8 * k8, b0 + (uint64_t)((k8 * 32) >> 4),
                      b0 + (uint64_t)((64 * 128 + k8 * 32) >> 4), (s | k8) != 0);
        commit(&a_empty[sa]);
      }
      __syncwarp();
      if (++sa == SA) { sa = 0; ph ^= 1; }
    }
    if (elect_one()) commit(&done);
    __syncwarp();
    bar_wait(&done, 0);
    const long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (warp >= 2) {   // producers: NG groups x 4 quadrants, group g takes stages g mod NG
    const int q = warp & 3, g = (warp - 2) >> 2;
    const int lt = 32 * q + lane;
    const uint32_t tq0 = ((uint32_t)(32 * q) << 16) + TA0;
    const uint32_t tile = smem_addr(sm + 32768) + (uint32_t)lt * 4u;
    int ts = g % SA;
    uint32_t ph = (g / SA) & 1;
    for (int s = g; s < stages; s += NG) {
      float v[32], lo[32];
      if (LDS) {
#pragma unroll
        for (int c = 0; c < 32; ++c) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v[c]) : "r"(tile + (uint32_t)(c * 512)));
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = (float)(c + lt + s);
      }
#pragma unroll
      for (int e = 0; e < 32; ++e) lo[e] = v[e] - tf32_trunc(v[e]);
      bar_wait(&a_empty[ts], ph ^ 1);
      tc_fence_after();
      st32(tq0 + 64u * (uint32_t)ts, v);
      st32(tq0 + 64u * (uint32_t)ts + 32, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(&a_full[ts]);
      ts += NG;
      while (ts >= SA) { ts -= SA; ph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(0u);
}

template <int SA, bool LDS, int NG>
void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  const int smem = 1024 + 32768 + 16384;
  cudaFuncSetAttribute(k<SA, LDS, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 6000;
  k<SA, LDS, NG><<<148, 32 * (2 + 4 * NG), smem>>>(stages, d);
  k<SA, LDS, NG><<<148, 32 * (2 + 4 * NG), smem>>>(stages, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("SA=%d LDS=%d groups=%d: %.1f cyc/stage (%.1f cyc/MMA)  %s\n", SA, (int)LDS, NG, h / (double)stages,
         h / (stages * 12.0), cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  run<2, false, 2>();
  run<3, false, 2>();
  run<3, false, 3>();
  run<2, true, 2>();
  run<3, true, 2>();
  run<3, true, 3>();
  run<3, true, 1>();
  return 0;
}
