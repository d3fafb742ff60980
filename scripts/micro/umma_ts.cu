// tcgen05.mma kind::tf32 with the A operand in TMEM ("ts"): layout check against a host
// reference, and throughput vs the SMEM-operand ("ss") form (not product code).
// A (128 x 8): row m in TMEM lane m, k in column a_col + k (written by tcgen05.st.32x32b.x8).
// B (N x 8, K-major): SMEM SWIZZLE_128B rows of 128 B (k < 8 uses the first 32 B of each row).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <cstdio>
#include <vector>

#include "../../paper_2506_04840_b200/csrc/rtk_sm100.cuh"
using namespace rtk::sm100;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ volatile int g_stop[148];
template <int N>
__global__ void __launch_bounds__(128, 1) ts_kernel(const float* A, const float* B, float* D, int iters, int ts,
                                                    unsigned long long* cyc, int hammer = 0) {
  extern __shared__ __align__(1024) char smraw[];
  char* sm = (char*)(((uintptr_t)smraw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tb;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, t = threadIdx.x;
  // B: N rows (n) x 8 k, K-major SW128 (row n at n*128, 16-B chunk (k/4) ^ (n & 7))
  for (int idx = t; idx < N * 8; idx += 128) {
    const int n = idx / 8, k = idx % 8;
    *(float*)(sm + sw128_offset(n, k)) = B[n * 8 + k];
  }
  // A in SMEM too (for the ss comparison): 128 rows x 8 k, K-major SW128 at +32 KB
  for (int idx = t; idx < 128 * 8; idx += 128) {
    const int m = idx / 8, k = idx % 8;
    *(float*)(sm + 32768 + sw128_offset(m, k)) = A[m * 8 + k];
  }
  if (t == 0) { bar_init(&done, 1); bar_fence_init(); }
  if (warp == 0) tmem_alloc<512>(&tb);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t acol = 256;   // A at TMEM column 256
  {
    float v[8];
    for (int k = 0; k < 8; ++k) v[k] = A[t * 8 + k];
    tmem_st8(tb + ((uint32_t)(32 * warp) << 16) + acol, v);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t IDESC = idesc_tf32(128, N, 0, 0);
  long long t0 = 0, t1 = 0;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp > 0 && hammer) {
    float v[32];
    for (int k = 0; k < 32; ++k) v[k] = (float)k;
    float acc = 0.f;
    long long n = 0;
    while (!stop) {
      if (hammer == 1) {   // TMEM stores into columns 384..447 of this warp's lane quadrant
        asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                     "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tb + ((uint32_t)(32 * warp) << 16) + 384),
                     "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
                     "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
                     "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
                     "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      } else {             // shared-memory loads (LDS.128) from a 16 KB region
        const float4* src = (const float4*)(sm + 49152);
#pragma unroll
        for (int r = 0; r < 8; ++r) { float4 x = src[(lane + 32 * r + (int)n) & 1023]; acc += x.x + x.w; }
      }
      ++n;
    }
    if (lane == 0 && acc == 12345.f) cyc[0] = 1;
  }
  if (warp == 0) {
    const uint64_t bd = sdesc_sw128(smem_addr(sm), 16, 1024);
    const uint64_t ad = sdesc_sw128(smem_addr(sm + 32768), 16, 1024);
    umma_ts(tb, tb + acol, bd, IDESC, 0);   // D = A B^T once (checked below)
    t0 = clock64();
    if (ts == 2) {
      // the fused kernel's stage: A hi/lo at TMEM cols 384 + 8 k8 (+32), B hi/lo planes at +0/+8 KB
      const uint64_t bd_lo = sdesc_sw128(smem_addr(sm + 8192), 16, 1024);
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k8 = 0; k8 < 4; ++k8) {
          const uint32_t ahi = tb + 384 + 8 * k8, alo = ahi + 32;
          umma_ts(tb + 128, alo, bd + 2 * k8, IDESC, 1);
          umma_ts(tb + 128, ahi, bd_lo + 2 * k8, IDESC, 1);
          umma_ts(tb + 128, ahi, bd + 2 * k8, IDESC, 1);
        }
      }
    } else if (ts) {
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 12; ++k) umma_ts(tb + 128, tb + acol, bd, IDESC, 1);
      }
    } else {
      for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 12; ++k) umma_tf32_e(tb + 128, ad, bd, IDESC, 1);
      }
    }
    umma_commit_e(&done);
    bar_wait(&done, 0);
    t1 = clock64();
    if (lane == 0 && cyc) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
    if (lane == 0) stop = 1;
  }
  __syncthreads();
  tc_fence_after();
  // D row m = lane (32 w + lane), columns n
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tb + ((uint32_t)(32 * warp) << 16) + c0, v);
    if (blockIdx.x == 0)
      for (int c = 0; c < 16; ++c) D[t * N + c0 + c] = v[c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

static float tf32t(float x) {
  unsigned u;
  memcpy(&u, &x, 4);
  u &= 0xFFFFE000u;
  float y;
  memcpy(&y, &u, 4);
  return y;
}

template <int N>
void run() {
  std::vector<float> A(128 * 8), B(N * 8), D(128 * N);
  for (int i = 0; i < 128 * 8; ++i) A[i] = (float)((i * 37) % 101) / 17.0f - 2.0f;
  for (int i = 0; i < N * 8; ++i) B[i] = (float)((i * 53) % 89) / 13.0f - 3.0f;
  float *dA, *dB, *dD;
  unsigned long long* dc;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 148 * 8);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  const int smem = 65536 + 1024;
  cudaFuncSetAttribute(ts_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ts_kernel<N><<<1, 128, smem>>>(dA, dB, dD, 1, 1, dc);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double err = 0, nrm = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < 8; ++k) s += (double)tf32t(A[m * 8 + k]) * tf32t(B[n * 8 + k]);
      err = fmax(err, fabs(s - D[m * N + n]));
      nrm = fmax(nrm, fabs(s));
    }
  unsigned long long c[148];
  const int iters = 2000;
  for (int hm = 0; hm <= 2; ++hm)
  for (int ts = 0; ts <= 2; ++ts) {
    ts_kernel<N><<<148, 128, smem>>>(dA, dB, dD, iters, ts, dc, hm);
    cudaDeviceSynchronize();
    cudaMemcpy(c, dc, 148 * 8, cudaMemcpyDeviceToHost);
    printf("N=%3d %s hammer=%s: %.2f cyc/mma   layout max err %.3e (|D| %.2f) [%s]\n", N, ts == 2 ? "stage pattern (TMEM A)" : ts ? "A in TMEM" : "A in SMEM",
           hm == 0 ? "none" : hm == 1 ? "tmem-st" : "lds", (double)c[1 % 148] / (iters * 12), err, nrm, cudaGetErrorString(cudaGetLastError()));
  }
}

int main() {
  run<64>();
  return 0;
}
