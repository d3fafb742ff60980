// rtk_tc.cu -- tcgen05 tensor-core path of the streaming steps (3xTF32, fp32 accumulate in TMEM).
//
// The power step Y = M (M^T Q) (Alg. 3/4 line 7) is split in two GEMMs that
// each stream the column-major unfolding M (n x m) once:
//   op1  W = M^T Q        (m x N, K = n):  A = M^T tile 128(j) x 32(i), K-major (TMA box {32,128});
//                                           B = Q tile N(c) x 32(i), K-major;   D = 128 x N in TMEM.
//                         Epilogue writes W as tf32 hi/lo planes (the B operand of op2), or -- for
//                         the ST shrink G x_k U_k^T -- the next unfolding.
//   op2  Y += M W         (n x N, K = m, split-K over CTAs): A = M tile 128(i) x 32(j), MN-major
//                         (4 TMA boxes {32,32}); B = W (or the RTK-GAUSS-2 sketch Omega_k, generated
//                         in shared memory: Y0 = M Omega_k, line 5) tile N(c) x 32(j), K-major;
//                         D = all ceil(n/128) row tiles x N columns resident in TMEM; the per-CTA
//                         partials go to the same fixed-order fp64 reduction as the FFMA path.
// 3xTF32: x = hi + lo with hi = tf32(x); D += A_hi B_hi + A_hi B_lo + A_lo B_hi.  The streamed A
// operand's lo plane is formed in shared memory by four "split" warps (lo = a - trunc_tf32(a),
// exact in fp32); B's planes are precomputed (Q, U, W) or generated (Omega) with hi = rna(x).
// Warp roles (320 threads): 0 TMA producer, 1 UMMA issuer (+TMEM owner), 2-5 split/generate,
// 6-9 epilogue (TMEM -> registers -> global).  Persistent CTAs, one per SM.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"
#include "rtk_sm100.cuh"

namespace rtk {
using namespace sm100;

constexpr int kTcThreads = 320;
constexpr int kBK = 32;            // K elements (fp32) per stage row = 128 B
constexpr int kTileBytesA = 128 * 128;

struct TcOp1Args {
  int n, N, l;         // rows of M, padded Q columns, valid columns
  int64_t m;           // columns of M
  int nk;              // ceil(n / 32)
  int64_t ntiles;      // ceil(m / 128)
  // normal epilogue: W planes [2N][ldw]
  float* W;
  int64_t ldw;
  // shrink epilogue
  int shrink;
  float* out;
  int64_t Rprev, nnext, ldnext;
};

struct TcOp2Args {
  int n, N, l;
  int64_t m;
  int nit;             // row tiles (<= 512 / N)
  int64_t nkc;         // ceil(m / 32)
  int G;               // CTAs
  float* Ypart;        // [G][N][nit*128]
  int sketch;
  uint64_t seed;
  uint32_t mode;
  float* xmax;         // sketch: atomicMax of max|M| (the fp16 pair engine's scale, rtk_fused2.cu)
  const float* om;   // materialised Omega_k [m][l] or nullptr (RTK-GAUSS-2 in place)
};

// ------------------------------------------------------------------ op1: W = M^T Q
template <int N>
__global__ void __launch_bounds__(kTcThreads, 1) tc_op1_kernel(const __grid_constant__ CUtensorMap tmM,
                                                               const __grid_constant__ CUtensorMap tmB,
                                                               const TcOp1Args a) {
  constexpr int S = 4;
  constexpr int BB = N * 128;                       // one B plane per stage
  constexpr int STAGE = 2 * kTileBytesA + 2 * BB;
  constexpr int TCOLS = (2 * N <= 32) ? 32 : (2 * N <= 64) ? 64 : 128;
  constexpr uint32_t IDESC = idesc_tf32(128, N, 0, 0);
  extern __shared__ __align__(1024) uint8_t smraw[];
  // 1024-B aligned base, derived by an offset from smraw so that the compiler keeps the shared
  // address space (LDS / STS instead of generic LD.E / ST.E through the smem window)
  uint8_t* sm = smraw + ((1024u - (smem_addr(smraw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[S], lofull[S], empty[S], accf[2], acce[2];
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { bar_init(&full[s], 1); bar_init(&lofull[s], 4); bar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { bar_init(&accf[b], 1); bar_init(&acce[b], 4); }
    bar_fence_init();
    tma_prefetch(&tmM);
    tma_prefetch(&tmB);
  }
  if (warp == 1) tmem_alloc<TCOLS>(&tbase_s);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int64_t it = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
        for (int kc = 0; kc < a.nk; ++kc, ++it) {
          const int s = (int)(it % S);
          const uint32_t ph = (uint32_t)((it / S) & 1);
          bar_wait(&empty[s], ph ^ 1);
          uint8_t* st = sm + s * STAGE;
          bar_expect_tx(&full[s], kTileBytesA + 2 * BB);
          tma_load_2d(st, &tmM, kc * kBK, (int)(t * 128), &full[s]);
          tma_load_2d(st + 2 * kTileBytesA, &tmB, kc * kBK, 0, &full[s]);
          tma_load_2d(st + 2 * kTileBytesA + BB, &tmB, kc * kBK, N, &full[s]);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- UMMA issuer (whole warp, uniform; one lane elected per instruction)
    {
      const uint64_t d0 = sdesc_sw128(smem_addr(sm), 16, 1024);   // stage 0, A hi; offsets added below
      int64_t it = 0;
      int lt = 0;
      for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++lt) {
        const int b = lt & 1;
        bar_wait(&acce[b], ((lt >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tbase + b * N;
        for (int kc = 0; kc < a.nk; ++kc, ++it) {
          const int s = (int)(it % S);
          const uint32_t ph = (uint32_t)((it / S) & 1);
          bar_wait(&full[s], ph);
          bar_wait(&lofull[s], ph);
          tc_fence_after();
          const uint64_t ds = d0 + (uint64_t)((s * STAGE) >> 4);
#pragma unroll
          for (int k8 = 0; k8 < 4; ++k8) {
            const uint64_t ahi = ds + (k8 * 32 >> 4);
            const uint64_t alo = ds + ((kTileBytesA + k8 * 32) >> 4);
            const uint64_t bhi = ds + ((2 * kTileBytesA + k8 * 32) >> 4);
            const uint64_t blo = ds + ((2 * kTileBytesA + BB + k8 * 32) >> 4);
            umma_tf32_e(d, alo, bhi, IDESC, (kc | k8) != 0);
            umma_tf32_e(d, ahi, blo, IDESC, 1);
            umma_tf32_e(d, ahi, bhi, IDESC, 1);
          }
          umma_commit_e(&empty[s]);
        }
        umma_commit_e(&accf[b]);
      }
    }
  } else if (warp < 6) {
    // ---------------- split warps: A_lo = A - trunc_tf32(A)
    const int tid = threadIdx.x - 64;    // 0..127
    int64_t it = 0;
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
      for (int kc = 0; kc < a.nk; ++kc, ++it) {
        const int s = (int)(it % S);
        const uint32_t ph = (uint32_t)((it / S) & 1);
        bar_wait(&full[s], ph);
        const float4* src = reinterpret_cast<const float4*>(sm + s * STAGE);
        float4* dst = reinterpret_cast<float4*>(sm + s * STAGE + kTileBytesA);
#pragma unroll
        for (int r = 0; r < kTileBytesA / 16 / 128; ++r) {
          const float4 v = src[tid + 128 * r];
          dst[tid + 128 * r] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                           v.w - tf32_trunc(v.w));
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) bar_arrive(&lofull[s]);
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> W planes / next unfolding
    const int q = warp & 3;              // TMEM lane quarter of this warp
    const int row = 32 * q + lane;
    int lt = 0;
    for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x, ++lt) {
      const int b = lt & 1;
      bar_wait(&accf[b], (lt >> 1) & 1);
      tc_fence_after();
      const int64_t j = t * 128 + row;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + b * N + c0, v);
        if (j < a.m) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const int cg = c0 + c;
            if (!a.shrink) {
              const float hi = tf32_rna(v[c]);
              a.W[(int64_t)cg * a.ldw + j] = hi;
              a.W[(int64_t)(N + cg) * a.ldw + j] = v[c] - hi;
            } else if (cg < a.l) {
              const int64_t aa = j % a.Rprev, tmp = j / a.Rprev;
              const int64_t bb = tmp % a.nnext, cc = tmp / a.nnext;
              const int64_t colo = aa + a.Rprev * (cg + (int64_t)a.l * cc);
              a.out[bb + a.ldnext * colo] = v[c];
              if (bb == a.nnext - 1)
                for (int64_t z = a.nnext; z < a.ldnext; ++z) a.out[z + a.ldnext * colo] = 0.f;
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive(&acce[b]);
    }
  }
  __syncthreads();
  if (warp == 1) tmem_dealloc<TCOLS>(tbase);
}

// ------------------------------------------------------------------ op2: Y += M W
template <int N>
__global__ void __launch_bounds__(kTcThreads, 1) tc_op2_kernel(const __grid_constant__ CUtensorMap tmM,
                                                               const __grid_constant__ CUtensorMap tmB,
                                                               const TcOp2Args a) {
  constexpr int SA = 4, SB = 2;
  constexpr int BB = N * 128;
  constexpr int STA = 2 * kTileBytesA;          // A hi + lo
  constexpr int STB = 2 * BB;                   // B hi + lo
  constexpr uint32_t IDESC = idesc_tf32(128, N, 1, 0);   // A MN-major, B K-major
  extern __shared__ __align__(1024) uint8_t smraw[];
  // 1024-B aligned base, derived by an offset from smraw so that the compiler keeps the shared
  // address space (LDS / STS instead of generic LD.E / ST.E through the smem window)
  uint8_t* sm = smraw + ((1024u - (smem_addr(smraw) & 1023u)) & 1023u);
  uint8_t* smA = sm;
  uint8_t* smB = sm + SA * STA;
  __shared__ __align__(8) uint64_t fullA[SA], loA[SA], emptyA[SA], fullB[SB], emptyB[SB], accf;
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t k0 = (int64_t)blockIdx.x * a.nkc / a.G;
  const int64_t k1 = (int64_t)(blockIdx.x + 1) * a.nkc / a.G;
  const int tcols = a.nit * N <= 32 ? 32 : a.nit * N <= 64 ? 64 : a.nit * N <= 128 ? 128 : a.nit * N <= 256 ? 256 : 512;

  if (threadIdx.x == 0) {
    for (int s = 0; s < SA; ++s) { bar_init(&fullA[s], 1); bar_init(&loA[s], 4); bar_init(&emptyA[s], 1); }
    for (int s = 0; s < SB; ++s) { bar_init(&fullB[s], a.sketch ? 4 : 1); bar_init(&emptyB[s], 1); }
    bar_init(&accf, 1);
    bar_fence_init();
    tma_prefetch(&tmM);
    if (!a.sketch) tma_prefetch(&tmB);
  }
  if (warp == 1) {
    switch (tcols) {
      case 32: tmem_alloc<32>(&tbase_s); break;
      case 64: tmem_alloc<64>(&tbase_s); break;
      case 128: tmem_alloc<128>(&tbase_s); break;
      case 256: tmem_alloc<256>(&tbase_s); break;
      default: tmem_alloc<512>(&tbase_s); break;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tbase_s;

  if (warp == 0) {
    if (lane == 0) {
      int64_t ia = 0;
      for (int64_t kc = k0; kc < k1; ++kc) {
        const int64_t ib = kc - k0;
        if (!a.sketch) {
          const int sb = (int)(ib % SB);
          bar_wait(&emptyB[sb], (uint32_t)(((ib / SB) & 1) ^ 1));
          bar_expect_tx(&fullB[sb], 2 * BB);
          tma_load_2d(smB + sb * STB, &tmB, (int)(kc * kBK), 0, &fullB[sb]);
          tma_load_2d(smB + sb * STB + BB, &tmB, (int)(kc * kBK), N, &fullB[sb]);
        }
        for (int itile = 0; itile < a.nit; ++itile, ++ia) {
          const int s = (int)(ia % SA);
          bar_wait(&emptyA[s], (uint32_t)(((ia / SA) & 1) ^ 1));
          bar_expect_tx(&fullA[s], kTileBytesA);
          uint8_t* st = smA + s * STA;
#pragma unroll
          for (int g = 0; g < 4; ++g)
            tma_load_2d(st + g * 4096, &tmM, itile * 128 + 32 * g, (int)(kc * kBK), &fullA[s]);
        }
      }
    }
  } else if (warp == 1) {
    {
      // MN-major A (SW128_BASE32B): K-step k8 = rows 8k8..8k8+7 of j at +1024*k8; MN groups of
      // 32 i at +4096 (LBO); 4-row K atoms at +512 (SBO).  Base descriptors once; offsets added.
      const uint64_t a0 = sdesc_sw128(smem_addr(smA), 4096, 512, kLayoutSW128Base32B);
      const uint64_t b0 = sdesc_sw128(smem_addr(smB), 16, 1024);
      int64_t ia = 0;
      for (int64_t kc = k0; kc < k1; ++kc) {
        const int64_t ib = kc - k0;
        const int sb = (int)(ib % SB);
        bar_wait(&fullB[sb], (uint32_t)((ib / SB) & 1));
        tc_fence_after();
        const uint64_t bs = b0 + (uint64_t)((sb * STB) >> 4);
        for (int itile = 0; itile < a.nit; ++itile, ++ia) {
          const int s = (int)(ia % SA);
          const uint32_t ph = (uint32_t)((ia / SA) & 1);
          bar_wait(&fullA[s], ph);
          bar_wait(&loA[s], ph);
          tc_fence_after();
          const uint64_t as = a0 + (uint64_t)((s * STA) >> 4);
          const uint32_t d = tbase + itile * N;
#pragma unroll
          for (int k8 = 0; k8 < 4; ++k8) {
            const uint64_t ahi = as + ((k8 * 1024) >> 4);
            const uint64_t alo = as + ((kTileBytesA + k8 * 1024) >> 4);
            const uint64_t bhi = bs + ((k8 * 32) >> 4);
            const uint64_t blo = bs + ((BB + k8 * 32) >> 4);
            umma_tf32_e(d, alo, bhi, IDESC, (kc != k0) || (k8 != 0));
            umma_tf32_e(d, ahi, blo, IDESC, 1);
            umma_tf32_e(d, ahi, bhi, IDESC, 1);
          }
          umma_commit_e(&emptyA[s]);
        }
        umma_commit_e(&emptyB[sb]);
      }
      umma_commit_e(&accf);
    }
  } else if (warp < 6) {
    const int tid = threadIdx.x - 64;    // 0..127
    int64_t ia = 0;
    float vmax = 0.f;
    for (int64_t kc = k0; kc < k1; ++kc) {
      const int64_t ib = kc - k0;
      if (a.sketch) {
        // B = Omega_k(j, c) for j in this chunk, c < N: hi/lo planes in the K-major SW128 layout
        const int sb = (int)(ib % SB);
        bar_wait(&emptyB[sb], (uint32_t)(((ib / SB) & 1) ^ 1));
        uint8_t* bt = smB + sb * STB;
        for (int it2 = tid; it2 < kBK * (N / 4); it2 += 128) {   // one Philox block per 4 columns
          const int jj = it2 % kBK, c4 = (it2 / kBK) * 4;
          const int64_t j = kc * kBK + jj;
          float z[4] = {0.f, 0.f, 0.f, 0.f};
          if (j < a.m && c4 < a.l) {
            if (a.om) {
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (c4 + u < a.l) z[u] = a.om[(uint64_t)j * a.l + c4 + u];
            } else {
              const uint4 x = omega_bits(a.seed, a.mode, (uint64_t)j, (uint32_t)(c4 >> 2));
              const float2 z01 = box_muller(x.x, x.y);
              z[0] = z01.x; z[1] = c4 + 1 < a.l ? z01.y : 0.f;
              if (c4 + 2 < a.l) {
                const float2 z23 = box_muller(x.z, x.w);
                z[2] = z23.x; z[3] = c4 + 3 < a.l ? z23.y : 0.f;
              }
            }
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float h = tf32_rna(z[u]);
            *reinterpret_cast<float*>(bt + sw128_offset(c4 + u, jj)) = h;
            *reinterpret_cast<float*>(bt + BB + sw128_offset(c4 + u, jj)) = z[u] - h;
          }
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) bar_arrive(&fullB[sb]);
      }
      for (int itile = 0; itile < a.nit; ++itile, ++ia) {
        const int s = (int)(ia % SA);
        bar_wait(&fullA[s], (uint32_t)((ia / SA) & 1));
        const float4* src = reinterpret_cast<const float4*>(smA + s * STA);
        float4* dst = reinterpret_cast<float4*>(smA + s * STA + kTileBytesA);
#pragma unroll
        for (int r = 0; r < kTileBytesA / 16 / 128; ++r) {
          const float4 v = src[tid + 128 * r];
          dst[tid + 128 * r] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y), v.z - tf32_trunc(v.z),
                                           v.w - tf32_trunc(v.w));
          if (a.xmax) vmax = fmaxf(fmaxf(vmax, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
        }
        fence_async_smem();
        __syncwarp();
        if (lane == 0) bar_arrive(&loA[s]);
      }
    }
    if (a.xmax) {   // every element of M passes through one split warp of one CTA
#pragma unroll
      for (int o = 16; o; o >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
      if (lane == 0) atomicMax(reinterpret_cast<unsigned int*>(a.xmax), __float_as_uint(vmax));
    }
  } else {
    // ---------------- epilogue: partial Y of this CTA -> Ypart[grp][c][i]
    const int q = warp & 3;
    const int rows = a.nit * 128;
    float* yp = a.Ypart + (int64_t)blockIdx.x * N * rows;
    if (k1 > k0) {
      bar_wait(&accf, 0);
      tc_fence_after();
    }
    for (int itile = 0; itile < a.nit; ++itile) {
      const int i = itile * 128 + 32 * q + lane;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        if (k1 > k0) tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + itile * N + c0, v);
        else {
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) yp[(int64_t)(c0 + c) * rows + i] = v[c];
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    switch (tcols) {
      case 32: tmem_dealloc<32>(tbase); break;
      case 64: tmem_dealloc<64>(tbase); break;
      case 128: tmem_dealloc<128>(tbase); break;
      case 256: tmem_dealloc<256>(tbase); break;
      default: tmem_dealloc<512>(tbase); break;
    }
  }
}

// ------------------------------------------------------------------ split kernel
// B planes for op1 from an fp64 (Q) or fp32 (U) column-major n x l matrix (ld = n):
// P[c][i] = hi, P[N + c][i] = lo for c < N, i < ldp (zero outside n x l).
__global__ void split_planes_kernel(const double* __restrict__ q64, const float* __restrict__ q32, int n, int l,
                                    int N, int ldp, float* __restrict__ P) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)N * ldp) return;
  const int c = (int)(idx / ldp), i = (int)(idx % ldp);
  float hi = 0.f, lo = 0.f;
  if (c < l && i < n) {
    if (q64) {
      const double v = q64[(int64_t)c * n + i];
      hi = tf32_rna((float)v);
      lo = (float)(v - (double)hi);
    } else {
      const float v = q32[(int64_t)c * n + i];
      hi = tf32_rna(v);
      lo = v - hi;
    }
  }
  P[(int64_t)c * ldp + i] = hi;
  P[(int64_t)(N + c) * ldp + i] = lo;
}

// ------------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                       const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                       CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled_t encode_fn() {
  static PFN_encodeTiled_t fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_encodeTiled_t)p;
  });
  return fn;
}

// 2-D fp32 map: dim0 (contiguous) = d0 elements, dim1 = d1 rows with pitch `pitch` elements
static bool make_map(CUtensorMap* map, const void* base, uint64_t d0, uint64_t d1, uint64_t pitch, uint32_t b0,
                     uint32_t b1, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  PFN_encodeTiled_t fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {d0, d1};
  cuuint64_t strides[1] = {pitch * 4};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int tc_npad(int l) { return l <= 16 ? 16 : l <= 32 ? 32 : l <= 48 ? 48 : l <= 64 ? 64 : 0; }

bool tc_supported(const View& v, int l) {
  if (getenv("RTK_PATH") && std::string(getenv("RTK_PATH")) == "ffma") return false;
  const int N = tc_npad(l);
  if (!N) return false;
  if (!(v.P == 1 && v.si == 1 && v.ss % 4 == 0 && ((uintptr_t)v.base % 16) == 0 && v.ss >= v.n)) return false;
  const int nit = (v.n + 127) / 128;
  if (nit * N > 512) return false;
  if (!encode_fn()) return false;
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  return major == 10;
}

static size_t op1_smem(int N) { return 4 * (2 * kTileBytesA + 2 * N * 128) + 1024; }
static size_t op2_smem(int N) { return 4 * 2 * kTileBytesA + 2 * 2 * N * 128 + 1024; }

template <int N>
static cudaError_t op1_launch(const CUtensorMap& mM, const CUtensorMap& mB, const TcOp1Args& a, int grid,
                              cudaStream_t st) {
  const size_t smem = op1_smem(N);
  cudaError_t e = cudaFuncSetAttribute(tc_op1_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tc_op1_kernel<N><<<grid, kTcThreads, smem, st>>>(mM, mB, a);
  return cudaGetLastError();
}
template <int N>
static cudaError_t op2_launch(const CUtensorMap& mM, const CUtensorMap& mB, const TcOp2Args& a, int grid,
                              cudaStream_t st) {
  const size_t smem = op2_smem(N);
  cudaError_t e = cudaFuncSetAttribute(tc_op2_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  tc_op2_kernel<N><<<grid, kTcThreads, smem, st>>>(mM, mB, a);
  return cudaGetLastError();
}

// B planes for op1 (from fp64 Q or fp32 U), ld = round4(n)
cudaError_t tc_split(const double* q64, const float* q32, int n, int l, float* planes, cudaStream_t st) {
  const int N = tc_npad(l);
  const int ldp = (n + 3) / 4 * 4;
  const int64_t tot = (int64_t)N * ldp;
  split_planes_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(q64, q32, n, l, N, ldp, planes);
  return cudaGetLastError();
}

// op1: W planes (or shrink output) from the column-major M (view v) and B planes (ld round4(n))
cudaError_t tc_op1(const View& v, int l, const float* planes, float* W, int64_t ldw, bool shrink, float* out,
                   int64_t Rprev, int64_t nnext, int64_t ldnext, cudaStream_t st, int max_ctas) {
  const int N = tc_npad(l);
  CUtensorMap mM, mB;
  const int ldp = (v.n + 3) / 4 * 4;
  if (!make_map(&mM, v.base, (uint64_t)v.n, (uint64_t)v.m(), (uint64_t)v.ss, 32, 128)) return cudaErrorInvalidValue;
  if (!make_map(&mB, planes, (uint64_t)v.n, (uint64_t)(2 * N), (uint64_t)ldp, 32, N)) return cudaErrorInvalidValue;
  TcOp1Args a;
  a.n = v.n; a.N = N; a.l = l; a.m = v.m(); a.nk = (v.n + kBK - 1) / kBK; a.ntiles = (v.m() + 127) / 128;
  a.W = W; a.ldw = ldw; a.shrink = shrink ? 1 : 0; a.out = out; a.Rprev = Rprev; a.nnext = nnext; a.ldnext = ldnext;
  const int grid = (int)std::min<int64_t>(max_ctas > 0 ? max_ctas : num_sms(), a.ntiles);
  switch (N) {
    case 16: return op1_launch<16>(mM, mB, a, grid, st);
    case 32: return op1_launch<32>(mM, mB, a, grid, st);
    case 48: return op1_launch<48>(mM, mB, a, grid, st);
    default: return op1_launch<64>(mM, mB, a, grid, st);
  }
}

// split-K CTAs of op2 for a grid of G: no more than the K chunks (an idle CTA would still write a
// zero Y partial that the reduction then reads)
int tc_op2_grid(const View& v, int G) {
  const int64_t nkc = (v.m() + kBK - 1) / kBK;
  return (int)std::max<int64_t>(1, std::min<int64_t>(G, nkc));
}

// op2: Ypart[G][N][nit*128] = per-CTA partial M W (or M Omega_k when sketch)
cudaError_t tc_op2(const View& v, int l, const float* W, int64_t ldw, bool sketch, uint64_t seed, uint32_t mode,
                   float* Ypart, int G, cudaStream_t st, const float* om, float* xmax) {
  const int N = tc_npad(l);
  CUtensorMap mM, mB;
  if (!make_map(&mM, v.base, (uint64_t)v.n, (uint64_t)v.m(), (uint64_t)v.ss, 32, 32,
                CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
    return cudaErrorInvalidValue;
  if (!sketch) {
    if (!make_map(&mB, W, (uint64_t)v.m(), (uint64_t)(2 * N), (uint64_t)ldw, 32, N)) return cudaErrorInvalidValue;
  } else {
    mB = mM;
  }
  TcOp2Args a;
  a.n = v.n; a.N = N; a.l = l; a.m = v.m(); a.nit = (v.n + 127) / 128; a.nkc = (v.m() + kBK - 1) / kBK;
  a.G = G; a.Ypart = Ypart; a.sketch = sketch ? 1 : 0; a.seed = seed; a.mode = mode; a.om = om;
  a.xmax = sketch ? xmax : nullptr;
  switch (N) {
    case 16: return op2_launch<16>(mM, mB, a, G, st);
    case 32: return op2_launch<32>(mM, mB, a, G, st);
    case 48: return op2_launch<48>(mM, mB, a, G, st);
    default: return op2_launch<64>(mM, mB, a, G, st);
  }
}

}  // namespace rtk
