// rtk_tile.cu -- the streaming kernels of the hot path (FP32 FFMA tiles).
//
// One templated kernel streams the mode-k unfolding M (n x m) ONCE, column
// block by column block, and per block J (b columns) computes
//
//   OP_SKETCH : W_J = Omega_k(J, :)                     (RTK-GAUSS-1, in registers/SMEM)
//               Y  += M_J W_J                           Alg. 3/4 line 5
//   OP_POWER  : W_J = M_J^T Q                           Alg. 3/4 line 7
//               Y  += M_J W_J                           -- fused single pass, M read once
//   OP_SHRINK : W_J = M_J^T U_k  -> written as rows of  G x_k U_k^T
//               the next mode's unfolding
//
// Each CTA owns LC columns of Q/Y (a "chunk"; Y = M M^T Q is column-separable)
// and a strided set of column blocks; Y partials are written per CTA and
// reduced in a fixed order by rtk_small.cu (run-to-run deterministic, no float
// atomics).  Tiles are double-buffered in shared memory with cp.async; the
// thread-level register tiles are R rows x TC columns of Q (step A) and of Y
// (step B).  -alpha Q is applied in the reduction epilogue.
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"

namespace rtk {

struct TileArgs {
  const float* M;
  int64_t P, S, sp, si, ss, m;
  int n, vec, n4;
  int n_rows, pitch, NRG, NCG, LC, nchunks, G, b;
  int64_t ntiles;
  int l;
  const float* Q;
  int qld;
  float* Ypart;
  int64_t yp_g;  // ltot * n_rows
  uint64_t seed;
  uint32_t mode;
  float* out;
  int64_t Rprev, nnext, ldnext;
};

// row held by thread row-group rg, element e (0 <= e < R)
template <int R>
__device__ __forceinline__ int row_of(int rg, int e, int NRG) {
  if constexpr (R >= 4) {
    return 4 * (rg + (e >> 2) * NRG) + (e & 3);
  } else {
    return rg * R + e;
  }
}

template <int R>
__device__ __forceinline__ void load_col(const float* __restrict__ col, int rg, int NRG, float (&m)[R]) {
  if constexpr (R >= 4) {
#pragma unroll
    for (int k = 0; k < R / 4; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(col + 4 * (rg + k * NRG));
      m[4 * k + 0] = v.x; m[4 * k + 1] = v.y; m[4 * k + 2] = v.z; m[4 * k + 3] = v.w;
    }
  } else if constexpr (R == 2) {
    const float2 v = *reinterpret_cast<const float2*>(col + 2 * rg);
    m[0] = v.x; m[1] = v.y;
  } else {
    m[0] = col[rg];
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Issue the asynchronous copy of tile `t` (columns [t*b, t*b+b)) into Ms (pitch floats per column).
__device__ __forceinline__ void issue_tile(const TileArgs& a, int64_t t, float* Ms) {
  const int64_t j0 = t * a.b;
  if (a.vec) {
    const int per_col = a.pitch >> 2;
    const int total = a.b * per_col;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int jj = idx / per_col;
      const int i = (idx - jj * per_col) << 2;
      const int64_t jg = j0 + jj;
      int bytes = 0;
      const float* src = a.M;
      if (jg < a.m && i < a.n4) {
        bytes = 16;
        src = a.M + jg * a.ss + i;
      }
      cp_async16(Ms + jj * a.pitch + i, src, bytes);
    }
  } else {
    const int total = a.b * a.pitch;
    for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
      const int jj = idx % a.b;
      const int i = idx / a.b;
      const int64_t jg = j0 + jj;
      int bytes = 0;
      const float* src = a.M;
      if (jg < a.m && i < a.n) {
        const int64_t p = jg % a.P, s = jg / a.P;
        src = a.M + p * a.sp + (int64_t)i * a.si + s * a.ss;
        bytes = 4;
      }
      cp_async4(Ms + jj * a.pitch + i, src, bytes);
    }
  }
}

template <int R, int TC, int OP, int U = 4>
__global__ void __launch_bounds__(256) tile_kernel(const TileArgs a) {
  extern __shared__ __align__(16) float smem[];
  float* Mbuf0 = smem;
  float* Mbuf1 = smem + a.b * a.pitch;
  float* Wsm = Mbuf1 + a.b * a.pitch;            // [b][LC]
  float* red = Wsm + a.b * a.LC;                 // [NW][b][LC]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int chunk = blockIdx.x % a.nchunks;
  const int grp = blockIdx.x / a.nchunks;
  const int cg = tid % a.NCG;
  const int rg = tid / a.NCG;
  const bool active = rg < a.NRG;
  const int c_base = chunk * a.LC + cg * TC;     // first global column of this thread

  // Q / U register tile (rows x TC), constant for the whole kernel
  float qv[R][TC];
  if constexpr (OP != OP_SKETCH) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int row = active ? row_of<R>(rg, e, a.NRG) : a.n;
#pragma unroll
      for (int c = 0; c < TC; ++c) {
        const int col = c_base + c;
        qv[e][c] = (row < a.n && col < a.l) ? a.Q[(int64_t)col * a.qld + row] : 0.f;
      }
    }
  }
  float acc[R][TC];
#pragma unroll
  for (int e = 0; e < R; ++e)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[e][c] = 0.f;

  int64_t t = grp;
  if (t < a.ntiles) issue_tile(a, t, Mbuf0);
  cp_async_commit();
  int buf = 0;
  for (; t < a.ntiles; t += a.G) {
    float* Ms = buf ? Mbuf1 : Mbuf0;
    const int64_t tn = t + a.G;
    if (tn < a.ntiles) issue_tile(a, tn, buf ? Mbuf0 : Mbuf1);
    cp_async_commit();
    const int64_t j0 = t * a.b;

    if constexpr (OP == OP_SKETCH) {
      // W_J = Omega_k(j0 + j, chunk*LC + c): one Box-Muller pair per work item
      const int npairs = a.b * (a.LC >> 1);
      for (int it = tid; it < npairs; it += blockDim.x) {
        const int j = it / (a.LC >> 1);
        const int c2 = (it - j * (a.LC >> 1)) << 1;   // even column within chunk
        const int cgl = chunk * a.LC + c2;             // global sketch column (even)
        const int64_t jg = j0 + j;
        float2 z = make_float2(0.f, 0.f);
        if (jg < a.m && cgl < a.l) z = omega_pair(a.seed, a.mode, (uint64_t)jg, cgl >> 2, (cgl >> 1) & 1);
        Wsm[j * a.LC + c2] = z.x;
        Wsm[j * a.LC + c2 + 1] = (cgl + 1 < a.l) ? z.y : 0.f;
      }
    }
    cp_async_wait<1>();
    __syncthreads();

    if constexpr (OP != OP_SKETCH) {
      // ---- step A: partial W over this thread's rows for U columns at a time, then
      // one batched transpose-reduce across the lanes sharing cg (lane bits >= log2 NCG).
      constexpr int NV = U * TC;
      const int nsteps = 5 - (31 - __clz(a.NCG));
      const int cnt = (nsteps >= 31 - __clz(NV)) ? 1 : (NV >> nsteps);
      for (int j0 = 0; j0 < a.b; j0 += U) {
        float mv[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (active) load_col<R>(Ms + (j0 + u) * a.pitch, rg, a.NRG, mv[u]);
          else {
#pragma unroll
            for (int e = 0; e < R; ++e) mv[u][e] = 0.f;
          }
        }
        float v[NV];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int c = 0; c < TC; ++c) {
            float s = 0.f;
#pragma unroll
            for (int e = 0; e < R; ++e) s = fmaf(mv[u][e], qv[e][c], s);
            v[u * TC + c] = s;
          }
        int coff = 0;
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          const int mask = 16 >> s;
          if (mask >= a.NCG) {
            if ((NV >> s) >= 2) {
              const bool up = (lane & mask) != 0;
#pragma unroll
              for (int i = 0; i < (NV >> (s + 1)); ++i) {
                const float send = up ? v[i] : v[i + (NV >> (s + 1))];
                const float keep = up ? v[i + (NV >> (s + 1))] : v[i];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, mask);
              }
              if (up) coff += NV >> (s + 1);
            } else {
              v[0] += __shfl_xor_sync(0xffffffffu, v[0], mask);
            }
          }
        }
        float* rw = red + ((size_t)warp * a.b + j0) * a.LC + cg * TC;
#pragma unroll
        for (int i = 0; i < NV; ++i)
          if (i < cnt) {
            const int f = coff + i;
            rw[(f / TC) * a.LC + (f % TC)] = v[i];
          }
      }
      __syncthreads();
      // ---- cross-warp sum in fixed order -> W ----
      for (int idx = tid; idx < a.b * a.LC; idx += blockDim.x) {
        float s = 0.f;
        for (int w = 0; w < nwarps; ++w) s += red[(size_t)w * a.b * a.LC + idx];
        Wsm[idx] = s;
      }
      __syncthreads();
    }

    if constexpr (OP == OP_SHRINK) {
      // ---- write W_J^T rows into the next unfolding: out(b', a + Rprev*t + Rprev*rk*c) ----
      const int tot = a.b * a.LC;
      for (int idx = tid; idx < tot; idx += blockDim.x) {
        const int c = idx / a.b;
        const int j = idx - c * a.b;
        const int tg = chunk * a.LC + c;
        const int64_t jg = j0 + j;
        if (jg < a.m && tg < a.l) {
          const int64_t aa = jg % a.Rprev;
          const int64_t tmp = jg / a.Rprev;
          const int64_t bb = tmp % a.nnext;
          const int64_t cc = tmp / a.nnext;
          const int64_t colo = aa + a.Rprev * (tg + (int64_t)a.l * cc);
          a.out[bb + a.ldnext * colo] = Wsm[j * a.LC + c];
          if (bb == a.nnext - 1)
            for (int64_t z = a.nnext; z < a.ldnext; ++z) a.out[z + a.ldnext * colo] = 0.f;
        }
      }
    } else {
      // ---- step B: Y += M_J W_J on this thread's rows x TC columns, U columns at a time ----
      if (active) {
        const float* wrow = Wsm + cg * TC;
        for (int j0 = 0; j0 < a.b; j0 += U) {
          float mv[U][R];
          float wv[U][TC];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            load_col<R>(Ms + (j0 + u) * a.pitch, rg, a.NRG, mv[u]);
#pragma unroll
            for (int c = 0; c < TC; c += 4) {
              const float4 w4 = *reinterpret_cast<const float4*>(wrow + (j0 + u) * a.LC + c);
              wv[u][c] = w4.x; wv[u][c + 1] = w4.y; wv[u][c + 2] = w4.z; wv[u][c + 3] = w4.w;
            }
          }
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < R; ++e)
#pragma unroll
              for (int c = 0; c < TC; ++c) acc[e][c] = fmaf(mv[u][e], wv[u][c], acc[e][c]);
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }
  cp_async_wait<0>();

  if constexpr (OP != OP_SHRINK) {
    if (active) {
      float* yp = a.Ypart + (int64_t)grp * a.yp_g;
#pragma unroll
      for (int c = 0; c < TC; ++c) {
        float* col = yp + (int64_t)(c_base + c) * a.n_rows;
#pragma unroll
        for (int e = 0; e < R; ++e) col[row_of<R>(rg, e, a.NRG)] = acc[e][c];
      }
    }
  }
}

// ------------------------------------------------------------------ host side
template <int R, int TC>
static cudaError_t launch_rt(const TileArgs& a, TileOp op, int grid, int nt, size_t smem,
                             cudaStream_t st) {
  void (*fn)(const TileArgs);
  if (op == OP_SKETCH) fn = tile_kernel<R, TC, OP_SKETCH>;
  else if (op == OP_POWER) fn = tile_kernel<R, TC, OP_POWER>;
  else fn = tile_kernel<R, TC, OP_SHRINK>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

int num_sms() {
  static int v = 0;
  if (!v) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
  }
  return v;
}

static size_t tile_smem(int b, int pitch, int LC, int NT) {
  return sizeof(float) * ((size_t)2 * b * pitch + (size_t)b * LC + (size_t)(NT / 32) * b * LC);
}

// Choose (R, TC, NCG, chunks, b, G) for an n x m view with l columns of Q.
TilePlan plan_tile(const View& v, int l, TileOp op, int nsm) {
  const int n = v.n;
  TilePlan best;
  double best_cost = 1e300;
  const int Rs[] = {1, 2, 4, 8, 16};
  const int TCs[] = {4, 8};
  for (int R : Rs) {
    for (int TC : TCs) {
      if (R * TC > 64 || (R == 16 && TC == 8)) continue;
      const int NRG = (n + R - 1) / R;
      for (int NCG = 1; NCG <= 32; NCG <<= 1) {
        const int lanes = 32 / NCG;
        const int NRGp = (NRG + lanes - 1) / lanes * lanes;
        const int NT = NRGp * NCG;
        const int regs = 2 * R * TC + 40;
        const int nt_max = std::min(256, (65536 / regs) / 32 * 32);
        if (NT > nt_max || NT < 32) continue;
        const int LC = NCG * TC;
        const int nchunks = (l + LC - 1) / LC;
        if (NCG > 1 && (nchunks * LC - l) >= LC / 2 && LC > 8) continue;  // mostly padding
        int pitch = (R * NRG + 3) / 4 * 4;
        // tile width: fill ~ 96 KB of double-buffered tile (2 CTAs/SM) or 200 KB (1 CTA/SM)
        const int occ_regs = std::max(1, 65536 / (NT * regs));
        int b = 64;
        size_t budget = occ_regs >= 2 ? 100 * 1024 : 200 * 1024;
        while (b > 4 && tile_smem(b, pitch, LC, NT) > budget) b -= 4;
        if (tile_smem(b, pitch, LC, NT) > 220 * 1024) continue;
        const size_t sm = tile_smem(b, pitch, LC, NT);
        const int occ = std::max(1, std::min<int>(occ_regs, (int)((228 * 1024) / (sm + 1024))));
        // cost model (cycles per column per SM, all chunks): FFMA / SMEM / SHFL
        const double nw = NT / 32.0;
        const double ffma = (op == OP_SKETCH ? 1.0 : (op == OP_POWER ? 2.0 : 1.0)) * nw * R * TC / 4.0;
        const double smem_wf = nw * ((op == OP_POWER ? 2.0 : 1.0) * R * lanes * 4.0 / 128.0 + TC / 4.0);
        const double shfl = (op == OP_SKETCH) ? 0.0 : nw * (TC + 2.0);
        double c = std::max(ffma, std::max(smem_wf, shfl)) * nchunks;
        c *= 1.0 + 8.0 / b;   // per-tile barrier / reduction overhead
        if (occ < 2) c *= 1.15;
        if (c < best_cost) {
          best_cost = c;
          best.R = R; best.TC = TC; best.NRG = NRG; best.NCG = NCG; best.LC = LC;
          best.nchunks = nchunks; best.NT = NT; best.b = b; best.pitch = pitch; best.smem = sm;
          best.G = std::max(1, nsm * occ / nchunks);
        }
      }
    }
  }
  // tuning override: RTK_PLAN_<op>="R,TC,NCG,b" (op = SKETCH|POWER|SHRINK) or RTK_PLAN
  const char* names[3] = {"RTK_PLAN_SKETCH", "RTK_PLAN_POWER", "RTK_PLAN_SHRINK"};
  const char* ov = getenv(names[op]);
  if (!ov) ov = getenv("RTK_PLAN");
  int oR, oTC, oNCG, ob;
  if (ov && sscanf(ov, "%d,%d,%d,%d", &oR, &oTC, &oNCG, &ob) == 4) {
    const int NRG = (n + oR - 1) / oR;
    const int lanes = 32 / oNCG;
    const int NRGp = (NRG + lanes - 1) / lanes * lanes;
    best.R = oR; best.TC = oTC; best.NCG = oNCG; best.NRG = NRG; best.LC = oNCG * oTC;
    best.nchunks = (l + best.LC - 1) / best.LC; best.NT = NRGp * oNCG; best.b = ob;
    best.pitch = (oR * NRG + 3) / 4 * 4;
    best.smem = tile_smem(ob, best.pitch, best.LC, best.NT);
    const int regs = 2 * oR * oTC + 40;
    const int occ = std::max(1, std::min<int>(std::max(1, 65536 / (best.NT * regs)),
                                              (int)((228 * 1024) / (best.smem + 1024))));
    best.G = std::max(1, nsm * occ / best.nchunks);
  }
  best.ntiles = (v.m() + best.b - 1) / best.b;
  if (best.G > best.ntiles) best.G = (int)best.ntiles;
  if (getenv("RTK_VERBOSE"))
    fprintf(stderr, "[rtk] plan op=%d n=%d m=%lld l=%d: R=%d TC=%d NCG=%d LC=%d chunks=%d NT=%d b=%d G=%d smem=%zu\n",
            (int)op, n, (long long)v.m(), l, best.R, best.TC, best.NCG, best.LC, best.nchunks, best.NT,
            best.b, best.G, best.smem);
  return best;
}

cudaError_t launch_tile(const TileLaunch& L, cudaStream_t st) {
  const TilePlan& p = L.tp;
  TileArgs a;
  a.M = L.v.base; a.P = L.v.P; a.S = L.v.S; a.sp = L.v.sp; a.si = L.v.si; a.ss = L.v.ss;
  a.m = L.v.m(); a.n = L.v.n;
  a.n4 = (L.v.n + 3) / 4 * 4;
  a.vec = (L.v.P == 1 && L.v.si == 1 && (L.v.ss % 4) == 0 && L.v.ss >= a.n4 &&
           ((uintptr_t)L.v.base % 16) == 0) ? 1 : 0;
  a.n_rows = p.n_rows(); a.pitch = p.pitch; a.NRG = p.NRG; a.NCG = p.NCG; a.LC = p.LC;
  a.nchunks = p.nchunks; a.G = p.G; a.b = p.b; a.ntiles = p.ntiles; a.l = L.l;
  a.Q = L.Q; a.qld = L.qld; a.Ypart = L.Ypart; a.yp_g = (int64_t)p.ltot() * p.n_rows();
  a.seed = L.seed; a.mode = L.mode; a.out = L.out; a.Rprev = L.Rprev; a.nnext = L.nnext;
  a.ldnext = L.ldnext;
  const int grid = p.G * p.nchunks;
  const size_t smem = tile_smem(p.b, p.pitch, p.LC, p.NT);
#define RTK_CASE(R_, TC_) \
  if (p.R == R_ && p.TC == TC_) return launch_rt<R_, TC_>(a, L.op, grid, p.NT, smem, st);
  RTK_CASE(1, 4) RTK_CASE(1, 8) RTK_CASE(2, 4) RTK_CASE(2, 8) RTK_CASE(4, 4) RTK_CASE(4, 8)
  RTK_CASE(8, 4) RTK_CASE(8, 8) RTK_CASE(16, 4)
#undef RTK_CASE
  return cudaErrorInvalidConfiguration;
}

}  // namespace rtk
