// rtk_tile.cu -- the streaming kernels of the hot path (FP32 FFMA tiles).
//
// One templated kernel streams the mode-k unfolding M (n x m) ONCE, column
// block by column block, and per block J (b columns) computes
//
//   OP_SKETCH : W_J = Omega_k(J, :)                     (RTK-GAUSS-2, generated in SMEM)
//               Y  += M_J W_J                           Alg. 3/4 line 5
//   OP_POWER  : W_J = M_J^T Q                           Alg. 3/4 line 7
//               Y  += M_J W_J                           -- fused single pass, M read once
//   OP_SHRINK : W_J = M_J^T U_k  -> written as rows of  G x_k U_k^T
//               the next mode's unfolding
//
// Each CTA owns LC columns of Q/Y (a "chunk"; Y = M M^T Q is column-separable)
// and a strided set of column blocks; Y partials are written per CTA and
// reduced in a fixed order by rtk_small.cu (run-to-run deterministic, no float
// atomics).  -alpha Q is applied in that reduction.
//
// Data movement: tiles are double-buffered in shared memory.  Column-major
// unfoldings (mode 1 and every ST-HOSVD mode, whose shrink writes the next
// unfolding contiguously) are loaded with TMA bulk copies (cp.async.bulk, one
// elected thread, mbarrier complete_tx); strided T-HOSVD views (P > 1) use a
// cp.async gather.  Thread work: thread (rg, cg) owns R rows x TC columns of Q
// (registers, step A) and of Y (registers, step B); warps are (32/NCG row groups)
// x NCG column groups, so the step-A row reduction is an in-warp transpose-reduce
// over the lane bits >= log2(NCG) plus a fixed-order cross-warp sum.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "rtk_gauss.cuh"
#include "rtk_internal.h"

namespace rtk {

struct TileArgs {
  const float* M;
  int64_t P, S, sp, si, ss, m;
  int n, bulk, n4;
  int n_rows, pitch, NRG, LC, nchunks, G, b;
  int64_t ntiles;
  int l;
  const float* Q;
  int qld;
  float* Ypart;
  int64_t yp_g;  // ltot * n_rows
  uint64_t seed;
  uint32_t mode;
  const float* om;   // materialised Omega_k [m][l] (Appendix D types) or nullptr (RTK-GAUSS-2)
  float* out;
  int64_t Rprev, nnext, ldnext;
};

// row held by thread row-group rg (0 <= rg < NRGp), element e (0 <= e < R)
template <int R>
__device__ __forceinline__ int row_of(int rg, int e, int NRGp) {
  if constexpr (R >= 4) {
    return 4 * (rg + (e >> 2) * NRGp) + (e & 3);
  } else {
    return rg * R + e;
  }
}

template <int R>
__device__ __forceinline__ void load_col(const float* __restrict__ col, int rg, int NRGp, float (&m)[R]) {
  if constexpr (R >= 4) {
#pragma unroll
    for (int k = 0; k < R / 4; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(col + 4 * (rg + k * NRGp));
      m[4 * k + 0] = v.x; m[4 * k + 1] = v.y; m[4 * k + 2] = v.z; m[4 * k + 3] = v.w;
    }
  } else if constexpr (R == 2) {
    const float2 v = *reinterpret_cast<const float2*>(col + 2 * rg);
    m[0] = v.x; m[1] = v.y;
  } else {
    m[0] = col[rg];
  }
}

// ---- async-copy primitives -----------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Issue tile `t` (columns [t*b, t*b+b)) into Ms.
//  bulk path : one elected thread posts expect_tx and the TMA bulk copies (one per column,
//              or a single copy when the tile is contiguous); tail columns of a ragged last
//              tile are zero-filled by all threads.
//  gather    : every thread issues 4-byte cp.async (zero-filled outside the matrix).
__device__ __forceinline__ void issue_tile(const TileArgs& a, int64_t t, float* Ms, uint64_t* bar) {
  const int64_t j0 = t * a.b;
  const int64_t rem = a.m - j0;
  const int jc = rem < (int64_t)a.b ? (int)rem : a.b;
  if (a.bulk) {
    if (jc < a.b) {
      for (int idx = threadIdx.x; idx < (a.b - jc) * a.pitch; idx += blockDim.x) Ms[jc * a.pitch + idx] = 0.f;
    }
    if (threadIdx.x == 0) {
      const unsigned colb = (unsigned)a.n4 * 4u;
      mbar_expect_tx(bar, colb * (unsigned)jc);
      if (a.ss == a.pitch && a.n4 == a.pitch) {
        bulk_g2s(Ms, a.M + j0 * a.ss, colb * (unsigned)jc, bar);
      } else {
        for (int jj = 0; jj < jc; ++jj) bulk_g2s(Ms + jj * a.pitch, a.M + (j0 + jj) * a.ss, colb, bar);
      }
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
    cp_async_commit();
  }
}

template <int R, int TC, int NCG, int OP>
__global__ void __launch_bounds__(256) tile_kernel(const TileArgs a) {
  constexpr int U = 4;                 // columns per inner batch (ILP)
  constexpr int LOG_NCG = NCG == 1 ? 0 : NCG == 2 ? 1 : NCG == 4 ? 2 : 3;
  constexpr int NSTEPS = 5 - LOG_NCG;  // lane bits that index row groups
  constexpr int NV = U * TC;
  constexpr int LOG_NV = NV >= 32 ? 5 : NV >= 16 ? 4 : NV >= 8 ? 3 : 2;
  constexpr int CNT = NSTEPS >= LOG_NV ? 1 : (NV >> NSTEPS);

  extern __shared__ __align__(128) float smem[];
  __shared__ __align__(8) uint64_t bars[2];
  const int pitch = a.pitch;
  float* Mbuf0 = smem;
  float* Mbuf1 = smem + a.b * pitch;
  float* Wsm = Mbuf1 + a.b * pitch;              // [b][LC]
  float* red = Wsm + a.b * a.LC;                 // [NW][b][LC]

  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int chunk = blockIdx.x % a.nchunks;
  const int grp = blockIdx.x / a.nchunks;
  const int cg = tid % NCG;
  const int rg = tid / NCG;                      // < NRGp (padded row groups; rows >= n are zero)
  const int NRGp = a.NRG;
  const int c_base = chunk * a.LC + cg * TC;     // first global column of this thread

  // zero the rows [n4, pitch) of both buffers once (never written by the copies)
  if (a.bulk) {
    const int w = pitch - a.n4;
    for (int idx = tid; idx < 2 * a.b * w; idx += blockDim.x) {
      const int col = idx / w, r = a.n4 + idx % w;
      smem[col * pitch + r] = 0.f;
    }
    if (tid == 0) {
      mbar_init(&bars[0], 1);
      mbar_init(&bars[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
  }
  __syncthreads();

  // Q / U register tile (rows x TC), constant for the whole kernel
  float qv[R][TC];
  if constexpr (OP != OP_SKETCH) {
#pragma unroll
    for (int e = 0; e < R; ++e) {
      const int row = row_of<R>(rg, e, NRGp);
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
  if (t < a.ntiles) issue_tile(a, t, Mbuf0, &bars[0]);
  else if (!a.bulk) cp_async_commit();
  int buf = 0;
  unsigned ph0 = 0, ph1 = 0;
  for (; t < a.ntiles; t += a.G) {
    float* Ms = buf ? Mbuf1 : Mbuf0;
    const int64_t tn = t + a.G;
    if (tn < a.ntiles) issue_tile(a, tn, buf ? Mbuf0 : Mbuf1, &bars[buf ^ 1]);
    else if (!a.bulk) cp_async_commit();
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
        if (jg < a.m && cgl < a.l) z = sketch_pair(a.om, a.l, a.seed, a.mode, (uint64_t)jg, cgl);
        Wsm[j * a.LC + c2] = z.x;
        Wsm[j * a.LC + c2 + 1] = (cgl + 1 < a.l) ? z.y : 0.f;
      }
    }
    if (a.bulk) {
      if (buf) { mbar_wait(&bars[1], ph1); ph1 ^= 1; }
      else { mbar_wait(&bars[0], ph0); ph0 ^= 1; }
    } else {
      cp_async_wait<1>();
    }
    __syncthreads();

    if constexpr (OP != OP_SKETCH) {
      // ---- step A: partial W over this thread's rows for U columns at a time, then
      // one batched transpose-reduce across the lanes sharing cg.
      for (int jb = 0; jb < a.b; jb += U) {
        float mv[U][R];
#pragma unroll
        for (int u = 0; u < U; ++u) load_col<R>(Ms + (jb + u) * pitch, rg, NRGp, mv[u]);
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
        for (int s = 0; s < NSTEPS; ++s) {
          const int mask = 16 >> s;
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
        // lanes that differ only in the lowest reduced bits hold identical values: one writes
        constexpr int LOWBITS = (NSTEPS > LOG_NV) ? ((1 << (NSTEPS - LOG_NV)) - 1) << LOG_NCG : 0;
        if ((lane & LOWBITS) == 0) {
          float* rw = red + ((size_t)warp * a.b + jb) * a.LC + cg * TC;
#pragma unroll
          for (int i = 0; i < CNT; ++i) {
            const int f = coff + i;
            rw[(f / TC) * a.LC + (f % TC)] = v[i];
          }
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
          int64_t aa, bb, cc;
          if (a.m < (1ll << 31)) {
            const uint32_t jj = (uint32_t)jg, rp = (uint32_t)a.Rprev, nn = (uint32_t)a.nnext;
            const uint32_t tmp = jj / rp;
            aa = jj - tmp * rp;
            const uint32_t c32 = tmp / nn;
            cc = c32;
            bb = tmp - c32 * nn;
          } else {
            aa = jg % a.Rprev;
            const int64_t tmp = jg / a.Rprev;
            bb = tmp % a.nnext;
            cc = tmp / a.nnext;
          }
          const int64_t colo = aa + a.Rprev * (tg + (int64_t)a.l * cc);
          a.out[bb + a.ldnext * colo] = Wsm[j * a.LC + c];
          if (bb == a.nnext - 1)
            for (int64_t z = a.nnext; z < a.ldnext; ++z) a.out[z + a.ldnext * colo] = 0.f;
        }
      }
    } else {
      // ---- step B: Y += M_J W_J on this thread's rows x TC columns, U columns at a time ----
      const float* wrow = Wsm + cg * TC;
      for (int jb = 0; jb < a.b; jb += U) {
        float mv[U][R];
        float wv[U][TC];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          load_col<R>(Ms + (jb + u) * pitch, rg, NRGp, mv[u]);
#pragma unroll
          for (int c = 0; c < TC; c += 4) {
            const float4 w4 = *reinterpret_cast<const float4*>(wrow + (jb + u) * a.LC + c);
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
    __syncthreads();
    buf ^= 1;
  }
  if (!a.bulk) cp_async_wait<0>();

  if constexpr (OP != OP_SHRINK) {
    float* yp = a.Ypart + (int64_t)grp * a.yp_g;
#pragma unroll
    for (int c = 0; c < TC; ++c) {
      float* col = yp + (int64_t)(c_base + c) * a.n_rows;
#pragma unroll
      for (int e = 0; e < R; ++e) col[row_of<R>(rg, e, NRGp)] = acc[e][c];
    }
  }
}

// ------------------------------------------------------------------ host side
template <int R, int TC, int NCG>
static cudaError_t launch_rt(const TileArgs& a, TileOp op, int grid, int nt, size_t smem,
                             cudaStream_t st) {
  void (*fn)(const TileArgs);
  if (op == OP_SKETCH) fn = tile_kernel<R, TC, NCG, OP_SKETCH>;
  else if (op == OP_POWER) fn = tile_kernel<R, TC, NCG, OP_POWER>;
  else fn = tile_kernel<R, TC, NCG, OP_SHRINK>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, nt, smem, st>>>(a);
  return cudaGetLastError();
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("RTK_PDL");
    v = (e && atoi(e) == 0) ? 0 : 1;
  }
  return v == 1;
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

static bool valid_combo(int R, int TC, int NCG) {
  const bool rt = (R == 1 || R == 2 || R == 4 || R == 8 || R == 16) && (TC == 4 || TC == 8) &&
                  R * TC <= 64;
  return rt && (NCG == 1 || NCG == 2 || NCG == 4 || NCG == 8);
}

static void finish_plan(TilePlan& p, int n, int l, int nsm) {
  const int NRG = (n + p.R - 1) / p.R;
  const int lanes = 32 / p.NCG;
  p.NRG = (NRG + lanes - 1) / lanes * lanes;   // padded row groups (extra rows are zero)
  p.NT = p.NRG * p.NCG;
  p.LC = p.NCG * p.TC;
  p.nchunks = (l + p.LC - 1) / p.LC;
  p.pitch = p.R * p.NRG;
  if (p.pitch % 4) p.pitch = (p.pitch + 3) / 4 * 4;
  p.smem = tile_smem(p.b, p.pitch, p.LC, p.NT);
  const int regs = 2 * p.R * p.TC + 48;
  const int occ = std::max(1, std::min<int>(std::max(1, 65536 / (p.NT * regs)),
                                            (int)((228 * 1024) / (p.smem + 2048))));
  p.G = std::max(1, nsm * occ / p.nchunks);
}

// Choose (R, TC, NCG, chunks, b) for an n x m view with l columns of Q.
TilePlan plan_tile(const View& v, int l, TileOp op, int nsm) {
  const int n = v.n;
  TilePlan best;
  double best_cost = 1e300;
  const int Rs[] = {1, 2, 4, 8, 16};
  const int TCs[] = {4, 8};
  for (int R : Rs) {
    for (int TC : TCs) {
      for (int NCG = 1; NCG <= 8; NCG <<= 1) {
        if (!valid_combo(R, TC, NCG)) continue;
        TilePlan p;
        p.R = R; p.TC = TC; p.NCG = NCG; p.b = 64;
        finish_plan(p, n, l, nsm);
        const int regs = 2 * R * TC + 48;
        if (p.NT > 256 || p.NT < 32 || p.NT * regs > 65536) continue;
        const int occ_regs = std::max(1, 65536 / (p.NT * regs));
        const size_t budget = occ_regs >= 2 ? 100 * 1024 : 200 * 1024;
        while (p.b > 4 && tile_smem(p.b, p.pitch, p.LC, p.NT) > budget) p.b -= 4;
        if (tile_smem(p.b, p.pitch, p.LC, p.NT) > 220 * 1024) continue;
        finish_plan(p, n, l, nsm);
        // cost model, cycles per column per SM summed over chunks: issue slots of the
        // FFMA work (+ reduction overhead) vs shared-memory wavefronts, padding included
        const double nw = p.NT / 32.0;
        const double rows_eff = (double)p.NRG * R;  // padded rows actually computed
        const double ffma = (op == OP_POWER ? 2.0 : 1.0) * rows_eff * p.LC / 32.0 / 4.0;
        const double lanes = 32.0 / NCG;
        const double red = (op == OP_SKETCH) ? 0.0 : nw * (3.0 * TC * (1.0 - 1.0 / lanes) + 2.0) / 4.0;
        const double smem_wf = nw * ((op == OP_POWER ? 2.0 : 1.0) * R * lanes * 4.0 / 128.0 + TC / 4.0);
        double c = (std::max(ffma + red, smem_wf)) * p.nchunks;
        c *= 1.0 + 6.0 / p.b;                        // per-tile barriers and cross-warp sum
        if (occ_regs < 2 && nw < 8) c *= 1.3;        // too few warps to hide latency
        if (c < best_cost) {
          best_cost = c;
          best = p;
        }
      }
    }
  }
  // tuning override: RTK_PLAN_<op>="R,TC,NCG,b" (op = SKETCH|POWER|SHRINK) or RTK_PLAN
  const char* names[3] = {"RTK_PLAN_SKETCH", "RTK_PLAN_POWER", "RTK_PLAN_SHRINK"};
  const char* ov = getenv(names[op]);
  if (!ov) ov = getenv("RTK_PLAN");
  int oR, oTC, oNCG, ob;
  if (ov && sscanf(ov, "%d,%d,%d,%d", &oR, &oTC, &oNCG, &ob) == 4 && valid_combo(oR, oTC, oNCG) &&
      ob % 4 == 0 && ob > 0) {
    best.R = oR; best.TC = oTC; best.NCG = oNCG; best.b = ob;
    finish_plan(best, n, l, nsm);
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
  a.bulk = (L.v.P == 1 && L.v.si == 1 && (L.v.ss % 4) == 0 && L.v.ss >= a.n4 && a.n4 <= p.pitch &&
            ((uintptr_t)L.v.base % 16) == 0) ? 1 : 0;
  a.n_rows = p.n_rows(); a.pitch = p.pitch; a.NRG = p.NRG; a.LC = p.LC;
  a.nchunks = p.nchunks; a.G = p.G; a.b = p.b; a.ntiles = p.ntiles; a.l = L.l;
  a.Q = L.Q; a.qld = L.qld; a.Ypart = L.Ypart; a.yp_g = (int64_t)p.ltot() * p.n_rows();
  a.seed = L.seed; a.mode = L.mode; a.om = L.om; a.out = L.out; a.Rprev = L.Rprev; a.nnext = L.nnext;
  a.ldnext = L.ldnext;
  const int grid = p.G * p.nchunks;
  const size_t smem = tile_smem(p.b, p.pitch, p.LC, p.NT);
#define RTK_CASE(R_, TC_, NCG_) \
  if (p.R == R_ && p.TC == TC_ && p.NCG == NCG_) return launch_rt<R_, TC_, NCG_>(a, L.op, grid, p.NT, smem, st);
#define RTK_CASES(R_, TC_) RTK_CASE(R_, TC_, 1) RTK_CASE(R_, TC_, 2) RTK_CASE(R_, TC_, 4) RTK_CASE(R_, TC_, 8)
  RTK_CASES(1, 4) RTK_CASES(1, 8) RTK_CASES(2, 4) RTK_CASES(2, 8) RTK_CASES(4, 4) RTK_CASES(4, 8)
  RTK_CASES(8, 4) RTK_CASES(8, 8) RTK_CASES(16, 4)
#undef RTK_CASES
#undef RTK_CASE
  return cudaErrorInvalidConfiguration;
}

}  // namespace rtk
