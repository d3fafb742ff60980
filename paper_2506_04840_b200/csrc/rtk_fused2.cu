// rtk_fused2.cu -- the fused single-HBM-pass 3xTF32 power step (Alg. 3/4 line 7, PAPER.md:261 /
// :304, Y = M (M^T Q)) on a CTA PAIR (tcgen05 cta_group::2, M = 256 across two SMs of a TPC).
//
// Why a pair.  Per 32-K stage (128 x 64 x 32, three tf32 products = 384 tensor cycles) the
// one-CTA engine (rtk_fused.cu) moves ~66 KB through each SM's shared memory: the streamed tile
// in (TMA) and out (producers), 24 KB of B operand read by the 12 MMAs and 16 KB of Q planes per
// op1 stage.  At 128 B/clk that is ~516 cycles -- more than the tensor work -- and the MMAs ran
// at ~58 instead of 32 cycles each (ncu: tensor pipe 52 % active).  With cta_group::2 each SM
// supplies only half of B (N/2 rows): 12 KB of B reads and 8 KB of Q per stage, ~385 cycles.
//
// Work split.  Pair-block J = 256 consecutive columns of the column-major unfolding M (n x m),
// CTA r owning columns [128 r, 128 r + 128) of it.
//   op1  W_J = M_J^T Q : M = 256 columns (CTA r's 128 as its TMEM lanes), K = all n rows
//        (32 per stage), N = l padded; B = Q's hi/lo planes, CTA r holding N-half r.
//        Every CTA ends with W for ITS 128 columns and all N -- no partial sums to exchange.
//   op2  Y += M_J W_J  : M = 256 rows per pair-tile (CTA r's 128 as its lanes), K = the 256
//        columns of J, N; B = W_J's hi/lo planes, CTA r holding N-half r: its own columns'
//        half r plus the peer's columns' half r, which the peer sends through DSMEM (16 KB).
// M_J is read from HBM by op1 and re-read (L2) by op2 one block later, as in the one-CTA engine.
// The streamed operand reaches the tensor core through TMEM: producer warps split x = hi + lo
// (hi = what the tf32 datapath reads, lo = x - trunc_tf32(x), exact) and tcgen05.st both planes;
// 3 MMAs per K-step (A_lo B_hi + A_hi B_lo + A_hi B_hi, fp32 accumulate in TMEM).
// Only the even CTA (the leader) issues MMAs; barriers that the MMA warp waits on live in the
// leader (the peer arrives remotely), MMA completion is multicast to both CTAs' barriers.
//
// Warp roles (480 threads per CTA): 0 TMA A tiles, 1 MMA issuer (leader) + TMEM owner,
// 2-9 producers (two groups alternating stages, one warp per TMEM lane quadrant), 10-13 epilogue
// (W -> exchange -> op2 B planes; final Y), 14 TMA Q half-planes.
// Y partials go to Ypart[pair][c][row] (row pitch nt * 256) for the fixed-order fp64 reduction.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "rtk_internal.h"
#include "rtk_sm100.cuh"

namespace rtk {
using namespace sm100;

namespace {

constexpr int kPThreads = 480;
constexpr int kPKS = 32;        // K per stage (4 MMA K-steps of 8)
constexpr int kPRA = 6;         // A tile ring slots (16 KB each)
constexpr int kPRQ = 6;         // Q half-plane ring slots
constexpr int kPTile = 128 * 32 * 4;
constexpr int kPBJ = 256;       // columns per pair-block
constexpr int kPRAH = 4;        // A ring slots of the fp16 engine (32 KB each)

// Role timers (-DRTK_PAIR_PROF=1 builds only; clock reads cost issue slots): summed wait / busy
// cycles of the two CTAs of pair 0, printed by the host at the next launch.
#ifndef RTK_PAIR_PROF
#define RTK_PAIR_PROF 0
#endif
#ifndef RTK_PAIR_ABL   // -DRTK_PAIR_ABL=1: RTK_PAIR_DBG ablations without the role timers
#define RTK_PAIR_ABL 0
#endif
#if RTK_PAIR_PROF
__device__ unsigned long long g_pair_prof[2][32];
#define PCLK() clock64()
#define PACC(slot, t0)                                                                                  \
  do {                                                                                                  \
    const int _w = threadIdx.x >> 5;                                                                    \
    if (blockIdx.x < 2 && (threadIdx.x & 31) == 0 && ((slot) < 8 || (slot) >= 16 || _w == 2) &&         \
        ((slot) < 20 || (slot) > 27 || _w == 10))                                                       \
      atomicAdd(&g_pair_prof[blockIdx.x][slot], (unsigned long long)(clock64() - (t0)));                \
  } while (0)
#else
#define PCLK() 0LL
#define PACC(slot, t0) do { (void)(t0); } while (0)
#endif

struct PairArgs {
  int n;
  int64_t m;
  int nt;          // pair row tiles (256 rows each), <= 4
  int nk1;         // op1 stages per pair-block: ceil(n / 32)
  int64_t nblk;    // pair-blocks: ceil(m / 256)
  float* Ypart;    // [P][N][nt * 256]
  const int* stop; // Alg. B.1 stop flag (nullptr: none)
  int lag;         // op1(b+1) stages issued before op2(b) (the lagged order, PSeg)
  int dbg;         // ablations (RTK_PAIR_DBG, timing only, results wrong): 1 no MMAs, 2 no A loads,
                   // 4 producers skip LDS, 8 producers skip TMEM stores, 16 no Q loads, 32 no W-plane
                   // writes, 64 no op1 A loads, 128 no op2 A loads
  int shrink;      // 1: the mode-k shrink G x_k U_k^T -- op1 only (W = M_J^T U), each CTA writes its
                   // 128 columns' W rows as the next unfolding (no exchange, no op2, no Y)
  float* out;      // shrink output (column-major, leading dimension ldnext)
  int64_t Rprev, nnext, ldnext;
  int lk;          // shrink: output columns (r_k <= N)
  int sketch;      // 1: the sketch Y = M Omega -- op2 only, B = the Omega planes streamed through the
                   // Q ring one 32-column K chunk at a time (K chunk outer, pair-tile inner), no W
  // fp16 two-plane power step (H = true, see pair_power_kernel): max|M| of this unfolding (device),
  // and cW = ceil(log2 sqrt(n)) for the W scale
  const float* xmax_in;
  int cW;
  float* xmax_out; // tf32 sketch / shrink: atomicMax of max|M| (sketch) or of the written entries (shrink)
  int op1pol;      // L2 policy of the power step's op1 tile loads: 0 evict_last, 1 evict_normal, 2 evict_first
};

// Stage order shared by the TMA, MMA and producer warps ("lagged" order):
//   op1(0)[0:L], then for each block b:  op1(b)[L:nk1], op1(b+1)[0:L], op2(b)
// op2(b) re-reads block b right after op1(b) finished it -- only op1(b+1)'s first L stages (which
// cover the W(b) exchange / op2-plane latency) sit in between -- so most of a 1 MB pair-block is
// re-read within ~L stages and the pair-blocks in flight stay far below the L2 size.  With the
// order op1(b+1), op2(b) the reuse distance was 1.5 blocks (74 pairs x 1.5 MB > the usable L2)
// and op2's re-reads missed to HBM: 8.2 GB per C5 step instead of 4.4 GB.
// Segment walker for the warps that only need the op of each stage (the producers):
struct PSeg {
  int nk1, nk2, L;
  int64_t nb, b;
  int sub;          // 0: op1(0)[0:L]; then per block 1: op1(b)[L:], 2: op1(b+1)[0:L], 3: op2(b)
  int op, rem;
  __device__ void init(int nk1_, int nk2_, int L_, int64_t nb_) {
    nk1 = nk1_; nk2 = nk2_; L = L_ < 0 ? 0 : (L_ > nk1_ ? nk1_ : L_); nb = nb_;
    b = 0; sub = 0; op = 1; rem = L;
    if (rem == 0) advance();
  }
  __device__ void advance() {   // to the next non-empty segment
    while (true) {
      if (sub == 0) { sub = 1; op = 1; rem = nk1 - L; }
      else if (sub == 1) { sub = 2; op = 1; rem = (b + 1 < nb) ? L : 0; }
      else if (sub == 2) { sub = 3; op = 2; rem = nk2; }
      else { ++b; sub = 1; op = 1; rem = (b < nb) ? nk1 - L : 0; if (b >= nb) return; }
      if (rem > 0) return;
    }
  }
  __device__ void step() { if (--rem <= 0) advance(); }
};

__device__ __forceinline__ uint32_t p_cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void p_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t p_mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// arrive on an mbarrier anywhere in the cluster (own CTA included), release at cluster scope:
// orders this thread's prior shared-memory writes / reads before the peer's acquire (per-block
// exchange handshakes only -- it costs a MEMBAR.GPU)
__device__ __forceinline__ void p_arrive_cluster(uint32_t caddr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
// per-stage signal (default .release.cta semantics, no GPU-scope membar): the TMEM stores it
// publishes are ordered by tcgen05.wait::st + tcgen05.fence::before_thread_sync
__device__ __forceinline__ void p_arrive_remote(uint32_t caddr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(caddr) : "memory");
}
__device__ __forceinline__ void p_wait_cluster(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE%=;\nbra.uni LAB_WAIT%=;\nDONE%=:\n}\n" ::"r"(smem_addr(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void p_wait_sleep(uint64_t* b, uint32_t phase) {
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(b)), "r"(phase)
        : "memory");
    if (ok) break;
    __nanosleep(64);
  }
}
__device__ __forceinline__ void p_st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(raddr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
               : "memory");
}
// local TMA load (own barrier) with an L2 cache policy
__device__ __forceinline__ void p_tma_load(void* dst, const CUtensorMap* m, int x, int y, uint64_t* b, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], "
      "%5;" ::"r"(smem_addr(dst)),
      "l"((uint64_t)m), "r"(x), "r"(y), "r"(smem_addr(b)), "l"(pol)
      : "memory");
}
// pair TMA load: data into this CTA's shared memory, completion signalled on the barrier at
// cluster address `cbar` (the leader's), .cta_group::2
__device__ __forceinline__ void p_tma_load_pair(void* dst, const CUtensorMap* m, int x, int y, uint32_t cbar,
                                                uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_addr(dst)),
      "l"((uint64_t)m), "r"(x), "r"(y), "r"(cbar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t p_policy_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t p_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Issue recipe (measured, scripts/micro/mma_stream.cu + the SASS): the MMA warp branches on
// elect.sync at the C++ level and the tcgen05 asm carries no predicate of its own; with the TMEM
// base a literal (a 512-column allocation starts at column 0) and the descriptors built from
// the shared-memory base and uniform loop counters, ptxas keeps every operand in uniform
// registers and emits back-to-back UTCHMMA.  With the elect inside each asm block every MMA paid
// ~5 R2UR conversions on the elected lane (~53 cycles per MMA against the 32-cycle tensor floor).
__device__ __forceinline__ uint32_t p_elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n.reg .b32 rx;\n.reg .pred px;\nelect.sync rx|px, 0xffffffff;\n@px mov.s32 %0, 1;\n}\n"
               : "+r"(pred));
  return pred;
}
template <uint32_t IDESC, bool H>
__device__ __forceinline__ void p_mma3(uint32_t d, uint32_t ahi, uint32_t alo, uint64_t bhi, uint64_t blo,
                                       uint32_t acc) {
  if constexpr (H) {   // fp16 planes (A from TMEM: two fp16 per 32-bit column), same operand walk
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %3, %6, p;\n"
        "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], [%1], %4, %6, 1;\n"
        "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
        "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
    return;
  }
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %5, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], [%2], %3, %6, p;\n"
      "tcgen05.mma.cta_group::2.kind::tf32.collector::a::fill [%0], [%1], %4, %6, 1;\n"
      "tcgen05.mma.cta_group::2.kind::tf32.collector::a::lastuse [%0], [%1], %3, %6, 1;\n}\n" ::"r"(d),
      "r"(ahi), "r"(alo), "l"(bhi), "l"(blo), "r"(acc), "n"(IDESC));
}
__device__ __forceinline__ void p_commit_one(uint64_t* b) {   // elected lane only
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_addr(b)),
      "h"((uint16_t)3)
      : "memory");
}
// both barriers' phases complete; the two try_waits are in flight together (one ~90-cycle
// latency instead of two)
__device__ __forceinline__ void bar_wait2(uint64_t* b1, uint32_t ph1, uint64_t* b2, uint32_t ph2) {
  asm volatile(
      "{\n.reg .pred P1, P2;\nLAB_WAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P2, [%2], %3;\n"
      "and.pred P1, P1, P2;\n"
      "@P1 bra.uni DONE%=;\nbra.uni LAB_WAIT%=;\nDONE%=:\n}\n" ::"r"(smem_addr(b1)),
      "r"(ph1), "r"(smem_addr(b2)), "r"(ph2)
      : "memory");
}
__device__ __forceinline__ void bar_wait_addr(uint32_t addr, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra.uni DONE%=;\nbra.uni LAB_WAIT%=;\nDONE%=:\n}\n" ::"r"(addr),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bar_arrive_addr(uint32_t addr) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ float4 lds128(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ float lds32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}
// both planes of a stage (hi at columns +0..31, lo at +32..63) in one 32x32b.x64 store
__device__ __forceinline__ void p_tmem_st64(uint32_t taddr, const float (&v)[32], const float (&w)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"
      "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31]),
      "f"(w[0]), "f"(w[1]), "f"(w[2]), "f"(w[3]), "f"(w[4]), "f"(w[5]), "f"(w[6]), "f"(w[7]), "f"(w[8]), "f"(w[9]),
      "f"(w[10]), "f"(w[11]), "f"(w[12]), "f"(w[13]), "f"(w[14]), "f"(w[15]), "f"(w[16]), "f"(w[17]), "f"(w[18]),
      "f"(w[19]), "f"(w[20]), "f"(w[21]), "f"(w[22]), "f"(w[23]), "f"(w[24]), "f"(w[25]), "f"(w[26]), "f"(w[27]),
      "f"(w[28]), "f"(w[29]), "f"(w[30]), "f"(w[31])
      : "memory");
}
__device__ __forceinline__ void p_tmem_st64u(uint32_t taddr, const uint32_t (&v)[32], const uint32_t (&w)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x64.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,"
      "%43,%44,%45,%46,%47,%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63,%64};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
      "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
      "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]),
      "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
      "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
      "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
      "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
      : "memory");
}
// 32 lanes x 32b, 64 consecutive columns, one wait
__device__ __forceinline__ void p_tmem_ld64(uint32_t taddr, float (&v)[64]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
      "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]), "=r"(r[32]),
        "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]), "=r"(r[40]),
        "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]), "=r"(r[48]),
        "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]), "=r"(r[56]),
        "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}
// warp max of v (>= 0), one atomicMax per warp on the float's bits (monotone for v >= 0)
__device__ __forceinline__ void p_atomic_max(float* dst, float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<unsigned int*>(dst), __float_as_uint(v));
}
// eA with max|M| 2^eA in [2^14, 2^15) (the fp16 engine's scale of M), clamped so that 2^eA and the
// Y factor stay normal floats
__device__ __forceinline__ int p_scale_exp(const float* xmax) {
  const float am = *xmax;
  const int e = (am > 0.f && am <= 3.4e38f) ? ilogbf(am) : 0;
  return max(-113, min(126, 14 - e));
}

}  // namespace

// SA: TMEM A stages (2: W double-buffered; 3: W single-buffered -- safe with this stage order,
// where op1(jb+1) follows op2(jb-1), long after W(jb) was drained -- and one more stage in flight)
//
// H = true: the power step with fp16 two-plane operands ("3xFP16") instead of 3xTF32.  Each operand
// x is scaled by a power of two s and split x s = h + l, h = fp16_rn(x s), l = fp16_rn(x s - h): 11 + 11
// significand bits, the same 22 bits a tf32 hi/lo pair carries, and the three products h h', h l',
// l h' are exact in the fp32 accumulator, so the result has the 3xTF32 error.  The
// fp16 exponent range is handled by the scales: M by 2^eA with max|M| 2^eA in [2^14, 2^15) (max|M| from
// the sketch / shrink pass that produced the unfolding), Q by 2^15 (|q| <= 1, the step kernel's
// planes), W = M^T Q by 2^-(15 + cW) (|W_jc| <= ||M_j|| ||Q_c|| <= sqrt(n) max|M|, Cauchy-Schwarz);
// every scale is exact and Y is multiplied back by 2^(cW - 2 eA) when it leaves TMEM.  Entries far
// below the maximum lose relative (not absolute) precision to fp16 gradual underflow: absolute error
// <= 2^-25 of the scaled unit, ~2^-40 of max|M| (2^-35 after the W bound).  A stage is 64 K (the
// fp16 MMA takes K = 16 per instruction in the same 32 bytes), so every per-stage handshake covers
// twice the data, and the TMEM A stage (hi 32 + lo 32 columns of packed pairs) keeps its size.
template <int N, int SA, bool H>
__global__ void __launch_bounds__(kPThreads, 1) pair_power_kernel(const __grid_constant__ CUtensorMap tmQ,
                                                                  const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmA2,
                                                                  const PairArgs a) {
  constexpr int N2 = N / 2;                  // B rows held by each CTA
  constexpr int KS = H ? 64 : kPKS;          // K per stage
  constexpr int SLOT = H ? 2 * kPTile : kPTile;   // A ring slot: one stage (H: two 32-K TMA boxes)
  constexpr int NRA = H ? kPRAH : kPRA;      // A ring slots
  constexpr int K2 = kPBJ / KS;              // op2 stages per pair-tile
  constexpr int QS = 2 * N2 * 128;           // Q ring slot: hi | lo half-planes of one stage (128-B rows)
  constexpr int PL = K2 * N2 * 128;          // one op2 B plane: 256 columns x N2
  constexpr uint32_t IDESC = H ? idesc_f16(256, N) : idesc_tf32(256, N, 0, 0);
  constexpr int NW = SA == 2 ? 2 : 1;         // W buffers
  constexpr int TA0 = 256 + NW * N;          // TMEM: Y tiles at 0, W buffers at 256, A ring
  static_assert(N % 16 == 0 && N >= 16 && N <= 64, "cta_group::2 N");
  static_assert(TA0 + 64 * SA <= 512, "TMEM budget");
  // the two producer groups take alternate stages and must own disjoint ring slots / TMEM stages
  // (a slot shared by both groups lets one group's parity wait pass on the other group's older
  // phase), so both ring depths are even
  static_assert(NRA % 2 == 0 && SA % 2 == 0 || SA == 3, "ring depth vs producer groups");
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (smem_addr(smraw) & 1023u)) & 1023u);
  uint8_t* smR = sm;                          // NRA x SLOT
  uint8_t* smQ = smR + NRA * SLOT;            // kPRQ x QS
  uint8_t* smP = smQ + kPRQ * QS;             // hi plane | lo plane
  float* rbuf = (float*)(smP + 2 * PL);       // 128 x N2 received from the peer
  __shared__ __align__(8) uint64_t r_full[NRA], r_empty[NRA], q_full[kPRQ], q_empty[kPRQ];
  __shared__ __align__(8) uint64_t a_full[SA], a_empty[SA], w_full[2], w_empty[2];
  __shared__ __align__(8) uint64_t p_full, p_empty, y_full, x_full, credit;
  __shared__ uint32_t tbase_s;

  pdl_wait();
  if (a.stop && *(volatile const int*)a.stop) return;   // uniform over the grid: before any barrier
  const int dbg = (RTK_PAIR_PROF || RTK_PAIR_ABL) ? a.dbg : 0;   // ablations only in diagnostic builds
  const bool SHR = a.shrink != 0;   // op1 only (a.nt == 0: no op2 stages, no Y)
  const bool SKT = a.sketch != 0;   // op2 only (no op1 stages, no W)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = p_cluster_rank(), peer = rank ^ 1u;
  const bool leader = rank == 0;
  const int64_t pid = blockIdx.x >> 1, P = gridDim.x >> 1;
  const int64_t nb = (a.nblk > pid) ? (a.nblk - pid + P - 1) / P : 0;   // pair-blocks of this pair
  const int nk1 = SKT ? 0 : a.nk1, nk2 = a.nt * K2;
  const int lagL = a.lag < 0 ? 0 : (a.lag > nk1 ? nk1 : a.lag);   // op1(b+1) stages ahead of op2(b)
  const int64_t total = nb * (nk1 + nk2);

  // stage order (TMA, MMA and producer warps alike): op1(0), [op1(1)], op2(0), op1(2), op2(1), ..., op2(nb-1)

  if (threadIdx.x == 0) {
    for (int s = 0; s < NRA; ++s) { bar_init(&r_full[s], 1); bar_init(&r_empty[s], 4); }
    for (int s = 0; s < kPRQ; ++s) { bar_init(&q_full[s], 1); bar_init(&q_empty[s], 1); }
    for (int s = 0; s < SA; ++s) { bar_init(&a_full[s], 8); bar_init(&a_empty[s], 1); }
    for (int b = 0; b < 2; ++b) { bar_init(&w_full[b], 1); bar_init(&w_empty[b], 8); }
    bar_init(&p_full, 8); bar_init(&p_empty, 1); bar_init(&y_full, 1);
    bar_init(&x_full, 1); bar_init(&credit, 4);
    bar_fence_init();
    tma_prefetch(&tmQ);
    tma_prefetch(&tmA);
    tma_prefetch(&tmA2);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(&tbase_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  p_cluster_sync();   // both CTAs' barriers initialised and TMEM allocated before any cross-CTA use
  tc_fence_after();
  // a 512-column allocation owns the whole TMEM: its base is column 0 of lane 0 (the literal keeps
  // the MMA operands uniform, see p_elect_one)
  if (tbase_s != 0u) __trap();
  constexpr uint32_t tbase = 0u;
  auto colbase = [&](int64_t jb) -> int64_t { return (pid + jb * P) * kPBJ; };

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA: A tiles (own ring)
    // walks the same segment sequence as the MMA warp: op1(0), [op1(1)], op2(0), op1(2), op2(1), ...
    if (lane == 0) {
      const uint64_t pol_drop = p_policy_first();
      uint64_t pol_keep = p_policy_last();
      if (a.op1pol == 1) asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_keep));
      if (a.op1pol == 2) pol_keep = pol_drop;
      int sl = 0;
      uint32_t ph = 0;
      auto load = [&](int op, int x, int64_t y) {
        { const long long _t0 = PCLK(); bar_wait(&r_empty[sl], ph ^ 1); PACC(17, _t0); }
        uint8_t* dst = smR + sl * SLOT;
        if ((dbg & 2) || (op == 1 && (dbg & 64)) || (op == 2 && (dbg & 128))) {
          bar_arrive(&r_full[sl]);
        } else {
          bar_expect_tx(&r_full[sl], SLOT);
          if (op == 1) {   // [128 j][32 i], SW128 (H: rows x.. and x + 32.. as two such tiles)
            p_tma_load(dst, &tmA, x, (int)y, &r_full[sl], SHR ? pol_drop : pol_keep);
            if constexpr (H) p_tma_load(dst + kPTile, &tmA, x + 32, (int)y, &r_full[sl], pol_keep);
          } else {         // [32 c][128 i] (H: [64 c][128 i])
            p_tma_load(dst, &tmA2, x, (int)y, &r_full[sl], pol_drop);
            if constexpr (H) p_tma_load(dst + kPTile, &tmA2, x, (int)y + 32, &r_full[sl], pol_drop);
          }
        }
        if (++sl == NRA) { sl = 0; ph ^= 1; }
      };
      const int L = lagL;
      auto seg1 = [&](int64_t blk, int k0, int k1) {   // all rows of this CTA's 128 columns
        const int64_t y = colbase(blk) + 128 * rank;
        for (int k = k0; k < k1; ++k) {
          load(1, KS * k, y);
        }
      };
      auto seg2 = [&](int64_t blk) {                    // this CTA's rows of each pair-tile x 256 columns
        const int64_t c0 = colbase(blk);
        if (SKT) {   // the MMA's sketch order: K chunk outer, pair-tile inner
          for (int kq = 0; kq < K2; ++kq)
            for (int tt = 0; tt < a.nt; ++tt) load(2, 256 * tt + 128 * (int)rank, c0 + KS * kq);
        } else {
          for (int tt = 0; tt < a.nt; ++tt)
            for (int kq = 0; kq < K2; ++kq) load(2, 256 * tt + 128 * (int)rank, c0 + KS * kq);
        }
      };
      if (nb > 0) seg1(0, 0, L);
      for (int64_t b = 0; b < nb; ++b) {
        seg1(b, L, nk1);
        if (b + 1 < nb) seg1(b + 1, 0, L);
        seg2(b);
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader)
    if (leader) {
      const uint64_t q0 = sdesc_sw128(smem_addr(smQ), 16, 1024);
      const uint64_t p0 = sdesc_sw128(smem_addr(smP), 16, 1024);
      const bool mma_on = !(dbg & 1);
      int sa = 0;            // TMEM A stage of the current stage (counter, no division)
      uint32_t aph = 0;      // its phase
      int qsl = 0;
      uint32_t qph = 0;
      auto next_a = [&]() { if (++sa == SA) { sa = 0; aph ^= 1; } };
      const long long _tm0 = PCLK();
      auto op1 = [&](int64_t blk, int k) {   // op1(blk) stage k -> W buffer blk % NW
        const int b = NW == 2 ? (int)(blk & 1) : 0;
        if (k == 0) {
          const int64_t wu = NW == 2 ? (blk >> 1) : blk;   // use count of buffer b
          { const long long _t0 = PCLK(); p_wait_cluster(&w_empty[b], (uint32_t)((wu & 1) ^ 1)); PACC(5, _t0); }
        }
        { const long long _t0 = PCLK(); bar_wait2(&q_full[qsl], qph, &a_full[sa], aph); PACC(1, _t0); }
        tc_fence_after();
        if (p_elect_one()) {
          const uint32_t d = 256u + (uint32_t)(b * N);
          const uint64_t qs = q0 + (uint64_t)((qsl * QS) >> 4);
          const uint32_t ta = (uint32_t)(TA0 + 64 * sa);
          if (mma_on) {
#pragma unroll
            for (int k8 = 0; k8 < 4; ++k8)
              p_mma3<IDESC, H>(d, ta + 8 * k8, ta + 32 + 8 * k8, qs + (uint64_t)((k8 * 32) >> 4),
                            qs + (uint64_t)((N2 * 128 + k8 * 32) >> 4), (k | k8) != 0);
          }
          p_commit_one(&a_empty[sa]);
          p_commit_one(&q_empty[qsl]);
          if (k == nk1 - 1) p_commit_one(&w_full[b]);
        }
        __syncwarp();
        if (++qsl == kPRQ) { qsl = 0; qph ^= 1; }
        next_a();
      };
      auto op2 = [&](int64_t blk) {           // op2(blk): pair-tile t, K chunk kq
        { const long long _t0 = PCLK(); p_wait_cluster(&p_full, (uint32_t)(blk & 1)); PACC(4, _t0); }
        for (int t = 0; t < a.nt; ++t) {
          const uint32_t d = (uint32_t)(t * N);
#pragma unroll 1
          for (int kq = 0; kq < K2; ++kq) {
            { const long long _t0 = PCLK(); bar_wait(&a_full[sa], aph); PACC(3, _t0); }
            tc_fence_after();
            if (p_elect_one()) {
              const uint32_t ta = (uint32_t)(TA0 + 64 * sa);
              if (mma_on) {
#pragma unroll
                for (int k8 = 0; k8 < 4; ++k8) {
                  const uint32_t boff = (uint32_t)(kq * (N2 * 128) + k8 * 32);
                  p_mma3<IDESC, H>(d, ta + 8 * k8, ta + 32 + 8 * k8, p0 + (uint64_t)(boff >> 4),
                                p0 + (uint64_t)((PL + boff) >> 4), (blk > 0 || kq > 0 || k8 > 0) ? 1u : 0u);
                }
              }
              p_commit_one(&a_empty[sa]);
            }
            __syncwarp();
            next_a();
          }
        }
        if (p_elect_one()) p_commit_one(&p_empty);
        __syncwarp();
      };
      auto op2s = [&](int64_t blk) {          // sketch op2(blk): K chunk kq (Omega, Q ring) x pair-tile t
#pragma unroll 1
        for (int kq = 0; kq < K2; ++kq) {
          { const long long _t0 = PCLK(); bar_wait(&q_full[qsl], qph); PACC(2, _t0); }
          const uint64_t qs = q0 + (uint64_t)((qsl * QS) >> 4);
#pragma unroll 1
          for (int t = 0; t < a.nt; ++t) {
            { const long long _t0 = PCLK(); bar_wait(&a_full[sa], aph); PACC(3, _t0); }
            tc_fence_after();
            if (p_elect_one()) {
              const uint32_t ta = (uint32_t)(TA0 + 64 * sa);
              if (mma_on) {
#pragma unroll
                for (int k8 = 0; k8 < 4; ++k8)
                  p_mma3<IDESC, H>((uint32_t)(t * N), ta + 8 * k8, ta + 32 + 8 * k8, qs + (uint64_t)((k8 * 32) >> 4),
                                qs + (uint64_t)((N2 * 128 + k8 * 32) >> 4), (blk > 0 || kq > 0 || k8 > 0) ? 1u : 0u);
              }
              p_commit_one(&a_empty[sa]);
            }
            __syncwarp();
            next_a();
          }
          if (p_elect_one()) p_commit_one(&q_empty[qsl]);
          __syncwarp();
          if (++qsl == kPRQ) { qsl = 0; qph ^= 1; }
        }
      };
      const int L = lagL;
      if (SKT) {
        for (int64_t b = 0; b < nb; ++b) op2s(b);
      } else {
        if (nb > 0)
          for (int k = 0; k < L; ++k) op1(0, k);
        for (int64_t b = 0; b < nb; ++b) {
          for (int k = L; k < nk1; ++k) op1(b, k);
          if (b + 1 < nb)
            for (int k = 0; k < L; ++k) op1(b + 1, k);
          if (!SHR) op2(b);
        }
      }
      if (p_elect_one()) p_commit_one(&y_full);
      __syncwarp();
      if (lane == 0) PACC(0, _tm0);
    }
  } else if (warp < 10) {
    // ---------------------------------------------------------------- producers: tile -> split -> TMEM
    // Instruction-lean loop (the producers' issue slots bound the stage rate): ring slot / TMEM
    // stage / phases are running counters, the stage walk is a segment counter (a producer needs
    // only the op of a stage), lo = x - trunc_tf32(x) in packed FADD2.
    const int q = warp & 3, g = (warp - 2) >> 2;
    const int lt = 32 * q + lane;   // TMEM lane = op1 column / op2 row within this CTA's 128
    const uint32_t tq0 = tbase + ((uint32_t)(32 * q) << 16) + TA0;
    const uint32_t afull_c0 = p_mapa(smem_addr(&a_full[0]), 0);   // the leader's barriers
    const uint32_t rfull0 = smem_addr(&r_full[0]), rempty0 = smem_addr(&r_empty[0]), aempty0 = smem_addr(&a_empty[0]);
    const uint32_t tile1 = smem_addr(smR) + (uint32_t)lt * 128u;   // op1: row lt of the SW128 tile
    const uint32_t tile2 = smem_addr(smR) + (uint32_t)lt * 4u;     // op2: column lt of [32 c][128 i]
    const uint32_t sw = (uint32_t)(lt & 7);
    PSeg w;
    w.init(nk1, nk2, lagL, nb);
    if (g == 1) w.step();
    int sl = g, ts = g;                            // ring slot / TMEM stage of this group's stage
    uint32_t rph = 0, tph = 0;
    float vmax = 0.f;                              // sketch: running max|M|
    float sA = 1.f;                                // H: the exact scale 2^eA of M
    if constexpr (H) sA = ldexpf(1.f, p_scale_exp(a.xmax_in));
    const long long _tp0 = PCLK();
    for (int64_t s = g; s < total; s += 2) {
      { const long long _t0 = PCLK(); bar_wait_addr(rfull0 + 8u * (uint32_t)sl, rph); PACC(9, _t0); }
      const long long _tl0 = PCLK();
      float v[kPKS], lo[kPKS];          // tf32: hi (the raw value) and lo planes
      uint32_t hv[32], lv[32];          // H: packed fp16 pairs (k, k + 1) of the hi and lo planes
      if constexpr (H) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {   // the stage's two 32-K halves
          float x[32];
          if (w.op == 1) {
            const uint32_t base = tile1 + (uint32_t)sl * SLOT + (uint32_t)(hf * kPTile);
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const float4 y = lds128(base + ((((uint32_t)c) ^ sw) << 4));
              x[4 * c] = y.x; x[4 * c + 1] = y.y; x[4 * c + 2] = y.z; x[4 * c + 3] = y.w;
            }
          } else {
            const uint32_t base = tile2 + (uint32_t)sl * SLOT + (uint32_t)(hf * kPTile);
#pragma unroll
            for (int c = 0; c < 32; ++c) x[c] = lds32(base + (uint32_t)(c * 512));
          }
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const float2 xs = __fmul2_rn(make_float2(x[e], x[e + 1]), make_float2(sA, sA));   // exact
            const __half2 h = __floats2half2_rn(xs.x, xs.y);
            const float2 hb = __half22float2(h);
            const float2 r = __fadd2_rn(xs, make_float2(-hb.x, -hb.y));                      // exact
            const __half2 l2 = __floats2half2_rn(r.x, r.y);
            hv[16 * hf + e / 2] = *reinterpret_cast<const uint32_t*>(&h);
            lv[16 * hf + e / 2] = *reinterpret_cast<const uint32_t*>(&l2);
          }
        }
      } else {
#if RTK_PAIR_PROF || RTK_PAIR_ABL
      if (dbg & 4) {
#pragma unroll
        for (int c = 0; c < kPKS; ++c) v[c] = (float)(c + lt);
      } else
#endif
      if (w.op == 1) {
        const uint32_t base = tile1 + (uint32_t)sl * SLOT;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = lds128(base + ((((uint32_t)c) ^ sw) << 4));
          v[4 * c] = x.x; v[4 * c + 1] = x.y; v[4 * c + 2] = x.z; v[4 * c + 3] = x.w;
        }
      } else {
        const uint32_t base = tile2 + (uint32_t)sl * SLOT;
#pragma unroll
        for (int c = 0; c < kPKS; ++c) v[c] = lds32(base + (uint32_t)(c * 512));
        if (SKT) {   // max|M| of the unfolding (every element passes through one sketch stage)
#pragma unroll
          for (int c = 0; c < kPKS; ++c) vmax = fmaxf(vmax, fabsf(v[c]));
        }
      }
#pragma unroll
      for (int e = 0; e < kPKS; e += 2) {
        const float2 d = __fadd2_rn(make_float2(v[e], v[e + 1]), make_float2(-tf32_trunc(v[e]), -tf32_trunc(v[e + 1])));
        lo[e] = d.x; lo[e + 1] = d.y;
      }
      }
      __syncwarp();
      PACC(12, _tl0);
      if (lane == 0) bar_arrive_addr(rempty0 + 8u * (uint32_t)sl);
      { const long long _t0 = PCLK(); bar_wait_addr(aempty0 + 8u * (uint32_t)ts, tph ^ 1u); PACC(10, _t0); }
      tc_fence_after();
      const uint32_t tq = tq0 + (uint32_t)(64 * ts);
#if RTK_PAIR_PROF || RTK_PAIR_ABL
      if (!(dbg & 8))
#endif
      {
        const long long _t0 = PCLK();
        if constexpr (H) p_tmem_st64u(tq, hv, lv);
        else p_tmem_st64(tq, v, lo);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        PACC(11, _t0);
      }
      const long long _ta0 = PCLK();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) p_arrive_remote(afull_c0 + 8u * (uint32_t)ts);
      PACC(13, _ta0);
      const long long _tw0 = PCLK();
      sl += 2;
      if (sl >= NRA) { sl -= NRA; rph ^= 1u; }
      ts += 2;
      if (ts >= SA) { ts -= SA; tph ^= 1u; }
      w.step();
      w.step();
      PACC(14, _tw0);
    }
    PACC(8, _tp0);
    if (SKT && a.xmax_out) p_atomic_max(a.xmax_out, vmax);
  } else if (warp < 14) {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;
    const int j = 32 * q + lane;   // this CTA's block column = TMEM lane of W
    const uint32_t wempty_c[2] = {p_mapa(smem_addr(&w_empty[0]), 0), p_mapa(smem_addr(&w_empty[1]), 0)};
    const uint32_t pfull_c = p_mapa(smem_addr(&p_full), 0);
    const uint32_t rdst = p_mapa(smem_addr(rbuf + j * N2), peer);
    const uint32_t rbar = p_mapa(smem_addr(&x_full), peer);
    const uint32_t rcredit = p_mapa(smem_addr(&credit), peer);
    float emax = 0.f;   // shrink: running max of the entries written
    float tW = 1.f;     // H: the exact scale 2^-(15 + cW) of W
    double yback = 1.0; // H: Y = TMEM value * 2^(cW - 2 eA)
    if constexpr (H) {
      const int eA = p_scale_exp(a.xmax_in);
      tW = ldexpf(1.f, -(15 + a.cW));
      yback = ldexp(1.0, a.cW - 2 * eA);
    }
    const long long _te0 = PCLK();
    for (int64_t jb = 0; jb < (SKT ? 0 : nb); ++jb) {
      const int b = NW == 2 ? (int)(jb & 1) : 0;
      { const long long _t0 = PCLK(); p_wait_sleep(&w_full[b], (uint32_t)((NW == 2 ? (jb >> 1) : jb) & 1)); PACC(21, _t0); }
      tc_fence_after();
      const long long _tld0 = PCLK();
      float w[N];
      if constexpr (N == 64) {
        p_tmem_ld64(tbase + ((uint32_t)(32 * q) << 16) + 256 + b * N, w);
      } else {
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
          float v[16];
          tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + 256 + b * N + c0, v);
#pragma unroll
          for (int c = 0; c < 16; ++c) w[c0 + c] = v[c];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) p_arrive_cluster(wempty_c[b]);
      PACC(25, _tld0);
      if (SHR) {
        // G x_k U_k^T: W(j, c) = sum_i M(i, j) U(i, c) is entry (c, j) of the shrunk unfolding; write
        // it at its place in the (k+1)-unfolding (Rprev x nnext x rest), rows padded to ldnext
        const int64_t col = colbase(jb) + 128 * (int64_t)rank + j;
        if (col < a.m) {
          const int64_t aa = col % a.Rprev, tmp = col / a.Rprev;
          const int64_t bb = tmp % a.nnext, cc = tmp / a.nnext;
          const int64_t cs = a.ldnext * a.Rprev;   // entry (c, col) at o[cs c]
          float* o = a.out + bb + a.ldnext * (aa + a.Rprev * (int64_t)a.lk * cc);
#pragma unroll
          for (int c = 0; c < N; ++c)
            if (c < a.lk) {
              o[cs * c] = w[c];
              emax = fmaxf(emax, fabsf(w[c]));
            }
          if (bb == a.nnext - 1 && a.ldnext > a.nnext)   // zero the row padding of this column
            for (int cr = 0; cr < a.lk; ++cr)
              for (int64_t z = 1; z < a.ldnext - a.nnext + 1; ++z) o[cs * cr + z] = 0.f;
        }
        continue;
      }
      // exchange: the peer's N-half of my column j goes to the peer's rbuf row j; I receive the
      // peer's column j, my N-half.  Row j's 16-B chunk c4 sits at (c4 + j) mod N2/4 so that the
      // reads below are bank-conflict-free.
      const uint32_t px = (uint32_t)(jb & 1);
      if (threadIdx.x == 10 * 32)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&x_full)),
                     "r"((uint32_t)(128 * N2 * 4))
                     : "memory");
      // own N-half / the peer's N-half of my column (selects keep the register indices static)
      float wo[N2], wsnd[N2];
#pragma unroll
      for (int c = 0; c < N2; ++c) {
        wo[c] = rank ? w[N2 + c] : w[c];
        wsnd[c] = rank ? w[c] : w[N2 + c];
      }
      { const long long _t0 = PCLK(); p_wait_cluster(&credit, px ^ 1); PACC(22, _t0); }   // the peer has read my previous send
#pragma unroll
      for (int c4 = 0; c4 < N2 / 4; ++c4)
        p_st_async_v4(rdst + 16 * ((c4 + j) % (N2 / 4)),
                      make_float4(wsnd[4 * c4], wsnd[4 * c4 + 1], wsnd[4 * c4 + 2], wsnd[4 * c4 + 3]), rbar);
      { const long long _t0 = PCLK(); p_wait_cluster(&x_full, px); PACC(22, _t0); }
      float pw[N2];
#pragma unroll
      for (int c4 = 0; c4 < N2 / 4; ++c4) {
        const float4 x = *reinterpret_cast<const float4*>(rbuf + j * N2 + 4 * ((c4 + j) % (N2 / 4)));
        pw[4 * c4] = x.x; pw[4 * c4 + 1] = x.y; pw[4 * c4 + 2] = x.z; pw[4 * c4 + 3] = x.w;
      }
      __syncwarp();
      if (lane == 0) p_arrive_cluster(rcredit);
      // op2 B planes of this CTA (N-half `rank`): own column at K index 128 rank + j, the peer's
      // column at 128 peer + j; hi = rna tf32, lo exact; once op2(jb-1) has released the planes
      { const long long _t0 = PCLK(); p_wait_sleep(&p_empty, (uint32_t)((jb & 1) ^ 1)); PACC(23, _t0); }
      const int ko = 128 * (int)rank + j, kp = 128 * (int)peer + j;
      const long long _tpl0 = PCLK();
      if (dbg & 32) {
      } else if constexpr (H) {   // fp16 planes [K/64][N2 c][64 k] (128-B rows, SW128), W scaled by tW
        const uint32_t ro = (uint32_t)((ko >> 6) * (N2 * 128) + (((ko & 63) >> 3) << 4) + ((ko & 7) << 1));
        const uint32_t rp = (uint32_t)((kp >> 6) * (N2 * 128) + (((kp & 63) >> 3) << 4) + ((kp & 7) << 1));
#pragma unroll
        for (int c = 0; c < N2; ++c) {
          const float xo = wo[c] * tW, xp = pw[c] * tW;
          const __half ho = __float2half_rn(xo), hp = __float2half_rn(xp);
          const __half lo2 = __float2half_rn(xo - __half2float(ho)), lp2 = __float2half_rn(xp - __half2float(hp));
          const uint32_t sw16 = (uint32_t)((c & 7) << 4), rb = (uint32_t)(c * 128);
          *reinterpret_cast<__half*>(smP + ((ro ^ sw16) + rb)) = ho;
          *reinterpret_cast<__half*>(smP + PL + ((ro ^ sw16) + rb)) = lo2;
          *reinterpret_cast<__half*>(smP + ((rp ^ sw16) + rb)) = hp;
          *reinterpret_cast<__half*>(smP + PL + ((rp ^ sw16) + rb)) = lp2;
        }
      } else {
#pragma unroll
      for (int c = 0; c < N2; ++c) {
        const float xo = wo[c], xp = pw[c];
        const float ho = tf32_rna(xo), hp = tf32_rna(xp);
        const uint32_t oo = (uint32_t)((ko >> 5) * (N2 * 128)) + sw128_offset(c, ko & 31);
        const uint32_t op = (uint32_t)((kp >> 5) * (N2 * 128)) + sw128_offset(c, kp & 31);
        *reinterpret_cast<float*>(smP + oo) = ho;
        *reinterpret_cast<float*>(smP + PL + oo) = xo - ho;
        *reinterpret_cast<float*>(smP + op) = hp;
        *reinterpret_cast<float*>(smP + PL + op) = xp - hp;
      }
      }
      fence_async_smem();
      __syncwarp();
      PACC(26, _tpl0);
      if (lane == 0) p_arrive_cluster(pfull_c);
    }
    PACC(20, _te0);
    if (SHR && a.xmax_out) p_atomic_max(a.xmax_out, emax);
    // ---- final: this CTA's Y rows (its half of every pair-tile) -> Ypart[pair][c][row]
    const int rows_tot = a.nt * 256;
    float* yp = a.Ypart + pid * (int64_t)N * rows_tot;
    if (nb > 0 && !SHR) {
      p_wait_sleep(&y_full, 0);
      tc_fence_after();
    }
    for (int t = 0; t < a.nt; ++t) {
      const int i = 256 * t + 128 * (int)rank + j;
#pragma unroll
      for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        if (nb > 0) tmem_ld16(tbase + ((uint32_t)(32 * q) << 16) + t * N + c0, v);
        else {
#pragma unroll
          for (int c = 0; c < 16; ++c) v[c] = 0.f;
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) yp[(int64_t)(c0 + c) * rows_tot + i] = H ? (float)((double)v[c] * yback) : v[c];
      }
    }
    tc_fence_before();
  } else if (lane == 0) {
    // ---------------------------------------------------------------- TMA: Q half-planes (pair)
    // op1 stage k of every block: rows 32k.., N-half `rank` of the hi and lo planes, completion on
    // the leader's q_full (which expects both halves)
    const uint64_t pol_keep = p_policy_last();
    const uint32_t qfull0 = p_mapa(smem_addr(&q_full[0]), 0);
    int sl = 0;
    uint32_t ph = 0;
    // sketch: the K chunks of the Omega planes (columns colbase + 32 kq of the pair-block), read once
    const uint64_t pol_q = SKT ? p_policy_first() : pol_keep;
    const int nq = SKT ? K2 : nk1;
    for (int64_t jb = 0; jb < nb; ++jb)
      for (int k = 0; k < nq; ++k) {
        { const long long _t0 = PCLK(); bar_wait(&q_empty[sl], ph ^ 1); PACC(24, _t0); }
        uint8_t* sq = smQ + sl * QS;
        const uint32_t cb = qfull0 + 8u * (uint32_t)sl;
        const int x = SKT ? (int)(colbase(jb) + KS * k) : KS * k;
        if (dbg & 16) {
          if (leader) bar_arrive(&q_full[sl]);
        } else {
          if (leader) bar_expect_tx(&q_full[sl], 2 * QS);   // both CTAs' halves
          p_tma_load_pair(sq, &tmQ, x, (int)rank * N2, cb, pol_q);
          p_tma_load_pair(sq + N2 * 128, &tmQ, x, N + (int)rank * N2, cb, pol_q);
        }
        if (++sl == kPRQ) { sl = 0; ph ^= 1; }
      }
  }
  __syncthreads();
  p_cluster_sync();   // no CTA releases TMEM / leaves while the peer may still use it
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

// ---------------------------------------------------------------------- test hook helpers
__global__ void absmax_kernel(const float* __restrict__ M, int n, int64_t m, int64_t ld, float* xmax) {
  float v = 0.f;
  for (int64_t j = blockIdx.x; j < m; j += gridDim.x)
    for (int i = threadIdx.x; i < n; i += blockDim.x) v = fmaxf(v, fabsf(M[j * ld + i]));
  p_atomic_max(xmax, v);
}
__global__ void split16_kernel(const float* __restrict__ Q, int n, int l, int N, int pld, __half* planes) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)N * pld;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / pld), i = (int)(idx % pld);
    const double x = (c < l && i < n) ? (double)Q[(int64_t)c * n + i] * 32768.0 : 0.0;
    const __half hi = __float2half_rn((float)x);
    planes[(int64_t)c * pld + i] = hi;
    planes[(int64_t)(N + c) * pld + i] = __float2half_rn((float)(x - (double)__half2float(hi)));
  }
}
cudaError_t pair_prepare16(const View& v, const float* Q, int l, int N, int pld, float* planes, float* xmax,
                           cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(xmax, 0, 4, st);
  if (e != cudaSuccess) return e;
  absmax_kernel<<<1024, 256, 0, st>>>(v.base, v.n, v.m(), v.ss, xmax);
  split16_kernel<<<256, 256, 0, st>>>(Q, v.n, l, N, pld, reinterpret_cast<__half*>(planes));
  return cudaGetLastError();
}

// ---------------------------------------------------------------------- host side
typedef CUresult (*PFN_encode2_t)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encode2_t pair_encode_fn() {
  static PFN_encode2_t fn = nullptr;
  static bool done = false;
  if (!done) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = (PFN_encode2_t)p;
    done = true;
  }
  return fn;
}

bool pair_supported(const View& v, int l) {
  // default for n_k > 256 (C3 / C5 mode 1): each CTA streams all rows of its 128 columns, which halves
  // the B-operand and Q traffic per SM; for n_k <= 256 the one-CTA engine's 128-row tiles waste less
  // (a pair-tile is 256 rows).  RTK_PAIR=0 / 1 forces it off / on.
  // and for unfoldings with at least one 256-column pair-block per two pairs: narrower ones (C5 mode
  // 3, m = 2500: 10 pair-blocks) are faster on the one-CTA engine's 128-column blocks (ncu, 1000 x
  // 2500: 27 vs 36 us; 1000 x 5e4: 99 vs 88 us -- scripts/ncu_small_m.sh; in the solve C3 mode 2,
  // 47 pair-blocks, stays faster on the pair)
  const char* e = getenv("RTK_PAIR");
  if (e && e[0] == '0') return false;
  if (!(e && e[0] == '1') && (v.n <= 256 || (v.m() + kPBJ - 1) / kPBJ < num_sms() / 4)) return false;
  const int N = tc_npad(l);
  if (!N) return false;
  if (!(v.P == 1 && v.si == 1 && v.ss >= v.n && v.ss % 4 == 0 && ((uintptr_t)v.base % 16) == 0)) return false;
  if (v.n > 1024) return false;
  return pair_encode_fn() != nullptr;
}

size_t pair_ypart_floats(const View& v, int l, int grid) {
  const int N = tc_npad(l), nt = (v.n + 255) / 256;
  return (size_t)(grid / 2) * N * nt * 256;
}

template <int N, int SA, bool H>
static cudaError_t pair_launch(const CUtensorMap& tq, const CUtensorMap& ta, const CUtensorMap& ta2, const PairArgs& a,
                               int grid, cudaStream_t st) {
  const size_t smem = 1024 + (size_t)(H ? kPRAH * 2 * kPTile : kPRA * kPTile) + (size_t)kPRQ * 2 * (N / 2) * 128 +
                      2 * (size_t)(kPBJ / (H ? 64 : 32)) * (N / 2) * 128 + (size_t)128 * (N / 2) * 4;
  cudaError_t e = cudaFuncSetAttribute(pair_power_kernel<N, SA, H>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kPThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  e = cudaLaunchKernelEx(&cfg, pair_power_kernel<N, SA, H>, tq, ta, ta2, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// One power step Y = M M^T Q on the pair engine from Q's hi/lo planes [2N][pld].
// Ypart[grid/2][N][nt*256]; returns the partial count and row pitch.
cudaError_t pair_power(const View& v, int l, const float* planes, int pld, float* Ypart, int grid, int* G_out,
                       int* rows_out, cudaStream_t st, const int* stop, float* shrink_out, int64_t Rprev,
                       int64_t nnext, int64_t ldnext, bool sketch, PairScale* ps) {
  // the fp16 two-plane power step: planes are fp16 [2N][pld] (pld a multiple of 8), scaled by 2^15
  const bool H = ps && ps->xmax_in && !sketch && !shrink_out;
  const int KS = H ? 64 : kPKS;
  const int N = tc_npad(l), nt = shrink_out ? 0 : (v.n + 255) / 256;
  const int64_t m = v.m();
  const int64_t nblk = (m + kPBJ - 1) / kPBJ;
  int pairs = std::max(1, grid / 2);
  pairs = (int)std::min<int64_t>(pairs, std::max<int64_t>(1, nblk));   // no idle pairs (zero partials)
  PairArgs a;
  a.n = v.n; a.m = m; a.nt = nt; a.nk1 = (v.n + KS - 1) / KS; a.nblk = nblk;
  a.Ypart = Ypart; a.stop = stop;
  a.lag = getenv("RTK_PAIR_LAG") ? atoi(getenv("RTK_PAIR_LAG")) : (H ? 1 : 8);   // stages (H: 64 rows each; lag 1 fastest of 0-4, DRAM 4.23 GB)
  a.dbg = getenv("RTK_PAIR_DBG") ? atoi(getenv("RTK_PAIR_DBG")) : 0;
  a.shrink = shrink_out ? 1 : 0;
  a.out = shrink_out;
  a.Rprev = Rprev; a.nnext = nnext; a.ldnext = ldnext;
  a.lk = l;
  a.sketch = sketch ? 1 : 0;
  a.op1pol = getenv("RTK_PAIR_OP1POL") ? atoi(getenv("RTK_PAIR_OP1POL")) : 0;
  a.xmax_in = H ? ps->xmax_in : nullptr;
  a.xmax_out = (ps && (sketch || shrink_out)) ? ps->xmax_out : nullptr;
  if (a.xmax_out) ps->wrote = true;
  a.cW = 0;
  while ((1ll << (2 * a.cW)) < (long long)v.n) ++a.cW;   // ceil(log2 sqrt(n))
  CUtensorMap tq, ta, ta2;
  memset(&tq, 0, sizeof(tq));
  memset(&ta, 0, sizeof(ta));
  memset(&ta2, 0, sizeof(ta2));
  const cuuint32_t es[2] = {1, 1};
  {   // op1 A tiles: box {32 rows, 128 columns}, SWIZZLE_128B ([128 j][32 i])
    cuuint64_t dims[2] = {(cuuint64_t)v.n, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)v.ss * 4};
    cuuint32_t box[2] = {32, 128};
    if (pair_encode_fn()(&ta, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(v.base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {   // op2 A tiles: box {128 rows, 32 columns}, no swizzle ([32 c][128 i])
    cuuint64_t dims[2] = {(cuuint64_t)v.n, (cuuint64_t)m};
    cuuint64_t strides[1] = {(cuuint64_t)v.ss * 4};
    cuuint32_t box[2] = {128, 32};
    if (pair_encode_fn()(&ta2, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(v.base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {   // Q planes [2N][pld]: box {32 rows i, N/2 columns c}, SWIZZLE_128B ([N/2 c][32 i]); the sketch's
      // Omega planes [2N][pld >= m] the same way with the unfolding's columns j in place of i.
      // H: fp16 planes, box {64 rows i, N/2 columns c} (128-B rows as well)
    cuuint64_t dims[2] = {(cuuint64_t)(sketch ? m : v.n), (cuuint64_t)(2 * N)};
    cuuint64_t strides[1] = {(cuuint64_t)pld * (H ? 2 : 4)};
    cuuint32_t box[2] = {(cuuint32_t)(H ? 64 : 32), (cuuint32_t)(N / 2)};
    if (H && (pld % 8)) return cudaErrorInvalidValue;
    if (pair_encode_fn()(&tq, H ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                         const_cast<float*>(planes), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  *G_out = pairs;
  *rows_out = nt * 256;
#if RTK_PAIR_PROF
  {   // role timers of the previous launch (pair 0), then reset
    static int calls = 0;
    unsigned long long h[2][32];
    if (calls++ > 0 && cudaMemcpyFromSymbol(h, g_pair_prof, sizeof(h)) == cudaSuccess)
      for (int r = 0; r < 2; ++r)
        fprintf(stderr,
                "[pair prof cta%d] mma total %llu wait a_full(op1) %llu q_full %llu a_full(op2) %llu p_full %llu "
                "w_empty %llu | prod total %llu r_full %llu a_empty %llu st %llu lds+split %llu arrive %llu walk %llu | tma r_empty %llu | epi total %llu "
                "w_full %llu exch %llu p_empty %llu tmem_ld %llu planes %llu | q q_empty %llu\n",
                r, h[r][0], h[r][1], h[r][2], h[r][3], h[r][4], h[r][5], h[r][8], h[r][9], h[r][10], h[r][11], h[r][12], h[r][13], h[r][14], h[r][17],
                h[r][20], h[r][21], h[r][22], h[r][23], h[r][25], h[r][26], h[r][24]);
    unsigned long long z[2][32] = {};
    cudaMemcpyToSymbol(g_pair_prof, z, sizeof(z));
  }
#endif
  const char* se = getenv("RTK_PAIR_SA");
  const bool sa3 = se && se[0] == '3';   // SA = 3 needs op1(b) to start after W(b-1) was drained
  if (H) {
    switch (N) {
      case 16: return pair_launch<16, 2, true>(tq, ta, ta2, a, 2 * pairs, st);
      case 32: return pair_launch<32, 2, true>(tq, ta, ta2, a, 2 * pairs, st);
      case 48: return pair_launch<48, 2, true>(tq, ta, ta2, a, 2 * pairs, st);
      default: return sa3 ? pair_launch<64, 3, true>(tq, ta, ta2, a, 2 * pairs, st)
                          : pair_launch<64, 2, true>(tq, ta, ta2, a, 2 * pairs, st);
    }
  }
  switch (N) {
    case 16: return sa3 ? pair_launch<16, 3, false>(tq, ta, ta2, a, 2 * pairs, st) : pair_launch<16, 2, false>(tq, ta, ta2, a, 2 * pairs, st);
    case 32: return sa3 ? pair_launch<32, 3, false>(tq, ta, ta2, a, 2 * pairs, st) : pair_launch<32, 2, false>(tq, ta, ta2, a, 2 * pairs, st);
    case 48: return sa3 ? pair_launch<48, 3, false>(tq, ta, ta2, a, 2 * pairs, st) : pair_launch<48, 2, false>(tq, ta, ta2, a, 2 * pairs, st);
    default: return sa3 ? pair_launch<64, 3, false>(tq, ta, ta2, a, 2 * pairs, st) : pair_launch<64, 2, false>(tq, ta, ta2, a, 2 * pairs, st);
  }
}

}  // namespace rtk
