// rtk_api.cu -- C ABI (include/rtucker.h): validation, planning, workspace carving and
// the per-mode launch sequence of Alg. 3 / Alg. 4.
//
// Host control only: every arithmetic step runs in the kernels of rtk_tile.cu /
// rtk_small.cu.  Nothing is copied back to the host during a solve (alpha lives in
// device memory), so the sequence is stream-ordered and CUDA-graph capturable.
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <mutex>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/rtucker.h"
#include "rtk_internal.h"

namespace rtk {
namespace {

thread_local std::string g_err;

// smallest unfolding width whose sketch runs on the fused engine (Omega planes precomputed) rather
// than tc_op2 (Omega generated in shared memory); RTK_FUSED_SKETCH_MIN overrides (measurement)
static int64_t fused_sketch_min() {   // read per call so that tests can switch it
  const char* e = getenv("RTK_FUSED_SKETCH_MIN");
  return e ? atoll(e) : 100000;   // measured: C5 mode 2 (m = 5e4) faster on tc_op2, C3 mode 1 (1.6e5) fused
}

// ---- launch accounting / optional event profile (rtk_profile_begin/end) ----
struct ProfRec {
  int kind, mode;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;
std::atomic<bool> g_prof_on{false};
std::atomic<long long> g_launches{0};

struct ProfScope {
  cudaEvent_t a = nullptr, b = nullptr;
  int kind, mode;
  cudaStream_t st;
  ProfScope(int kind_, int mode_, cudaStream_t st_) : kind(kind_), mode(mode_), st(st_) {
    if (g_prof_on.load()) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~ProfScope() {
    if (a) {
      cudaEventRecord(b, st);
      std::lock_guard<std::mutex> lk(g_prof_mu);
      g_prof.push_back({kind, mode, a, b});
    }
  }
};

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

// Sticky RTK_ERR_NUMERIC (include/rtucker.h): every solve ends with a one-thread kernel that sets a
// per-device flag in mapped pinned host memory when any mode's status word reports a numeric
// failure.  A call without a report cannot wait for its own result (it is asynchronous), so the
// NEXT call on that device returns RTK_ERR_NUMERIC (and clears the flag) once the failing solve
// has executed; a call with a report returns it directly.
__global__ void numeric_flag_kernel(const int* status, int d, int* flag) {
  int bad = 0;
  for (int k = 0; k < d; ++k) bad |= (status[4 * k] != 0);
  if (bad) *(volatile int*)flag = 1;
}

int* numeric_flag_host(int dev) {   // nullptr if the pinned allocation failed (check then skipped)
  static int* flags[64] = {};
  static std::mutex mu;
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!flags[dev]) {
    int* h = nullptr;
    if (cudaHostAlloc((void**)&h, sizeof(int), cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    *h = 0;
    flags[dev] = h;
  }
  return flags[dev];
}

constexpr int kLMaxApi = 96;
constexpr int kNMax = 4096;

size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

int64_t pad4(int64_t n) { return (n + 3) / 4 * 4; }
int64_t pad8(int64_t n) { return (n + 7) / 8 * 8; }

struct Problem {
  int d = 0;
  std::vector<int64_t> dims;
  std::vector<int> ranks;
  int p = 0, q = 0;
  bool seq = true;
  double pve = 0.0;   // > 0: Alg. B.1 tolerance, q is q_max
  bool a2 = false;    // Alg. A.2: each mode keeps all l_k columns, then ST-HOSVD of the l-core
  int omega = 0;      // sketch type: 0 RTK-GAUSS-2, 1 uniform, 2 KR-Gaussian, 3 KR-uniform
  std::vector<int> keep;   // columns kept by mode k's shrink: r_k, or l_k = r_k + p (A.2)
  // multi-GPU last-mode shard: dims[d-1] is this rank's slab, full_last the whole
  // extent, sh_begin the slab's first index; modes < d-1 all-reduce Y after every streaming pass
  int64_t full_last = 0, sh_begin = 0;
  bool sh_root = true;                 // the rank that applies -alpha Q (once) before the all-reduce
  rtk_allreduce_fn ar = nullptr;
  void* ar_ctx = nullptr;
};

void set_keep(Problem& P) {
  P.keep.resize(P.d);
  for (int k = 0; k < P.d; ++k) P.keep[k] = P.ranks[k] + (P.a2 ? P.p : 0);
}

// extents of the tensor whose mode-k unfolding mode k factors (T: A; ST: the shrunk G)
std::vector<int64_t> cur_dims(const Problem& P, int k) {
  std::vector<int64_t> e(P.dims);
  if (P.seq)
    for (int j = 0; j < k; ++j) e[j] = P.keep[j];
  return e;
}

// the same with the last mode at its full (unsharded) extent: Omega_k's row structure
std::vector<int64_t> cur_dims_full(const Problem& P, int k) {
  std::vector<int64_t> e = cur_dims(P, k);
  if (P.full_last) e[P.d - 1] = P.full_last;
  return e;
}

// m_k: columns of the matrix mode k factors (PAPER.md:257 vs :300)
int64_t mode_cols(const Problem& P, int k) {
  int64_t m = 1;
  for (int j = 0; j < P.d; ++j) {
    if (j == k) continue;
    m *= (P.seq && j < k) ? P.keep[j] : P.dims[j];
  }
  return m;
}

int validate(const Problem& P) {
  if (P.d < 2 || P.d > 8) return fail(RTK_ERR_ARG, "d must be in [2, 8]");
  for (int k = 0; k < P.d; ++k) {
    if (P.dims[k] < 1) return fail(RTK_ERR_ARG, "dims[k] must be >= 1");
    if (P.ranks[k] < 1 || P.ranks[k] > P.dims[k]) return fail(RTK_ERR_ARG, "ranks[k] must be in [1, n_k]");
  }
  if (P.p < 0) return fail(RTK_ERR_ARG, "oversampling p must be >= 0");
  if (P.q < 1) return fail(RTK_ERR_ARG, "power parameter q must be >= 1 (PAPER.md:253)");
  for (int k = 0; k < P.d; ++k) {
    const int64_t l = (int64_t)P.ranks[k] + P.p;
    const int64_t m = mode_cols(P, k);
    if (l > P.dims[k] || l > m)
      return fail(RTK_ERR_SHAPE, "l_k = r_k + p exceeds min(n_k, m_k) in mode " + std::to_string(k + 1) +
                                     " (PAPER.md:272)");
    if (l > kLMaxApi) return fail(RTK_ERR_SHAPE, "l_k > 96 is not supported by the one-CTA small solves");
    if (P.a2 && l > kSolveLMax) return fail(RTK_ERR_SHAPE, "Alg. A.2 needs l_k = r_k + p <= 64");
    if (P.dims[k] > kNMax) return fail(RTK_ERR_SHAPE, "n_k > 4096 is not supported by the tile kernels");
  }
  return RTK_OK;
}

// Views: the range-finder matrix of mode k, and the shrink input of mode k.
View range_view(const Problem& P, int k, const float* A, const float* buf) {
  View v;
  v.n = (int)P.dims[k];
  if (!P.seq || k == 0) {
    int64_t Pk = 1, Sk = 1;
    for (int j = 0; j < k; ++j) Pk *= P.dims[j];
    for (int j = k + 1; j < P.d; ++j) Sk *= P.dims[j];
    v.base = A;
    if (Pk == 1) {  // column-major n_k x m
      v.P = 1; v.S = Sk; v.sp = 1; v.si = 1; v.ss = P.dims[k];
    } else {
      v.P = Pk; v.S = Sk; v.sp = 1; v.si = Pk; v.ss = Pk * P.dims[k];
    }
  } else {
    v.base = buf;
    v.P = 1; v.S = mode_cols(P, k); v.sp = 1; v.si = 1; v.ss = pad4(P.dims[k]);
  }
  return v;
}

// Shrink of mode k reads the (k)-unfolding stored contiguously (k == 0: A itself).
View shrink_view(const Problem& P, int k, const float* A, const float* buf) {
  View v;
  v.n = (int)P.dims[k];
  v.P = 1;
  int64_t m = 1;
  for (int j = 0; j < P.d; ++j)
    if (j != k) m *= (j < k) ? P.keep[j] : P.dims[j];
  v.S = m;
  v.sp = 1; v.si = 1;
  if (k == 0) { v.base = A; v.ss = P.dims[0]; }
  else { v.base = buf; v.ss = pad4(P.dims[k]); }
  return v;
}

// the fused single-pass engine applies (RTK_FUSED=0: off, measurement)
bool fused_ok(const View& v, int l) {
  const char* fz = getenv("RTK_FUSED");
  if (fz && fz[0] == '0') return false;
  const char* pe = getenv("RTK_PATH");
  if (pe && std::string(pe) == "ffma") return false;
  return fused_supported(v, l);
}

struct Layout {
  size_t planes = 0, wbuf = 0;
  int64_t ldw = 0;
  std::vector<char> tc_range, tc_shrink;
  size_t ypart = 0, y = 0, q1 = 0, qd = 0, qs = 0, gpart = 0, T = 0, lam = 0;
  size_t alpha = 0, trace = 0, sigma = 0, status = 0, sighat = 0, shr0 = 0, shr1 = 0, total = 0;
  size_t g2part = 0, gsum = 0, amax = 0, lamx = 0, gbar = 0;
  size_t xmax = 0;   // [8] floats: max|M| of each mode's unfolding (the fp16 pair engine's scale)
  size_t a2q = 0, a2b = 0, a2g0 = 0, a2g1 = 0, a2gram = 0, a2v = 0;   // Alg. A.2 only
  size_t om = 0, omtab = 0;                                         // Appendix D sketches only
  size_t mode_size = 0;   // bytes of one mode's scratch region (T-HOSVD: one region per mode)
  int nregions = 1;
  size_t shr_elems = 0;
  std::vector<TilePlan> sk, pw, sh;
};

Layout plan(const Problem& P, int nsm, const float* A, int path) {
  Layout L;
  size_t ypart = 0, nl = 0, qsz = 0, gp = 0, ll = 0, lmax = 0, planes = 0, wbuf = 0;
  int wN = 0;   // largest padded N over the tcgen05 range modes
  L.sk.resize(P.d); L.pw.resize(P.d); L.sh.resize(P.d);
  L.tc_range.assign(P.d, 0);
  L.tc_shrink.assign(P.d, 0);
  size_t shr = 0;
  int64_t ldw = 4;
  for (int k = 0; k < P.d; ++k) {
    const int l = P.ranks[k] + P.p;
    View rv = range_view(P, k, nullptr, nullptr);
    // tcgen05 eligibility is a property of the view's shape / stride (alignment of the real
    // pointers is re-checked at launch time; A's base decides for the views that read it)
    View rvp = rv;
    rvp.base = (!P.seq || k == 0) ? A : (const float*)nullptr;
    View svp = shrink_view(P, k, nullptr, nullptr);
    svp.base = k == 0 ? A : (const float*)nullptr;
    if (path != 1) {
      // contiguous views: tcgen05 (fused or two-kernel); Alg. 3's strided views: the fused engine only
      L.tc_range[k] = (rvp.P > 1 ? (l <= kSolveLMax && fused_ok(rvp, l)) : tc_supported(rvp, l)) ? 1 : 0;
      L.tc_shrink[k] = tc_supported(svp, P.keep[k]) ? 1 : 0;
    }
    if (L.tc_range[k]) {
      const int N = tc_npad(l), nit = (rv.n + 127) / 128;
      ypart = std::max(ypart, (size_t)nsm * N * nit * 128);
      planes = std::max(planes, (size_t)2 * N * pad4(rv.n));
      ldw = std::max<int64_t>(ldw, pad4(rv.m()));
      wN = std::max(wN, N);
    }
    if (L.tc_shrink[k]) planes = std::max(planes, (size_t)2 * tc_npad(P.keep[k]) * pad4(rv.n));
    L.sk[k] = plan_tile(rv, l, OP_SKETCH, nsm);
    L.pw[k] = plan_tile(rv, l, OP_POWER, nsm);
    View sv = shrink_view(P, k, nullptr, nullptr);
    L.sh[k] = plan_tile(sv, P.keep[k], OP_SHRINK, nsm);
    for (const TilePlan* tp : {&L.sk[k], &L.pw[k]})
      ypart = std::max(ypart, (size_t)tp->G * tp->ltot() * tp->n_rows());
    const size_t n = (size_t)P.dims[k];
    nl = std::max(nl, n * l);
    qsz = std::max(qsz, n * l);
    gp = std::max(gp, (size_t)((n + 63) / 64) * l * (l + 1) / 2);
    if (l <= kSolveLMax) gp = std::max(gp, solve_gpart_doubles((int)n, l));
    ll = std::max(ll, (size_t)l * l);
    lmax = std::max(lmax, (size_t)l);
    if (k + 1 < P.d) {
      // output of shrink k: (r_1..r_k) x pad4(n_{k+1}) x (n_{k+2}..n_d)
      size_t e = (size_t)pad4(P.dims[k + 1]);
      for (int j = 0; j <= k; ++j) e *= P.keep[j];
      for (int j = k + 2; j < P.d; ++j) e *= P.dims[j];
      shr = std::max(shr, e);
    }
  }
  // W (two-kernel path: 2N rows of W) and the fused sketch's Omega planes (2N rows) are both
  // addressed with the common leading dimension ldw = max pad4(m_k): size for the largest N
  // times that ldw, not per mode (a mode with a larger N but a smaller m would overrun)
  wbuf = (size_t)2 * wN * (size_t)ldw;
  L.shr_elems = shr;
  size_t off = 0;
  auto take = [&](size_t bytes) { const size_t o = off; off += align_up(std::max<size_t>(bytes, 16)); return o; };
  L.ldw = ldw;
  // global region: per-mode report slots, the shrink chain buffers, Alg. A.2's l-core stage
  L.alpha = take(P.d * 8);
  L.trace = take((size_t)P.d * P.q * 8);
  L.sigma = take((size_t)P.d * 128 * 8);
  L.status = take((size_t)P.d * 4 * 4);
  L.xmax = take(8 * 4);
  L.shr0 = take(shr * 4);
  L.shr1 = take(shr * 4);
  if (P.a2) {
    size_t qa = 0, lt = 1;
    for (int k = 0; k < P.d; ++k) { qa += (size_t)P.dims[k] * P.keep[k]; lt *= (size_t)P.keep[k]; }
    L.a2q = take(qa * 8);
    L.a2b = take(lt * 4);
    L.a2g0 = take(lt * 8);
    L.a2g1 = take(lt * 8);
    L.a2gram = take((size_t)kSolveLMax * kSolveLMax * 8);
    L.a2v = take((size_t)kSolveLMax * kSolveLMax * 8);
  }
  // mode region (offsets of region 0; T-HOSVD gives every mode its own copy so that the modes,
  // which are independent in Alg. 3, run concurrently on their own streams)
  const size_t mode0 = off;
  L.planes = take(planes * 4);
  L.wbuf = take(wbuf * 4);
  L.ypart = take(ypart * 4);
  L.y = take(nl * 8);
  L.q1 = take(nl * 8);
  L.qd = take(nl * 8);
  L.qs = take(qsz * 4);
  L.gpart = take(gp * 8);
  L.T = take(ll * 8);
  L.lam = take(lmax * 8);
  L.sighat = take(lmax * 8);
  L.g2part = take((size_t)32 * kSolveLMax * (kSolveLMax + 1) / 2 * 8);   // <= 32 step-kernel CTAs
  L.gsum = take((size_t)kSolveLMax * (kSolveLMax + 1) / 2 * 8);
  L.amax = take((size_t)32 * 3 * kSolveLMax * 8);   // (max, index) pairs + the tie-pivot indices, <= 32 CTAs
  L.lamx = take((size_t)kSolveLMax * 8);            // eigenvalues shared across the step cluster
  L.gbar = take(16);                                 // the step kernel's grid barrier
  if (P.omega || P.full_last) {   // materialised Omega_k (Appendix D types; every type on a shard)
    size_t oms = 0, tabs = 0;
    for (int k = 0; k < P.d; ++k) {
      const int l = P.ranks[k] + P.p;
      oms = std::max(oms, (size_t)mode_cols(P, k) * l);
      const std::vector<int64_t> e = cur_dims_full(P, k);
      tabs = std::max(tabs, sketch_tab_floats(e.data(), P.d, k + 1, l));
    }
    L.om = take(oms * 4);
    L.omtab = take(tabs * 4);
  }
  L.mode_size = off - mode0;
  L.nregions = P.seq ? 1 : P.d;
  off += (size_t)(L.nregions - 1) * L.mode_size;
  L.total = off;
  return L;
}

// Side stream + events (per device) for the deferred shift update (alpha_kernel, rtk_solve.cu):
// it overlaps the next power step's streaming kernels, which then leave one SM free.
struct Side {
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_step = nullptr, ev_alpha = nullptr;
};
// The pools are per host thread (thread_local): concurrent rtk_solve calls from different host
// threads never share fork/join events or side streams.
cudaError_t side_streams(Side** out, int idx = 0) {   // idx: one set per concurrently running mode
  static thread_local Side S[64][8];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64 || idx < 0 || idx >= 8) return cudaErrorInvalidDevice;
  Side& s = S[dev][idx];
  if (!s.aux) {
    e = cudaStreamCreateWithFlags(&s.aux, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.ev_step, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.ev_alpha, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  *out = &s;
  return cudaSuccess;
}

// plan() is pure host work (tile-plan search per mode); repeated solves of one shape reuse it.
// The key holds every input plan() reads, including its environment overrides.
const Layout& plan_cached(const Problem& P, int nsm, const float* A, int path) {
  static thread_local std::vector<std::pair<std::string, Layout>> cache;
  std::string key;
  auto add = [&](long long x) { key += std::to_string(x); key += ','; };
  add(P.d); add(P.p); add(P.q); add(P.seq); add(P.a2); add(P.omega); add(nsm); add(path); add(P.full_last);
  add((long long)((uintptr_t)A % 16));
  for (int k = 0; k < P.d; ++k) { add(P.dims[k]); add(P.ranks[k]); add(P.keep[k]); }
  for (const char* ev : {"RTK_PATH", "RTK_PLAN", "RTK_PLAN_SKETCH", "RTK_PLAN_POWER", "RTK_PLAN_SHRINK", "RTK_FUSED",
                         "RTK_FUSED_STRIDED"}) {
    const char* v = getenv(ev);
    key += v ? v : "-";
    key += ';';
  }
  for (auto& kv : cache)
    if (kv.first == key) return kv.second;
  if (cache.size() >= 16) cache.erase(cache.begin());
  cache.emplace_back(key, plan(P, nsm, A, path));
  return cache.back().second;
}

// Per-device streams + fork/join events for Alg. 3's concurrent modes.
struct ModeStreams {
  cudaStream_t s[8] = {};
  cudaEvent_t fork = nullptr, join[8] = {};
};
cudaError_t mode_streams(ModeStreams** out) {
  static thread_local ModeStreams M[64];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  ModeStreams& m = M[dev];
  if (!m.fork) {
    for (int i = 0; i < 8 && e == cudaSuccess; ++i) {
      e = cudaStreamCreateWithFlags(&m.s[i], cudaStreamNonBlocking);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m.join[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m.fork, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  *out = &m;
  return cudaSuccess;
}

#define RTK_CK(x)                                                                          \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) return fail(RTK_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Alg. 3/4 lines 3-12 for one mode (mode index k, 0-based); writes U_k.
// max|M| bookkeeping for the fp16 pair power step (rtk_fused2.cu): xmax[k] holds max|M| of mode k's
// unfolding once a pair sketch of mode k or the pair shrink of mode k-1 has written it (ready[k]).
struct XState {
  float* xmax = nullptr;
  char ready[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

static bool pair_f16_enabled() {
  const char* e = getenv("RTK_PAIR_F16");
  return !(e && e[0] == '0');
}

int run_mode(const Problem& P, const Layout& L, char* ws, int k, const View& v, uint64_t seed,
             bool shift, float* Uk, cudaStream_t st, XState* xs = nullptr) {
  const int n = v.n, r = P.ranks[k], l = r + P.p;
  char* mw = ws + (P.seq ? 0 : (size_t)k * L.mode_size);   // this mode's scratch region
  ModeBufs B;
  B.n = n; B.l = l; B.r = P.a2 ? l : r;   // A.2: the step kernel pins all l columns of Q
  B.Ypart = (float*)(mw + L.ypart);
  B.Y = (double*)(mw + L.y);
  B.Q1 = (double*)(mw + L.q1);
  B.Qd = (double*)(mw + L.qd);
  B.Qs = (float*)(mw + L.qs);
  B.gpart = (double*)(mw + L.gpart);
  B.nblk = (n + 63) / 64;   // kGB-row Gram blocks (rtk_small.cu)
  B.T = (double*)(mw + L.T);
  B.lam = (double*)(mw + L.lam);
  B.alpha = (double*)(ws + L.alpha) + k;
  B.trace = (double*)(ws + L.trace) + (size_t)k * P.q;
  B.sigma = (double*)(ws + L.sigma) + (size_t)k * 128;
  B.status = (int*)(ws + L.status) + 4 * k;
  B.sighat = (double*)(mw + L.sighat);
  B.g2part = (double*)(mw + L.g2part);
  B.gsum = (double*)(mw + L.gsum);
  B.amax = (double*)(mw + L.amax);
  B.lamx = (double*)(mw + L.lamx);
  B.gbar = (unsigned int*)(mw + L.gbar);
  const bool fast = l <= kSolveLMax;   // cluster small solver (rtk_solve.cu)
  RTK_CK(cudaMemsetAsync(B.alpha, 0, sizeof(double), st));   // alpha = 0 (line 5)
  RTK_CK(cudaMemsetAsync(B.gbar, 0, 16, st));                 // step-kernel grid barrier
  const uint32_t mode1 = (uint32_t)(k + 1);
  const bool strided = v.P > 1;
  const bool tc = L.tc_range[k] && (strided ? (fast && fused_ok(v, l)) : tc_supported(v, l));
  Side* side = nullptr;
  const bool fused = tc && fast && fused_ok(v, l);   // single-pass power step (strided views: always)
  const bool pve = P.pve > 0.0;   // Alg. B.1: the step kernel decides the stop, alpha inline
  const int* stop = pve ? B.status + 3 : nullptr;
  if (pve) RTK_CK(cudaMemsetAsync(B.sighat, 0, (size_t)l * sizeof(double), st));   // sigmahat = 0
  const bool defer = fast && tc && P.q > 1 && !pve;   // deferred shift updates on the side stream
  if (defer) RTK_CK(side_streams(&side, k));
  bool pending = false;                       // an alpha_kernel is in flight on side->aux
  // a shard's mode k < d-1 factors the column range [j0, j0 + m) of the full unfolding (i_d is the
  // slowest column index): its partial Y sums to the full one after the all-reduce
  const bool shard = P.full_last && k < P.d - 1;
  const float* om = nullptr;   // Appendix D sketch types (and shards): Omega_k materialised once per mode
  if (P.omega || shard) {
    const std::vector<int64_t> e = cur_dims_full(P, k);
    int64_t j0 = 0;
    if (shard) {
      int64_t stride = 1;   // column stride of i_d in the mode-k unfolding
      for (int j = 0; j < P.d - 1; ++j)
        if (j != k) stride *= e[j];
      j0 = stride * P.sh_begin;
    }
    ProfScope ps(0, k, st);
    om = (const float*)(mw + L.om);
    if (P.omega)
      RTK_CK(sketch_materialize(P.omega, seed, k + 1, e.data(), P.d, j0, v.m(), l, (float*)(mw + L.omtab),
                                (float*)(mw + L.om), st));
    else
      RTK_CK(launch_omega(seed, (uint32_t)(k + 1), j0, v.m(), l, (float*)(mw + L.om), st));
    g_launches += 1 + (P.omega >= 2 ? P.d - 1 : 0);
  }
  // the power steps run on the fp16 pair engine when max|M| of this unfolding is known (decided
  // after the sketch, which may provide it)
  const bool h16c = xs && fast && fused && pair_supported(v, l) && pair_f16_enabled();
  bool h16 = false;
  for (int step = 0; step <= P.q; ++step) {
    const TilePlan& tp = step == 0 ? L.sk[k] : L.pw[k];
    if (tc) {
      ProfScope ps(step == 0 ? 0 : 1, k, st);
      float* planes = (float*)(mw + L.planes);
      float* W = (float*)(mw + L.wbuf);
      const int G = pending ? num_sms() - 1 : num_sms();   // leave the alpha_kernel its SM
      // sketch on the fused engine only for long unfoldings (Omega-plane generation has a fixed
      // cost; tc_op2 generates Omega in shared memory and is faster for small m)
      if (fused && (step > 0 || strided || v.m() >= fused_sketch_min())) {   // sketch: Omega planes in the W buffer (ld = ldw >= m)
        int Gf = 0, rows = 0;
        const bool sk = step == 0;
        PairScale ps;
        if (h16c) {
          if (sk) ps.xmax_out = xs->xmax + k;
          else ps.xmax_in = h16 ? xs->xmax + k : nullptr;
        }
        RTK_CK(fused_power(v, l, sk ? W : planes, sk ? (int)L.ldw : (h16 ? (int)pad8(n) : (int)pad4(n)), sk, seed,
                           mode1, B.Ypart, pending ? num_sms() - fused_cluster(n) : num_sms(), &Gf, &rows, st,
                           nullptr, 1, 1, 1, sk ? nullptr : stop, om, &ps));
        if (ps.wrote) xs->ready[k] = 1;
        g_launches += (sk && !fused_sketch_gen(om)) ? 1 : 0;   // omega_planes_kernel
        g_launches += 1;
        B.G = Gf; B.ltot = tc_npad(l); B.n_rows = rows;
      } else {
      const int G2 = tc_op2_grid(v, G);
      if (step == 0) {   // (records max|M| for the fp16 pair power steps, like the pair sketch)
        RTK_CK(tc_op2(v, l, nullptr, 0, true, seed, mode1, B.Ypart, G2, st, om, h16c ? xs->xmax + k : nullptr));
        if (h16c) xs->ready[k] = 1;
        g_launches += 1;
      } else {
        if (!fast) RTK_CK(tc_split(B.Qd, nullptr, n, l, planes, st));   // else: written by step_kernel
        RTK_CK(tc_op1(v, l, planes, W, L.ldw, false, nullptr, 1, 1, 1, st, G));
        RTK_CK(tc_op2(v, l, W, L.ldw, false, 0, 0, B.Ypart, G2, st));
        g_launches += 3;
      }
      B.G = G2; B.ltot = tc_npad(l); B.n_rows = ((n + 127) / 128) * 128;
      }
    } else {
    TileLaunch T;
    T.v = v;
    T.op = step == 0 ? OP_SKETCH : OP_POWER;
    T.tp = tp;
    T.l = l;
    T.Q = B.Qs;
    T.qld = n;
    T.Ypart = B.Ypart;
    T.seed = seed;
    T.om = om;
    T.mode = mode1;
    {
      ProfScope ps(step == 0 ? 0 : 1, k, st);
      RTK_CK(launch_tile(T, st));
      g_launches += 1;
    }
    B.G = tp.G; B.ltot = tp.ltot(); B.n_rows = tp.n_rows();
    }
    if (step == 0) h16 = h16c && xs->ready[k];   // the planes the step kernels write from here on
    if (fast) {
      ProfScope ps(3, k, st);
      float* planes = tc ? (float*)(mw + L.planes) : nullptr;
      if (pending) {   // the previous step's alpha is needed by this reduce (Y = M M^T Q - alpha Q)
        RTK_CK(cudaStreamWaitEvent(st, side->ev_alpha, 0));
        pending = false;
      }
      if (shard) {   // Y = sum over ranks of the partial Y (-alpha Q applied once, by the root)
        RTK_CK(launch_reduce_gram2(B, step > 0 && P.sh_root, st, nullptr, 1));
        if (P.ar((void*)B.Y, (int64_t)B.n * B.l, 1, (void*)st, P.ar_ctx) != 0)
          return fail(RTK_ERR_CUDA, "all-reduce callback failed (mode " + std::to_string(k + 1) + ")");
        RTK_CK(launch_reduce_gram2(B, false, st, nullptr, 2));
        g_launches += 1;
      } else {
        RTK_CK(launch_reduce_gram2(B, step > 0, st, step > 0 ? stop : nullptr));
      }
      const bool dstep = defer && step > 0 && step < P.q;
      if (dstep) {   // the shift update reads the reduce's Gram partials: it runs beside step_kernel
        RTK_CK(cudaEventRecord(side->ev_step, st));
        RTK_CK(cudaStreamWaitEvent(side->aux, side->ev_step, 0));
        RTK_CK(launch_alpha(B, step, shift, side->aux));
        RTK_CK(cudaEventRecord(side->ev_alpha, side->aux));
        pending = true;
        g_launches += 1;
      }
      // B.1 may stop at any power step: U_k is written by the step that stops (or the last)
      // A.2: the pinned fp32 basis replaces the shadow Qs (the shrink's matrix), Qd pinned in place
      float* uout = P.a2 ? (float*)(mw + L.qs) : Uk;
      RTK_CK(launch_step(B, step, P.q, shift, (step == P.q || (pve && step > 0)) ? uout : nullptr, seed, mode1,
                         planes, tc_npad(l), h16 ? (int)pad8(n) : (int)pad4(n), dstep, pve ? P.pve : 0.0, st, P.a2,
                         h16));
      g_launches += 2;
    } else {
      ProfScope ps(3, k, st);
      RTK_CK(launch_reduce_gram(B, step > 0, st));
      RTK_CK(launch_eig(B, step, P.q, shift, 0.0, st));
      RTK_CK(launch_apply(B, seed, mode1, step, st));
      RTK_CK(launch_chol(B, st));
      RTK_CK(launch_apply2(B, st));
      g_launches += 6;
    }
  }
  if (!fast) {
    RTK_CK(launch_final_u(B, Uk, st));
    g_launches += 1;
  }
  return RTK_OK;
}

// G x_k U_k^T written as the next unfolding (or the canonical core after mode d).
int run_shrink(const Problem& P, const Layout& L, char* ws, int k, const View& v, const float* Uk, float* out,
               cudaStream_t st, XState* xs = nullptr) {
  TileLaunch T;
  T.v = v;
  T.op = OP_SHRINK;
  T.tp = L.sh[k];
  T.l = P.keep[k];
  T.Q = Uk;
  T.qld = (int)P.dims[k];
  int64_t Rprev = 1;
  for (int j = 0; j < k; ++j) Rprev *= P.keep[j];
  T.Rprev = Rprev;
  if (k + 1 < P.d) { T.nnext = P.dims[k + 1]; T.ldnext = pad4(P.dims[k + 1]); }
  else { T.nnext = 1; T.ldnext = 1; }
  T.out = out;
  ProfScope ps(2, k, st);
  const char* fz = getenv("RTK_FUSED");
  const int kk = P.keep[k];
  if (L.tc_shrink[k] && tc_supported(v, kk) && !(fz && fz[0] == '0') && fused_supported(v, kk)) {
    float* planes = (float*)(ws + L.planes);
    RTK_CK(tc_split(nullptr, Uk, v.n, kk, planes, st));
    int Gf = 0, rows = 0;
    PairScale ps;   // the pair shrink records max|M| of the next unfolding it writes
    if (xs && k + 1 < P.d && pair_f16_enabled()) ps.xmax_out = xs->xmax + k + 1;
    RTK_CK(fused_power(v, kk, planes, (int)pad4(v.n), false, 0, 0, nullptr, num_sms(), &Gf, &rows, st, out,
                       T.Rprev, T.nnext, T.ldnext, nullptr, nullptr, &ps));
    if (ps.wrote) xs->ready[k + 1] = 1;
    g_launches += 2;
    return RTK_OK;
  }
  if (L.tc_shrink[k] && tc_supported(v, kk)) {
    float* planes = (float*)(ws + L.planes);
    RTK_CK(tc_split(nullptr, Uk, v.n, kk, planes, st));
    RTK_CK(tc_op1(v, kk, planes, nullptr, 0, true, out, T.Rprev, T.nnext, T.ldnext, st));
    g_launches += 2;
    return RTK_OK;
  }
  RTK_CK(launch_tile(T, st));
  g_launches += 1;
  return RTK_OK;
}

int solve(const rtk_options& opt, const float* A, const int64_t* dims, int32_t d, const int32_t* ranks,
          int32_t p, int32_t q, uint64_t seed, float* const* U, float* core, void* ws_in,
          size_t ws_bytes, void* stream, rtk_report* rep) {
  if (!A || !dims || !ranks || !U || !core) return fail(RTK_ERR_ARG, "NULL pointer argument");
  if (d < 2 || d > 8) return fail(RTK_ERR_ARG, "d must be in [2, 8]");
  Problem P;
  P.d = d; P.p = p; P.q = q; P.seq = opt.sequential != 0;
  P.dims.assign(dims, dims + d);
  P.ranks.assign(ranks, ranks + d);
  if (opt.variant < 0 || opt.variant > 1) return fail(RTK_ERR_ARG, "variant must be 0 (Alg. 2/3/4) or 1 (Alg. A.2)");
  if (opt.omega < 0 || opt.omega > 3)
    return fail(RTK_ERR_ARG, "omega must be 0 (Gaussian), 1 (uniform), 2 (KR-Gaussian) or 3 (KR-uniform)");
  P.omega = opt.omega;
  P.a2 = opt.variant == 1;
  if (P.a2 && !P.seq) return fail(RTK_ERR_ARG, "Alg. A.2 is the sequential (ST-HOSVD) variant: set sequential = 1");
  if (P.a2 && opt.pve_tol > 0.0) return fail(RTK_ERR_ARG, "PVE (Alg. B.1) is stated for Alg. 4, not Alg. A.2");
  set_keep(P);
  for (int k = 0; k < d; ++k)
    if (!U[k]) return fail(RTK_ERR_ARG, "NULL U[k]");
  int rc = validate(P);
  if (rc) return rc;
  if ((uintptr_t)A % 4) return fail(RTK_ERR_ALIGN, "A must be 4-byte aligned");
  if (opt.pve_tol > 0.0) {   // Alg. B.1 is stated for Alg. 4
    if (!P.seq) return fail(RTK_ERR_ARG, "PVE (Alg. B.1) applies to the sequential algorithm (Alg. 4) only");
    if (p < 1) return fail(RTK_ERR_ARG, "PVE (Alg. B.1) needs p >= 1 (it compares against sigma_{r+1})");
    if (q < 1) return fail(RTK_ERR_ARG, "PVE (Alg. B.1) needs q_max >= 1");
    for (int k = 0; k < d; ++k)
      if (ranks[k] + p > kSolveLMax) return fail(RTK_ERR_ARG, "PVE (Alg. B.1) needs r_k + p <= 64");
    P.pve = opt.pve_tol;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (opt.path < 0 || opt.path > 2) return fail(RTK_ERR_ARG, "path must be 0 (auto), 1 (FFMA) or 2 (tcgen05)");
  int dev = 0;
  RTK_CK(cudaGetDevice(&dev));
  int* nflag = numeric_flag_host(dev);
  if (nflag && *(volatile int*)nflag) {
    *(volatile int*)nflag = 0;
    return fail(RTK_ERR_NUMERIC, "an earlier solve on this device hit a numeric failure (non-finite iterate or "
                                 "unrepairable Cholesky breakdown); its outputs are unreliable");
  }
  const Layout L = plan_cached(P, num_sms(), A, opt.path);
  if (opt.path == 2)
    for (int k = 0; k < d; ++k)
      if (!L.tc_range[k]) return fail(RTK_ERR_SHAPE, "tcgen05 path unavailable for mode " + std::to_string(k + 1));
  char* ws = (char*)ws_in;
  bool own = false;
  if (!ws) {
    RTK_CK(cudaMallocAsync((void**)&ws, L.total, st));
    own = true;
  } else if (ws_bytes < L.total) {
    return fail(RTK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(L.total) + " bytes");
  }
  RTK_CK(cudaMemsetAsync(ws + L.status, 0, (size_t)d * 4 * 4, st));
  RTK_CK(cudaMemsetAsync(ws + L.trace, 0, (size_t)d * q * 8, st));
  RTK_CK(cudaMemsetAsync(ws + L.xmax, 0, 8 * 4, st));
  XState xst;
  xst.xmax = (float*)(ws + L.xmax);
  float* shr[2] = {(float*)(ws + L.shr0), (float*)(ws + L.shr1)};
  const bool shift = opt.shift != 0;
  if (P.a2) {
    // Alg. A.2: mode k runs Alg. 4's shifted range finder on B_(k) and
    // keeps all l_k columns, B = B x_k Q_k^T (U[k] is scratch until a2_finish writes it)
    std::vector<double*> qk(d);
    size_t qoff = 0;
    for (int k = 0; k < d; ++k) {
      const float* cur = k == 0 ? A : shr[(k - 1) & 1];
      const View rv = range_view(P, k, A, cur);
      rc = run_mode(P, L, ws, k, rv, seed, shift, U[k], st, &xst);
      if (rc) return rc;
      qk[k] = (double*)(ws + L.a2q) + qoff;
      qoff += (size_t)P.dims[k] * P.keep[k];
      RTK_CK(cudaMemcpyAsync(qk[k], ws + L.qd, (size_t)P.dims[k] * P.keep[k] * 8, cudaMemcpyDeviceToDevice, st));
      const View sv = shrink_view(P, k, A, cur);
      rc = run_shrink(P, L, ws, k, sv, (const float*)(ws + L.qs), k + 1 < d ? shr[k & 1] : (float*)(ws + L.a2b), st,
                      &xst);
      if (rc) return rc;
    }
    {   // lines 14-15: ST-HOSVD of the l_1 x ... x l_d tensor, U_k = Q_k V_k
      ProfScope ps(3, d - 1, st);
      RTK_CK(a2_finish((const float*)(ws + L.a2b), d, P.keep.data(), P.ranks.data(), P.dims.data(), qk.data(),
                       (double*)(ws + L.a2g0), (double*)(ws + L.a2g1), (double*)(ws + L.a2gram),
                       (double*)(ws + L.a2v), U, core, st));
      g_launches += 2 + 4 * d;
    }
  } else if (P.seq) {
    // Alg. 4: factor G_(k), then G = G x_k U_k^T
    for (int k = 0; k < d; ++k) {
      const float* cur = k == 0 ? A : shr[(k - 1) & 1];
      const View rv = range_view(P, k, A, cur);
      rc = run_mode(P, L, ws, k, rv, seed, shift, U[k], st, &xst);
      if (rc) return rc;
      const View sv = shrink_view(P, k, A, cur);
      rc = run_shrink(P, L, ws, k, sv, U[k], k + 1 < d ? shr[k & 1] : core, st, &xst);
      if (rc) return rc;
    }
  } else {
    // Alg. 3: every mode factors the original A_(k) through its strided view; the modes are
    // independent, so each runs on its own stream in its own scratch region (fork / join events)
    ModeStreams* ms = nullptr;
    RTK_CK(mode_streams(&ms));
    RTK_CK(cudaEventRecord(ms->fork, st));
    for (int k = 0; k < d; ++k) {
      RTK_CK(cudaStreamWaitEvent(ms->s[k], ms->fork, 0));
      const View rv = range_view(P, k, A, nullptr);
      rc = run_mode(P, L, ws, k, rv, seed, shift, U[k], ms->s[k], &xst);
      if (rc) return rc;
      RTK_CK(cudaEventRecord(ms->join[k], ms->s[k]));
    }
    for (int k = 0; k < d; ++k) RTK_CK(cudaStreamWaitEvent(st, ms->join[k], 0));
    // core = A x_1 U_1^T ... x_d U_d^T, same shrink chain
    for (int k = 0; k < d; ++k) {
      const float* cur = k == 0 ? A : shr[(k - 1) & 1];
      const View sv = shrink_view(P, k, A, cur);
      rc = run_shrink(P, L, ws, k, sv, U[k], k + 1 < d ? shr[k & 1] : core, st);
      if (rc) return rc;
    }
  }
  if (nflag) {
    int* dflag = nullptr;
    RTK_CK(cudaHostGetDevicePointer((void**)&dflag, nflag, 0));
    numeric_flag_kernel<<<1, 1, 0, st>>>((const int*)(ws + L.status), d, dflag);
    RTK_CK(cudaGetLastError());
    g_launches += 1;
  }
  bool numeric = false;
  if (rep) {
    RTK_CK(cudaStreamSynchronize(st));
    std::vector<int> status((size_t)d * 4);
    RTK_CK(cudaMemcpy(status.data(), ws + L.status, status.size() * 4, cudaMemcpyDeviceToHost));
    if (rep->alpha_trace)
      RTK_CK(cudaMemcpy(rep->alpha_trace, ws + L.trace, (size_t)d * q * 8, cudaMemcpyDeviceToHost));
    if (rep->sigma)
      RTK_CK(cudaMemcpy(rep->sigma, ws + L.sigma, (size_t)d * 128 * 8, cudaMemcpyDeviceToHost));
    rep->fallback = 0;
    rep->numeric = 0;
    for (int k = 0; k < d; ++k) {
      if (rep->q_used) rep->q_used[k] = status[4 * k + 2];
      rep->fallback += status[4 * k + 1];
      if (status[4 * k]) rep->numeric = RTK_ERR_NUMERIC;
    }
    numeric = rep->numeric != 0;
    if (numeric && nflag) *(volatile int*)nflag = 0;   // reported now, not again at the next call
  }
  if (own) RTK_CK(cudaFreeAsync(ws, st));
  RTK_CK(cudaGetLastError());
  if (numeric)
    return fail(RTK_ERR_NUMERIC, "numeric failure (non-finite iterate or unrepairable Cholesky breakdown); "
                                 "outputs written but unreliable");
  return RTK_OK;
}

// ---- multi-GPU last-mode shard -------------------------------------------------
struct ShardPlan {
  Problem loc, full;            // the slab (modes < d-1 run on it) and the whole problem (mode d-1)
  Layout Lloc, Lfull;           // copies: plan_cached's references do not outlive the next insertion
  size_t gather = 0, total = 0; // offset of the gathered mode-d unfolding, workspace bytes
  int64_t M = 1, ldf = 0;       // its columns (prod_{j<d-1} r_j) and leading dimension pad4(n_d)
};

int shard_setup(const rtk_options& o, const float* A, const int64_t* dims, int32_t d, int64_t last_begin,
                int64_t last_count, const int32_t* ranks, int32_t p, int32_t q, ShardPlan& S) {
  if (!dims || !ranks) return fail(RTK_ERR_ARG, "NULL pointer argument");
  if (d < 2 || d > 8) return fail(RTK_ERR_ARG, "d must be in [2, 8]");
  if (o.sequential != 1 || o.variant != 0 || o.pve_tol > 0.0)
    return fail(RTK_ERR_ARG, "the last-mode shard runs Alg. 4 (sequential = 1, variant 0, no PVE)");
  if (o.omega < 0 || o.omega > 3) return fail(RTK_ERR_ARG, "omega must be in [0, 3]");
  Problem& F = S.full;
  F.d = d; F.p = p; F.q = q; F.seq = true; F.omega = o.omega;
  F.dims.assign(dims, dims + d);
  F.ranks.assign(ranks, ranks + d);
  set_keep(F);
  int rc = validate(F);
  if (rc) return rc;
  if (last_count < 1 || last_begin < 0 || last_begin + last_count > dims[d - 1])
    return fail(RTK_ERR_ARG, "the slab [last_begin, last_begin + last_count) must lie inside mode d");
  for (int k = 0; k + 1 < d; ++k)
    if (ranks[k] + p > kSolveLMax) return fail(RTK_ERR_ARG, "the shard needs l_k = r_k + p <= 64 for k < d");
  S.loc = F;
  S.loc.dims[d - 1] = last_count;
  S.loc.full_last = dims[d - 1];
  S.loc.sh_begin = last_begin;
  S.Lloc = plan_cached(S.loc, num_sms(), A, o.path);
  S.Lfull = plan_cached(F, num_sms(), A, o.path);
  S.M = 1;
  for (int k = 0; k + 1 < d; ++k) S.M *= F.keep[k];
  S.ldf = pad4(dims[d - 1]);
  S.gather = align_up(std::max(S.Lloc.total, S.Lfull.total));
  S.total = S.gather + align_up((size_t)S.ldf * S.M * 4);
  return RTK_OK;
}

int solve_shard(const rtk_options& o, const float* A, const int64_t* dims, int32_t d, int64_t last_begin,
                int64_t last_count, int32_t root, const int32_t* ranks, int32_t p, int32_t q, uint64_t seed,
                float* const* U, float* core, void* ws_in, size_t ws_bytes, void* stream, rtk_allreduce_fn ar,
                void* ctx) {
  if (!A || !U || !core || !ar) return fail(RTK_ERR_ARG, "NULL pointer argument");
  ShardPlan S;
  int rc = shard_setup(o, A, dims, d, last_begin, last_count, ranks, p, q, S);
  if (rc) return rc;
  for (int k = 0; k < d; ++k)
    if (!U[k]) return fail(RTK_ERR_ARG, "NULL U[k]");
  if ((uintptr_t)A % 4) return fail(RTK_ERR_ALIGN, "A must be 4-byte aligned");
  S.loc.sh_root = root != 0;
  S.loc.ar = ar;
  S.loc.ar_ctx = ctx;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0;
  RTK_CK(cudaGetDevice(&dev));
  int* nflag = numeric_flag_host(dev);
  if (nflag && *(volatile int*)nflag) {
    *(volatile int*)nflag = 0;
    return fail(RTK_ERR_NUMERIC, "an earlier solve on this device hit a numeric failure");
  }
  char* ws = (char*)ws_in;
  bool own = false;
  if (!ws) {
    RTK_CK(cudaMallocAsync((void**)&ws, S.total, st));
    own = true;
  } else if (ws_bytes < S.total) {
    return fail(RTK_ERR_WORKSPACE, "workspace too small: need " + std::to_string(S.total) + " bytes");
  }
  const Layout& Ll = S.Lloc;
  const Layout& Lf = S.Lfull;
  // the report slots sit at the same offsets in both layouts (they depend on d and q only)
  RTK_CK(cudaMemsetAsync(ws + Lf.status, 0, (size_t)d * 4 * 4, st));
  RTK_CK(cudaMemsetAsync(ws + Lf.trace, 0, (size_t)d * q * 8, st));
  RTK_CK(cudaMemsetAsync(ws + Ll.xmax, 0, 8 * 4, st));   // same offset in both layouts (d, q only)
  XState xs_slab;   // fp16 pair engine on the slab: each rank scales by its own slab's max|M|
  xs_slab.xmax = (float*)(ws + Ll.xmax);
  const bool shift = o.shift != 0;
  float* shr[2] = {(float*)(ws + Ll.shr0), (float*)(ws + Ll.shr1)};
  // modes 1 .. d-1 on the slab; the last shrink leaves the slab's mode-d unfolding in shr[(d-2)&1]
  for (int k = 0; k + 1 < d; ++k) {
    const float* cur = k == 0 ? A : shr[(k - 1) & 1];
    const View rv = range_view(S.loc, k, A, cur);
    rc = run_mode(S.loc, Ll, ws, k, rv, seed, shift, U[k], st, &xs_slab);
    if (rc) return rc;
    const View sv = shrink_view(S.loc, k, A, cur);
    rc = run_shrink(S.loc, Ll, ws, k, sv, U[k], shr[k & 1], st, &xs_slab);
    if (rc) return rc;
  }
  // gather: the slab's rows [last_begin, +last_count) of the mode-d unfolding, zero elsewhere, summed
  float* full = (float*)(ws + S.gather);
  const float* slab = shr[(d - 2) & 1];
  RTK_CK(cudaMemsetAsync(full, 0, (size_t)S.ldf * S.M * 4, st));
  RTK_CK(cudaMemcpy2DAsync(full + last_begin, (size_t)S.ldf * 4, slab, (size_t)pad4(last_count) * 4,
                           (size_t)last_count * 4, (size_t)S.M, cudaMemcpyDeviceToDevice, st));
  if (ar((void*)full, (int64_t)S.ldf * S.M, 0, (void*)st, ctx) != 0)
    return fail(RTK_ERR_CUDA, "all-reduce callback failed (mode-d gather)");
  // mode d and the core, redundantly on the whole (small) problem
  {
    const int k = d - 1;
    const View rv = range_view(S.full, k, A, full);
    // the gathered unfolding's max|M| is known only once its own sketch has run (the slab's shrink
    // saw one rank's rows; its atomicMax is a lower bound the sketch's raises to the full maximum)
    XState xs_full;
    xs_full.xmax = (float*)(ws + Lf.xmax);
    rc = run_mode(S.full, Lf, ws, k, rv, seed, shift, U[k], st, &xs_full);
    if (rc) return rc;
    const View sv = shrink_view(S.full, k, A, full);
    rc = run_shrink(S.full, Lf, ws, k, sv, U[k], core, st);
    if (rc) return rc;
  }
  if (nflag) {
    int* dflag = nullptr;
    RTK_CK(cudaHostGetDevicePointer((void**)&dflag, nflag, 0));
    numeric_flag_kernel<<<1, 1, 0, st>>>((const int*)(ws + Lf.status), d, dflag);
    RTK_CK(cudaGetLastError());
    g_launches += 1;
  }
  if (own) RTK_CK(cudaFreeAsync(ws, st));
  RTK_CK(cudaGetLastError());
  return RTK_OK;
}

// ---------------------------------------------------------------- CUDA-graph replay of a solve
// A solve is ~100-300 launches (PDL chains, side-stream forks, memsets) whose host enqueue and
// launch gaps cost up to ~3 % of a small config (C4).  Repeated calls with IDENTICAL arguments
// (every pointer, extent, option, the seed, the device and every RTK_* environment override) replay
// one captured graph instead: the first call of a key runs directly (it also creates the lazily
// allocated streams / events / pinned flags), the second captures the enqueue on a private stream
// (relaxed capture mode) and launches the graph on the caller's stream, later calls only launch.
// Replay reads and writes the same buffers through the same kernels, so results are bit-identical
// to the direct path (tests/test_gpu_graph.py).  Bypassed when a report is requested (it needs a
// host sync), when the library allocates the workspace, while per-launch profiling or the step-clock
// diagnostics are active, when the caller's stream is itself capturing, and with RTK_GRAPH=0.
// The sticky RTK_ERR_NUMERIC check runs on the host before every replay, as on the direct path.
struct GraphEntry {
  std::string key;
  int seen = 0;                 // direct runs of this key so far
  bool bad = false;             // capture failed once: always direct
  cudaGraphExec_t exec = nullptr;
  long long launches = 0;       // kernel launches the captured enqueue counted
};

std::string graph_key(const rtk_options& o, const float* A, const int64_t* dims, int32_t d, const int32_t* ranks,
                      int32_t p, int32_t q, uint64_t seed, float* const* U, float* core, void* ws, size_t ws_bytes,
                      int dev) {
  std::string key;
  key.reserve(512);
  auto add = [&](unsigned long long x) { key += std::to_string(x); key += ','; };
  add((unsigned)dev); add((unsigned)o.sequential); add((unsigned)o.shift); add((unsigned)o.path);
  add((unsigned)o.variant); add((unsigned)o.omega);
  unsigned long long pb = 0;
  std::memcpy(&pb, &o.pve_tol, sizeof(pb));
  add(pb);
  add((uintptr_t)A); add((unsigned)d); add((unsigned)p); add((unsigned)q); add(seed);
  for (int k = 0; k < d; ++k) { add((unsigned long long)dims[k]); add((unsigned)ranks[k]); add((uintptr_t)U[k]); }
  add((uintptr_t)core); add((uintptr_t)ws); add(ws_bytes);
  // every RTK_* override (path and engine switches are read at enqueue time)
  for (char** e = ::environ; e && *e; ++e)
    if (std::strncmp(*e, "RTK_", 4) == 0) { key += *e; key += ';'; }
  return key;
}

bool graph_enabled() {
  const char* g = getenv("RTK_GRAPH");
  return !(g && g[0] == '0');
}

int solve_entry(const rtk_options& o, const float* A, const int64_t* dims, int32_t d, const int32_t* ranks,
                int32_t p, int32_t q, uint64_t seed, float* const* U, float* core, void* ws, size_t ws_bytes,
                void* stream, rtk_report* rep) {
  cudaStream_t st = (cudaStream_t)stream;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (rep || !ws || g_prof_on.load() || g_step_dbg || !graph_enabled() || !A || !dims || !ranks || !U || !core ||
      d < 2 || d > 8 || cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return solve(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
  }
  int dev = 0;
  RTK_CK(cudaGetDevice(&dev));
  const std::string key = graph_key(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, dev);
  static std::mutex mu;
  static std::vector<GraphEntry> cache;   // most recently used last
  std::unique_lock<std::mutex> lk(mu);
  size_t idx = cache.size();
  for (size_t i = 0; i < cache.size(); ++i)
    if (cache[i].key == key) { idx = i; break; }
  if (idx == cache.size()) {
    if (cache.size() >= 32) {   // evict the least recently used graph (no launch of it may be pending)
      if (cache.front().exec) {
        cudaDeviceSynchronize();
        cudaGraphExecDestroy(cache.front().exec);
      }
      cache.erase(cache.begin());
    }
    GraphEntry e;
    e.key = key;
    cache.push_back(std::move(e));
    idx = cache.size() - 1;
  } else if (idx + 1 != cache.size()) {
    std::rotate(cache.begin() + idx, cache.begin() + idx + 1, cache.end());
    idx = cache.size() - 1;
  }
  GraphEntry& E = cache[idx];
  if (!E.exec && (E.bad || E.seen == 0)) {   // first sight (or uncapturable): direct
    lk.unlock();
    const int rc = solve(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
    lk.lock();
    for (auto& c : cache)
      if (c.key == key && rc == RTK_OK) c.seen += 1;
    return rc;
  }
  if (!E.exec) {   // second sight: capture the enqueue on a private stream
    static thread_local cudaStream_t cs[64] = {};
    if (dev < 0 || dev >= 64) return solve(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
    if (!cs[dev]) RTK_CK(cudaStreamCreateWithFlags(&cs[dev], cudaStreamNonBlocking));
    const long long l0 = g_launches.load();
    RTK_CK(cudaStreamBeginCapture(cs[dev], cudaStreamCaptureModeRelaxed));
    const int rc = solve(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, (void*)cs[dev], nullptr);
    cudaGraph_t g = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(cs[dev], &g);
    cudaGraphExec_t ex = nullptr;
    cudaError_t ei = cudaErrorUnknown;
    if (rc == RTK_OK && ec == cudaSuccess && g) ei = cudaGraphInstantiate(&ex, g, 0);
    if (g) cudaGraphDestroy(g);
    if (rc != RTK_OK) return rc;   // argument / numeric errors: nothing was enqueued
    if (ec != cudaSuccess || ei != cudaSuccess) {   // not capturable: direct from now on
      cudaGetLastError();
      if (ex) cudaGraphExecDestroy(ex);
      E.bad = true;
      lk.unlock();
      return solve(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
    }
    E.exec = ex;
    E.launches = g_launches.load() - l0;
  }
  int* nflag = numeric_flag_host(dev);
  if (nflag && *(volatile int*)nflag) {
    *(volatile int*)nflag = 0;
    return fail(RTK_ERR_NUMERIC, "an earlier solve on this device hit a numeric failure (non-finite iterate or "
                                 "unrepairable Cholesky breakdown); its outputs are unreliable");
  }
  RTK_CK(cudaGraphLaunch(E.exec, st));
  g_launches += E.launches;
  return RTK_OK;
}

}  // namespace
}  // namespace rtk

using namespace rtk;

extern "C" {

int rtk_solve(const rtk_options* opt, const float* A, const int64_t* dims, int32_t d, const int32_t* ranks,
              int32_t p, int32_t q, uint64_t seed, float* const* U, float* core, void* ws,
              size_t ws_bytes, void* stream, rtk_report* rep) {
  rtk_options o = {1, 1, 0.0, 0, 0, 0};
  if (opt) o = *opt;
  return rtk::solve_entry(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
}

int rtk_rthosvd(const float* A, const int64_t* dims, int32_t d, const int32_t* ranks, int32_t p,
                int32_t q, uint64_t seed, float* const* U, float* core, void* ws, size_t ws_bytes,
                void* stream, rtk_report* rep) {
  rtk_options o = {0, 1, 0.0, 0, 0, 0};
  return rtk::solve_entry(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
}

int rtk_rsthosvd(const float* A, const int64_t* dims, int32_t d, const int32_t* ranks, int32_t p,
                 int32_t q, uint64_t seed, float* const* U, float* core, void* ws, size_t ws_bytes,
                 void* stream, rtk_report* rep) {
  rtk_options o = {1, 1, 0.0, 0, 0, 0};
  return rtk::solve_entry(o, A, dims, d, ranks, p, q, seed, U, core, ws, ws_bytes, stream, rep);
}

size_t rtk_workspace_bytes(int32_t algo, const int64_t* dims, int32_t d, const int32_t* ranks, int32_t p,
                           int32_t q) {
  if (!dims || !ranks || d < 2 || d > 8) {
    g_err = "invalid arguments";
    return 0;
  }
  Problem P;
  P.d = d; P.p = p; P.q = q; P.seq = algo != 0;
  P.a2 = algo == 2;
  P.dims.assign(dims, dims + d);
  P.ranks.assign(ranks, ranks + d);
  set_keep(P);
  if (validate(P)) return 0;
  return plan(P, num_sms(), nullptr, 0).total;
}

int rtk_sketch(int32_t kind, uint64_t seed, int32_t mode, const int64_t* dims, int32_t d, int64_t row0, int64_t rows,
               int32_t l, float* out, void* stream) {
  if (kind == 0) return rtk_omega(seed, mode, row0, rows, l, out, stream);
  if (!out || !dims || d < 2 || d > 8 || mode < 1 || mode > d || rows < 0 || row0 < 0 || l < 1 || kind < 0 ||
      kind > 3)
    return fail(RTK_ERR_ARG, "invalid rtk_sketch arguments");
  int64_t m = 1;
  for (int j = 0; j < d; ++j) {
    if (dims[j] < 1) return fail(RTK_ERR_ARG, "dims[k] must be >= 1");
    if (j + 1 != mode) m *= dims[j];
  }
  if (row0 + rows > m) return fail(RTK_ERR_ARG, "rows past the unfolding's column count");
  if (rows == 0) return RTK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  float* tabs = nullptr;
  const size_t tf = std::max<size_t>(sketch_tab_floats(dims, d, mode, l), 1);
  RTK_CK(cudaMallocAsync((void**)&tabs, tf * 4, st));
  RTK_CK(sketch_materialize(kind, seed, mode, dims, d, row0, rows, l, tabs, out, st));
  RTK_CK(cudaFreeAsync(tabs, st));
  return RTK_OK;
}

int rtk_rsthosvd_shard(const rtk_options* opt, const float* A_slab, const int64_t* dims, int32_t d,
                       int64_t last_begin, int64_t last_count, int32_t root, const int32_t* ranks, int32_t p,
                       int32_t q, uint64_t seed, float* const* U, float* core, void* ws, size_t ws_bytes,
                       void* stream, rtk_allreduce_fn allreduce, void* ctx) {
  rtk_options o = {1, 1, 0.0, 0, 0, 0};
  if (opt) o = *opt;
  return rtk::solve_shard(o, A_slab, dims, d, last_begin, last_count, root, ranks, p, q, seed, U, core, ws,
                          ws_bytes, stream, allreduce, ctx);
}

size_t rtk_workspace_bytes_shard(const rtk_options* opt, const int64_t* dims, int32_t d, int64_t last_count,
                                 const int32_t* ranks, int32_t p, int32_t q) {
  rtk_options o = {1, 1, 0.0, 0, 0, 0};
  if (opt) o = *opt;
  rtk::ShardPlan S;
  if (!dims || d < 2 || d > 8) {
    g_err = "invalid arguments";
    return 0;
  }
  if (rtk::shard_setup(o, nullptr, dims, d, 0, last_count, ranks, p, q, S)) return 0;
  return S.total;
}

size_t rtk_workspace_bytes_ex(const rtk_options* opt, const int64_t* dims, int32_t d, const int32_t* ranks,
                              int32_t p, int32_t q) {
  rtk_options o = {1, 1, 0.0, 0, 0, 0};
  if (opt) o = *opt;
  if (!dims || !ranks || d < 2 || d > 8 || o.omega < 0 || o.omega > 3 || o.variant < 0 || o.variant > 1) {
    g_err = "invalid arguments";
    return 0;
  }
  Problem P;
  P.d = d; P.p = p; P.q = q; P.seq = o.sequential != 0;
  P.a2 = o.variant == 1;
  P.omega = o.omega;
  P.dims.assign(dims, dims + d);
  P.ranks.assign(ranks, ranks + d);
  set_keep(P);
  if (validate(P)) return 0;
  return plan_cached(P, num_sms(), nullptr, o.path).total;
}

int rtk_omega(uint64_t seed, int32_t mode, int64_t row0, int64_t rows, int32_t l, float* out, void* stream) {
  if (!out || rows < 0 || row0 < 0 || l < 1 || mode < 0) return fail(RTK_ERR_ARG, "invalid rtk_omega arguments");
  if (rows == 0) return RTK_OK;
  cudaError_t e = launch_omega(seed, (uint32_t)mode, row0, rows, l, out, (cudaStream_t)stream);
  if (e != cudaSuccess) return fail(RTK_ERR_CUDA, cudaGetErrorString(e));
  return RTK_OK;
}

int rtk_power_step(const float* M, int64_t n, int64_t m, int64_t ld, const float* Q, int32_t l, double* Y,
                   void* stream) {
  if (!M || !Q || !Y || n < 1 || m < 1 || ld < n || l < 1 || n > kNMax)
    return fail(RTK_ERR_ARG, "invalid rtk_power_step arguments");
  cudaStream_t st = (cudaStream_t)stream;
  View v;
  v.base = M; v.n = (int)n; v.P = 1; v.S = m; v.sp = 1; v.si = 1; v.ss = ld;
  const char* pe = getenv("RTK_PATH");
  const char* fz = getenv("RTK_FUSED");
  if (!(pe && std::string(pe) == "ffma") && tc_supported(v, l) && !(fz && fz[0] == '0') && fused_supported(v, l)) {
    // the fused single-pass engine of the solver (rtk_fused.cu)
    const int N = tc_npad(l), G = num_sms();
    // RTK_POWER_F16=1 (test hook only): the fp16 pair engine, with max|M| and the fp16 Q planes
    // prepared here the way the solver's sketch / shrink and step kernels prepare them
    const char* pf = getenv("RTK_POWER_F16");
    const bool h16 = pf && pf[0] == '1' && pair_supported(v, l);
    const int64_t pld = h16 ? pad8(n) : pad4(n);
    float *planes = nullptr, *yp = nullptr, *xm = nullptr;
    RTK_CK(cudaMallocAsync((void**)&planes, (size_t)2 * N * pld * 4, st));
    RTK_CK(cudaMallocAsync((void**)&yp, fused_ypart_floats(v, l, G) * 4, st));
    PairScale ps;
    if (h16) {
      RTK_CK(cudaMallocAsync((void**)&xm, 4, st));
      RTK_CK(pair_prepare16(v, Q, l, N, (int)pld, planes, xm, st));
      ps.xmax_in = xm;
    } else {
      RTK_CK(tc_split(nullptr, Q, (int)n, l, planes, st));
    }
    int Gf = 0, rows = 0;
    RTK_CK(fused_power(v, l, planes, (int)pld, false, 0, 0, yp, G, &Gf, &rows, st, nullptr, 1, 1, 1, nullptr,
                       nullptr, &ps));
    RTK_CK(launch_sum_partials(yp, Gf, N, rows, (int)n, l, Y, st));
    RTK_CK(cudaFreeAsync(planes, st));
    RTK_CK(cudaFreeAsync(yp, st));
    if (xm) RTK_CK(cudaFreeAsync(xm, st));
    return RTK_OK;
  }
  if (!(pe && std::string(pe) == "ffma") && tc_supported(v, l)) {
    const int N = tc_npad(l), nit = (int)((n + 127) / 128), G = num_sms();
    const int64_t ldw = pad4(m);
    float *planes = nullptr, *W = nullptr, *yp = nullptr;
    RTK_CK(cudaMallocAsync((void**)&planes, (size_t)2 * N * pad4(n) * 4, st));
    RTK_CK(cudaMallocAsync((void**)&W, (size_t)2 * N * ldw * 4, st));
    RTK_CK(cudaMallocAsync((void**)&yp, (size_t)G * N * nit * 128 * 4, st));
    RTK_CK(tc_split(nullptr, Q, (int)n, l, planes, st));
    RTK_CK(tc_op1(v, l, planes, W, ldw, false, nullptr, 1, 1, 1, st));
    RTK_CK(tc_op2(v, l, W, ldw, false, 0, 0, yp, G, st));
    RTK_CK(launch_sum_partials(yp, G, N, nit * 128, (int)n, l, Y, st));
    RTK_CK(cudaFreeAsync(planes, st));
    RTK_CK(cudaFreeAsync(W, st));
    RTK_CK(cudaFreeAsync(yp, st));
    return RTK_OK;
  }
  TileLaunch T;
  T.v = v;
  T.op = OP_POWER;
  T.tp = plan_tile(v, l, OP_POWER, num_sms());
  T.l = l;
  T.Q = Q;
  T.qld = (int)n;
  float* yp = nullptr;
  const size_t bytes = (size_t)T.tp.G * T.tp.ltot() * T.tp.n_rows() * 4;
  RTK_CK(cudaMallocAsync((void**)&yp, bytes, st));
  T.Ypart = yp;
  RTK_CK(launch_tile(T, st));
  RTK_CK(launch_sum_partials(yp, T.tp.G, T.tp.ltot(), T.tp.n_rows(), (int)n, l, Y, st));
  RTK_CK(cudaFreeAsync(yp, st));
  return RTK_OK;
}

int rtk_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  g_launches = 0;
  g_prof_on = true;
  return RTK_OK;
}

int rtk_profile_end(rtk_prof_stats* out) {
  g_prof_on = false;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (out) std::memset(out, 0, sizeof(*out));
  int rc = RTK_OK;
  for (auto& r : g_prof) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess) rc = fail(RTK_ERR_CUDA, cudaGetErrorString(e));
    if (out && r.kind >= 0 && r.kind < 4 && r.mode >= 0 && r.mode < 8) {
      out->ms[r.kind][r.mode] += ms;
      out->count[r.kind][r.mode] += 1;
    }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  if (out) out->launches = g_launches.load();
  return rc;
}

int rtk_debug_step_clocks(void* dev_buf) {
  rtk::g_step_dbg = (double*)dev_buf;
  return RTK_OK;
}

const char* rtk_last_error(void) { return g_err.c_str(); }

const char* rtk_version(void) { return "rtucker 0.1.0 sm_100a"; }

}  // extern "C"
