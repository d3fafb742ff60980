/*
 * rtucker.h -- C ABI of the B200-native adaptive-shift randomized Tucker hot path.
 *
 * Implements the per-mode randomized range finder with adaptive shifted power
 * iteration of Che, Wei, Wu, Yan, arXiv 2506.04840:
 *   Alg. 3 "shifted randomized T-HOSVD"   PAPER.md:250-270   -> rtk_rthosvd
 *   Alg. 4 "shifted randomized ST-HOSVD"  PAPER.md:293-313   -> rtk_rsthosvd
 *   Alg. 2 (alpha = 0) and Alg. B.1 (PVE stop,
 *   PAPER.md:1145-1172) through rtk_solve() options.
 * Per mode k (order 1..d): Omega_k (RTK-GAUSS-2),
 * Y = M Omega_k, Q = orth(Y), alpha = 0; q times { Y = M (M^T Q) - alpha Q;
 * [Q,Sigma] = svd(Y); if Sigma(l,l) > alpha: alpha = (Sigma(l,l)+alpha)/2 };
 * U_k = Q(:,1:r_k) (sign-pinned); M = A_(k) (Alg. 3) or G_(k) (Alg. 4), and
 * Alg. 4 shrinks G = G x_k U_k^T after each mode.
 *
 * LAYOUT.  All tensors are float32, COLUMN-MAJOR (mode-1 index fastest; the
 * MATLAB / Kolda-Bader convention):  A[i_1 + n_1 (i_2 + n_2 (...))].
 * That is the same byte layout as a C-contiguous torch tensor of shape
 * (n_d, ..., n_1).  U[k] is n_k x r_k column-major (leading dimension n_k).
 * core is r_1 x ... x r_d column-major.  A, U[k] and core are DEVICE pointers.
 *
 * OWNERSHIP.  The caller allocates and owns A, every U[k], core and ws; the
 * library never frees them and never writes A.  The library keeps no state
 * between calls except a per-thread error string, cached kernel attributes and,
 * per host thread and device, a small pool of internal streams and events (the
 * side stream of the deferred shift update and Alg. 3's per-mode streams, joined
 * back into `stream` before the call returns its work) and the CUDA graphs of
 * repeated calls (REPEATED CALLS below).  A ws shared by two
 * calls must not be in use by both at once (ordinary stream ordering suffices).
 * If ws == NULL the call allocates (cudaMallocAsync) and frees its own
 * workspace on the stream.
 *
 * EXECUTION.  Asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 * stream).  Outputs are valid once the stream is synchronised.  If `rep` is
 * non-NULL the call synchronises the stream and fills the report.
 *
 * ERRORS.  Every function returns an rtk_status; nothing throws across the ABI.
 * All argument checks run before any launch; on a non-zero status other than
 * RTK_ERR_NUMERIC no output is written.  rtk_last_error() returns a thread-local
 * message for the last non-zero status of this thread.
 *
 * NUMERIC FAILURES (RTK_ERR_NUMERIC).  A solve that meets a non-finite iterate (a NaN /
 * inf in A, or an iterate Y = M M^T Q beyond the fp32 range: the stream squares the
 * scale of A, so max|A| must stay well below ~1e13) or a Cholesky breakdown its basis
 * completion cannot repair still writes its outputs (unreliable).  With a report (rep != NULL) that call returns RTK_ERR_NUMERIC and
 * sets rep->numeric.  Without a report the call is asynchronous and cannot see its
 * own result: the failure is latched in a per-device flag and the NEXT solver call
 * on that device (once the failing solve has executed) returns RTK_ERR_NUMERIC
 * without launching anything and clears the flag (CUDA sticky-error style).
 *
 * LIMITS.  n_k <= 4096 (tile kernels), l_k = r_k + p <= 96 (one-CTA small solves;
 * l_k <= 64 takes the cluster small solver), Alg. A.2 and Alg. B.1 need l_k <= 64.
 *
 * STREAMING PATHS (chosen per mode, results equal up to rounding; rtk_options.path
 * forces one).  tcgen05 when l_k <= 64, the view is 16-byte aligned and
 * its leading dimension a multiple of 4:
 *   - contiguous views (mode 1 of A, every Alg. 4 mode, since Alg. 4 writes each shrunk
 *     unfolding contiguously) with n_k > 256 and at least one 256-column pair-block per two
 *     SM pairs: the CTA-pair engine (cta_group::2); its power steps use fp16 two-plane
 *     operands (3xFP16) once max|M| of the unfolding is known, else 3xTF32;
 *   - other contiguous views with n_k <= 1024: the one-CTA fused single-HBM-pass engine;
 *   - Alg. 3's strided views (modes >= 2 of A): the one-CTA fused engine through 3-D TMA
 *     tensor maps {p, i, s} (no permute copy);
 *   - contiguous views with n_k > 1024: the two-kernel tcgen05 path.
 * l_k > 64, unaligned data and views the engines do not take use the FP32 FFMA tile
 * kernels (bulk-copy row loads, no permute).
 * ACCURACY NOTE.  The tcgen05 engines accumulate in the tensor core's fp32 accumulator, which
 * rounds toward zero: on same-sign data a power step's Y comes out uniformly smaller by up to
 * ~1e-4 relative at C5 size (mixed-sign data: ~1e-5), alpha by twice that; the column space
 * (U_k, RE) is unaffected to first order.  path = 1 (FFMA tiles) has no such bias
 * (profiles/r2m_rz_probe.md).
 *
 * REPEATED CALLS (CUDA graphs).  rtk_solve / rtk_rthosvd / rtk_rsthosvd called again with
 * IDENTICAL arguments (every pointer, extent, option, the seed, the device and every RTK_*
 * environment variable) replay a CUDA graph of the first call's launch sequence: the second
 * call of such a key captures it (on a private stream) and launches it on `stream`, later
 * calls only launch it.  The graph reads the CURRENT contents of A and writes the same
 * outputs, bit-identical to the direct path.  A graph exists only for arguments that passed
 * every check once; the sticky RTK_ERR_NUMERIC check runs before every replay.  Not used when rep != NULL, ws == NULL, per-launch
 * profiling is on, `stream` is being captured by the caller, or RTK_GRAPH=0; at most 32
 * graphs are kept (least recently used evicted after a device synchronise).
 */
#ifndef RTUCKER_H
#define RTUCKER_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define RTK_API __attribute__((visibility("default")))
#else
#define RTK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rtk_status {
  RTK_OK = 0,
  RTK_ERR_ARG = 1,       /* NULL pointer; d < 2 or d > 8; n_k < 1; r_k not in [1,n_k]; p < 0; q < 1 */
  RTK_ERR_SHAPE = 2,     /* l_k = r_k + p > min(n_k, m_k); n_k > 4096 or l_k > 96
                          * (kernel limits); Alg. A.2 with l_k > 64; path = 2 where tcgen05 n/a */
  RTK_ERR_ALIGN = 3,     /* A not 4-byte aligned */
  RTK_ERR_WORKSPACE = 4, /* ws_bytes < rtk_workspace_bytes(...) */
  RTK_ERR_CUDA = 5,      /* launch / runtime error; message kept */
  RTK_ERR_NUMERIC = 6    /* non-finite iterate or unrepairable Cholesky breakdown: returned by the
                          * call itself when rep != NULL, else by the next call (see above) */
} rtk_status;

/* Optional host-side report (SPEC ShiftTrace analogue).  Any pointer may be NULL. */
typedef struct rtk_report {
  double* alpha_trace;  /* [d * q] : alpha after power step t of mode k at [k*q + t]     */
  double* sigma;        /* [d * 128]: final diag(Sigma_k)+alpha of mode k at [k*128 + i] */
  int32_t* q_used;      /* [d]   : power steps actually taken (== q unless PVE stopped)  */
  int32_t fallback;     /* out   : # of rank-deficient basis completions performed        */
  int32_t numeric;      /* out   : 0 ok, else RTK_ERR_NUMERIC                              */
} rtk_report;

/* Solver options for rtk_solve (defaults: {1, 1, 0.0, 0, 0}). */
typedef struct rtk_options {
  int32_t sequential; /* 0: T-HOSVD (Alg. 3, every mode factors A_(k)); 1: ST-HOSVD (Alg. 4) */
  int32_t shift;      /* 1: adaptive shift (Alg. 3/4); 0: alpha == 0 (Alg. 2)                */
  double pve_tol;     /* > 0: Alg. B.1 per mode, q is q_max: after power
                       * step j, sigma = diag(Sigma)+alpha; stop (U_k = that step's basis, no
                       * shift update) when max_{i<=r_k}|sigma_i - sigmahat_i| <= pve_tol *
                       * sigma_{r_k+1}.  RTK_ERR_ARG unless sequential, p >= 1, r_k+p <= 64.
                       * q_used / alpha_trace report the steps taken (trace zero past them). */
  int32_t path;       /* 0: auto, 1: FP32 FFMA tiles, 2: tcgen05 3xTF32 (RTK_ERR_SHAPE if n/a)  */
  int32_t variant;    /* 0: Alg. 2/3/4 as selected above; 1: Alg. A.2 (A.1 with
                       * shift = 0): every mode keeps all l_k = r_k + p columns (B = B x_k Q_k^T),
                       * then a deterministic fp64 ST-HOSVD of the l_1 x ... x l_d tensor gives
                       * V_k and U_k = Q_k V_k (sign pin C6).  Needs sequential = 1, pve_tol = 0,
                       * l_k <= 64 and l_k <= min(n_k, m_k) with m_k over l_1..l_{k-1}
                       * (RTK_ERR_ARG / RTK_ERR_SHAPE otherwise). */
  int32_t omega;      /* sketch type (Appendix D): 0 standard Gaussian
                       * (RTK-GAUSS-2, generated inside the sketch kernels), 1 uniform U[-1,1]
                       * (RTK-UNIF-1), 2 Khatri-Rao product of Gaussian factors, 3 Khatri-Rao
                       * product of uniform factors (RTK-KR-1); types 1-3 are materialised once per
                       * mode in the workspace (rtk_workspace_bytes_ex sizes it) */
} rtk_options;

/*
 * Shifted randomized T-HOSVD, Alg. 3.
 *   A      device, float32, column-major n_1 x ... x n_d, 4-byte aligned (16-byte and
 *          n_1 % 4 == 0 select the fast vector loader; otherwise a scalar loader)
 *   dims   host, d entries n_k >= 1;   d in [2, 8]
 *   ranks  host, d entries r_k in [1, n_k]
 *   p      oversampling s_k (same for all modes), l_k = r_k + p
 *   q      power steps >= 1
 *   seed   Omega seed (RTK-GAUSS-2 key); mode k uses counter word 3 = k (1-based)
 *   U      host array of d DEVICE pointers, U[k] -> n_k x r_k float32 (written)
 *   core   device, r_1 x ... x r_d float32 (written); core = A x_1 U_1^T ... x_d U_d^T
 *   ws     device workspace of ws_bytes (>= rtk_workspace_bytes), or NULL
 *   stream cudaStream_t
 *   rep    optional host report (NULL: fully asynchronous)
 */
RTK_API int rtk_rthosvd(const float* A, const int64_t* dims, int32_t d, const int32_t* ranks,
                int32_t p, int32_t q, uint64_t seed, float* const* U, float* core,
                void* ws, size_t ws_bytes, void* stream, rtk_report* rep);

/* Shifted randomized ST-HOSVD, Alg. 4, processing order 1..d.
 * Arguments as rtk_rthosvd; core = G after the last shrink G = G x_d U_d^T. */
RTK_API int rtk_rsthosvd(const float* A, const int64_t* dims, int32_t d, const int32_t* ranks,
                 int32_t p, int32_t q, uint64_t seed, float* const* U, float* core,
                 void* ws, size_t ws_bytes, void* stream, rtk_report* rep);

/* General entry: Alg. 2 / 3 / 4 / B.1 selected by *opt (NULL -> ST-HOSVD, shift on). */
RTK_API int rtk_solve(const rtk_options* opt, const float* A, const int64_t* dims, int32_t d,
              const int32_t* ranks, int32_t p, int32_t q, uint64_t seed, float* const* U,
              float* core, void* ws, size_t ws_bytes, void* stream, rtk_report* rep);

/* Workspace bytes for (algo: 0 = T-HOSVD, 1 = ST-HOSVD, 2 = Alg. A.2) with the Gaussian sketch.
 * Returns 0 on invalid arguments (message in rtk_last_error()). */
RTK_API size_t rtk_workspace_bytes(int32_t algo, const int64_t* dims, int32_t d, const int32_t* ranks,
                           int32_t p, int32_t q);

/* ---- Multi-GPU: Alg. 4 with A split along its LAST mode ----------------------
 *
 * In-place sum of `count` elements (dtype 0: float32, 1: float64) of the DEVICE buffer `buf` over
 * all ranks of the caller's group, ordered on `stream` (the work enqueued before the call produces
 * buf, the work enqueued after it reads the sum).  Every rank must obtain bit-identical sums (NCCL
 * and gloo all-reduce do).  Returns 0 on success. */
typedef int (*rtk_allreduce_fn)(void* buf, int64_t count, int32_t dtype, void* stream, void* ctx);

/* Alg. 4 (R-ST-HOSVD, sequential = 1, shift as opt->shift, variant 0, no PVE) on one rank of a
 * group that holds A split along mode d: A_slab is this rank's column-major slab, extents
 * dims[0..d-2] x last_count, covering indices [last_begin, last_begin + last_count) of mode d
 * (dims[d-1] = the FULL extent; slabs of all ranks tile it).  For every mode k < d the slab is a
 * contiguous range of the unfolding's columns (i_d is the slowest column index), so the rank
 * streams its own columns (sketch against rows [j0, j0 + m) of Omega_k of the full problem, power
 * steps, shrink) and `allreduce` sums the n_k x l_k Y after every streaming pass (float64; `root`
 * != 0 on exactly one rank, which applies -alpha Q once); the small solves then run redundantly and
 * bit-identically everywhere.  Before mode d the rank's shrunk slab is placed at its rows of the
 * mode-d unfolding and all-reduced (float32, zero elsewhere), and mode d plus the core run
 * redundantly.  Outputs as rtk_solve, identical on every rank.  The tensor is split, not
 * replicated: each GPU holds 1 / world of it.  l_k <= 64 for k < d (RTK_ERR_ARG otherwise);
 * ws: rtk_workspace_bytes_shard; NULL ws allocates with cudaMallocAsync. */
RTK_API int rtk_rsthosvd_shard(const rtk_options* opt, const float* A_slab, const int64_t* dims, int32_t d,
                               int64_t last_begin, int64_t last_count, int32_t root, const int32_t* ranks,
                               int32_t p, int32_t q, uint64_t seed, float* const* U, float* core, void* ws,
                               size_t ws_bytes, void* stream, rtk_allreduce_fn allreduce, void* ctx);
RTK_API size_t rtk_workspace_bytes_shard(const rtk_options* opt, const int64_t* dims, int32_t d,
                                         int64_t last_count, const int32_t* ranks, int32_t p, int32_t q);

/* Workspace bytes for rtk_solve with these options (NULL -> ST-HOSVD defaults); 0 on error. */
RTK_API size_t rtk_workspace_bytes_ex(const rtk_options* opt, const int64_t* dims, int32_t d,
                                      const int32_t* ranks, int32_t p, int32_t q);

/* Test hook: rows [row0, row0+rows) of Omega_mode (l columns) in RTK-GAUSS-2,
 * written row-major to the DEVICE buffer out[(j-row0)*l + c] (float32). */
RTK_API int rtk_omega(uint64_t seed, int32_t mode, int64_t row0, int64_t rows, int32_t l, float* out,
              void* stream);

/* Test hook: rows [row0, row0+rows) x l of mode `mode`'s sketch Omega_mode of type `kind` (as
 * rtk_options.omega) for the mode-`mode` unfolding of a tensor with extents dims[0..d-1] (host;
 * for ST modes the CURRENT extents r_1..r_{k-1}, n_k..n_d), row-major to the DEVICE buffer
 * out[(j-row0)*l + c].  kind 0 ignores dims (rtk_omega).  RTK_ERR_ARG on bad arguments or
 * row0 + rows > prod_{j != mode} dims[j]; allocates its Khatri-Rao factor scratch with
 * cudaMallocAsync on `stream`. */
RTK_API int rtk_sketch(int32_t kind, uint64_t seed, int32_t mode, const int64_t* dims, int32_t d, int64_t row0,
                       int64_t rows, int32_t l, float* out, void* stream);

/* Test hook: one fused power step Y = M (M^T Q) on the column-major n x m matrix M (ld)
 * with Q (n x l, column-major, ld n; device, float32); Y (n x l, column-major fp64, device).
 * No shift, no orthonormalisation: exercises the streaming kernel alone. */
RTK_API int rtk_power_step(const float* M, int64_t n, int64_t m, int64_t ld, const float* Q, int32_t l,
                   double* Y, void* stream);

/* Device-time profile of the library's own launches (bench / roofline evidence).
 * Between rtk_profile_begin() and rtk_profile_end() every streaming-kernel launch
 * (and every per-step small-solve sequence) is bracketed by CUDA events on the
 * launching stream; rtk_profile_end() synchronises those events and reports the
 * summed milliseconds and counts by (kind, mode), plus the number of kernels the
 * library launched.  kind: 0 sketch tile, 1 power-step tile, 2 shrink tile,
 * 3 small solves (reduce..apply2 of one step).  mode: 0-based, < 8. */
typedef struct rtk_prof_stats {
  double ms[4][8];
  int32_t count[4][8];
  int64_t launches;
} rtk_prof_stats;
RTK_API int rtk_profile_begin(void);
RTK_API int rtk_profile_end(rtk_prof_stats* out);

/* Diagnostics: when dev_buf (device, 8*8*16 doubles) is non-NULL, every l <= 64 small-solve
 * launch of later calls writes its phase clock counts to dev_buf[((mode*8)+step)*16 + ...]
 * (SM cycles, CTA 0 of the cluster).  NULL disables.  Not needed for normal use. */
RTK_API int rtk_debug_step_clocks(void* dev_buf);

/* Thread-local message for the last non-zero status. */
RTK_API const char* rtk_last_error(void);

/* Library version string, "rtucker <semver> sm_100a". */
RTK_API const char* rtk_version(void);

#ifdef __cplusplus
}
#endif

#endif /* RTUCKER_H */
