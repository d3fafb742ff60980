// rtk_internal.h -- host-side plumbing shared by the CUDA translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

namespace rtk {

// Matrix view of a mode-k unfolding M (n x m), column j = p + P*s  (p < P, s < S):
// element (i, j) at base[p*sp + i*si + s*ss].  A column-major matrix with leading
// dimension ld is the view P = 1, S = m, si = 1, ss = ld.
struct View {
  const float* base = nullptr;
  int64_t P = 1, S = 1;
  int64_t sp = 1, si = 1, ss = 1;
  int n = 0;
  int64_t m() const { return P * S; }
};

enum TileOp { OP_SKETCH = 0, OP_POWER = 1, OP_SHRINK = 2 };

// Tile-kernel configuration chosen by the planner (rtk_plan.cu).
struct TilePlan {
  int R = 4;       // rows per thread
  int TC = 8;      // columns per thread
  int NRG = 0;     // row groups (n_rows = R*NRG)
  int NCG = 1;     // column groups per chunk (power of two, divides 32)
  int LC = 8;      // columns per chunk = NCG*TC
  int nchunks = 1;
  int NT = 32;     // threads per CTA (multiple of 32, >= NRG_pad*NCG)
  int b = 16;      // tile width (columns)
  int pitch = 0;   // SMEM column pitch (floats)
  int G = 1;       // CTAs per chunk
  int64_t ntiles = 0;
  size_t smem = 0;
  int n_rows() const { return R * NRG; }
  int ltot() const { return nchunks * LC; }
};

struct TileLaunch {
  View v;
  TileOp op;
  TilePlan tp;
  int l = 0;                  // valid columns (sketch l or shrink r)
  const float* Q = nullptr;   // POWER: fp32 Q [c][i] (ld qld); SHRINK: U n x r col-major (ld qld)
  int qld = 0;
  float* Ypart = nullptr;     // [G][ltot][n_rows]
  uint64_t seed = 0;
  uint32_t mode = 0;
  const float* om = nullptr;  // SKETCH: materialised Omega_k [m][l] (Appendix D types) or nullptr
  float* out = nullptr;       // SHRINK destination
  int64_t Rprev = 1, nnext = 1, ldnext = 1;
};

TilePlan plan_tile(const View& v, int l, TileOp op, int num_sms);
cudaError_t launch_tile(const TileLaunch& L, cudaStream_t st);

// ---- small-solve kernels (rtk_small.cu) -------------------------------------
struct ModeBufs {
  int n = 0, l = 0, r = 0, G = 1, ltot = 0, n_rows = 0;
  float* Ypart = nullptr;   // [G][ltot][n_rows]
  double* Y = nullptr;      // [l][n]
  double* Q1 = nullptr;     // [l][n]
  double* Qd = nullptr;     // [l][n]  fp64 master basis
  float* Qs = nullptr;      // [l][n]  fp32 shadow for the stream
  double* gpart = nullptr;  // [nblk][l][l]
  int nblk = 0;
  double* T = nullptr;      // [l][l] (column-major)
  double* lam = nullptr;    // [l]
  double* alpha = nullptr;  // device scalar for this mode
  double* trace = nullptr;  // [q] alpha trace
  double* sigma = nullptr;  // [128] final sigma estimates
  int* status = nullptr;    // [0]=numeric, [1]=fallback count, [2]=q_used, [3]=pve_stop
  double* sighat = nullptr; // [l] B.1 sigma-hat
  // cluster solver (rtk_solve.cu, l <= 64)
  double* g2part = nullptr; // [8][np] second-pass Gram partials
  double* gsum = nullptr;   // [np]
  double* amax = nullptr;   // [8][128] sign-pin argmax exchange
  double* lamx = nullptr;   // [64] eigenvalues exchanged across the cluster (final / B.1 steps)
  unsigned int* gbar = nullptr;   // [2] step-kernel grid barrier (zeroed at mode start)
};

cudaError_t launch_reduce_gram(const ModeBufs& B, bool power, cudaStream_t st);
cudaError_t launch_eig(const ModeBufs& B, int step, int q, bool shift, double pve_tol,
                       cudaStream_t st);
cudaError_t launch_apply(const ModeBufs& B, uint64_t seed, uint32_t mode, int step,
                         cudaStream_t st);
cudaError_t launch_chol(const ModeBufs& B, cudaStream_t st);
cudaError_t launch_apply2(const ModeBufs& B, cudaStream_t st);
cudaError_t launch_final_u(const ModeBufs& B, float* U, cudaStream_t st);
cudaError_t launch_omega(uint64_t seed, uint32_t mode, int64_t row0, int64_t rows, int l,
                         float* out, cudaStream_t st);
cudaError_t launch_sum_partials(const float* Ypart, int G, int ltot, int n_rows, int n, int l,
                                double* Y, cudaStream_t st);

int num_sms();
bool pdl_enabled();   // programmatic dependent launch for the per-step kernels (RTK_PDL=0: off)

// ---- cluster small solver (rtk_solve.cu), l <= 64 ------------------------------
constexpr int kSolveLMax = 64;
extern double* g_step_dbg;
size_t solve_gpart_doubles(int n, int l);      // Gram partials of reduce_gram_kernel
// gmode 0: Y = sum of the partials (- alpha Q) and the Gram partials; 1: Y only; 2: the Gram
// partials of the Y already in B.Y (multi-GPU shards all-reduce Y in between)
cudaError_t launch_reduce_gram2(const ModeBufs& B, bool power, cudaStream_t st, const int* stop = nullptr,
                                int gmode = 0);
cudaError_t launch_step(const ModeBufs& B, int step, int q, bool shift, float* U, uint64_t seed, uint32_t mode1,
                        float* planes, int pN, int pld, bool defer_alpha, double pve_tol, cudaStream_t st,
                        bool pin_q = false, bool planes16 = false);
cudaError_t launch_alpha(const ModeBufs& B, int step, bool shift, cudaStream_t st);
// Alg. A.2 lines 14-15 (rtk_solve.cu): deterministic ST-HOSVD of the l_1 x ... x l_d fp32 tensor B
// and U_k = Q_k V_k (sign-pinned); g0/g1 hold prod(l) doubles each, gram/V 64*64 doubles.
cudaError_t a2_finish(const float* B, int d, const int* l, const int* r, const int64_t* n, double* const* Qk,
                      double* g0, double* g1, double* gram, double* V, float* const* U, float* core, cudaStream_t st);

// ---- tcgen05 3xTF32 path (rtk_tc.cu) -------------------------------------------
int tc_npad(int l);                                   // l padded to the UMMA N (16..64), 0 if > 64
int tc_op2_grid(const View& v, int G);   // split-K grid of tc_op2 (<= K chunks)
bool tc_supported(const View& v, int l);              // contiguous column-major view, sm_100
cudaError_t tc_split(const double* q64, const float* q32, int n, int l, float* planes, cudaStream_t st);
cudaError_t tc_op1(const View& v, int l, const float* planes, float* W, int64_t ldw, bool shrink, float* out,
                   int64_t Rprev, int64_t nnext, int64_t ldnext, cudaStream_t st, int max_ctas = 0);
cudaError_t tc_op2(const View& v, int l, const float* W, int64_t ldw, bool sketch, uint64_t seed, uint32_t mode,
                   float* Ypart, int G, cudaStream_t st, const float* om = nullptr, float* xmax = nullptr);

// The fp16 two-plane power step and its scale (rtk_fused2.cu): xmax_in = max|M| of the
// unfolding (device) selects it for a power step (planes are then fp16 [2N][pld], pld % 8 == 0, scaled
// by 2^15); xmax_out receives (atomicMax) max|M| from a pair sketch, or the max of the entries a pair
// shrink writes (the next unfolding's max|M|).
struct PairScale {
  const float* xmax_in = nullptr;
  float* xmax_out = nullptr;
  bool wrote = false;   // set by pair_power when its launch writes xmax_out
};

// ---- fused single-pass power step (rtk_fused.cu) -----------------------------------
int fused_cluster(int n);
bool fused_sketch_gen(const float* om);   // fused sketch generates Omega in-kernel (no planes kernel)
bool fused_supported(const View& v, int l);
size_t fused_ypart_floats(const View& v, int l, int grid);
cudaError_t fused_power(const View& v, int l, const float* planes, int pld, bool sketch, uint64_t seed,
                        uint32_t mode1, float* Ypart, int grid, int* G_out, int* rows_out, cudaStream_t st,
                        float* shrink_out = nullptr, int64_t Rprev = 1, int64_t nnext = 1, int64_t ldnext = 1,
                        const int* stop = nullptr, const float* om = nullptr, PairScale* ps = nullptr);

// ---- fused power step on a CTA pair, tcgen05 cta_group::2 (rtk_fused2.cu) ---------------
bool pair_supported(const View& v, int l);
size_t pair_ypart_floats(const View& v, int l, int grid);
// shrink_out != nullptr: the mode shrink G x_k U_k^T instead (op1 only, planes = U's, l = r_k),
// written as the next unfolding (Rprev, nnext, ldnext as in TileLaunch).  sketch: Y = M Omega_k
// (op2 only) with planes = the Omega planes [2N][pld >= m] of omega_planes_kernel.
// test hook support (rtk_power_step with RTK_POWER_F16=1): max|M| into xmax and the fp16 planes of
// the fp32 Q (n x l, column-major) as the step kernel writes them (2^15 q = hi + lo)
cudaError_t pair_prepare16(const View& v, const float* Q, int l, int N, int pld, float* planes, float* xmax,
                           cudaStream_t st);
cudaError_t pair_power(const View& v, int l, const float* planes, int pld, float* Ypart, int grid, int* G_out,
                       int* rows_out, cudaStream_t st, const int* stop, float* shrink_out = nullptr,
                       int64_t Rprev = 1, int64_t nnext = 1, int64_t ldnext = 1, bool sketch = false,
                       PairScale* ps = nullptr);

// ---- Appendix D sketch types (rtk_omega.cu) ------------------------------------------
// Materialise Omega_k rows [row0, row0 + rows) x l (row-major [j][l]) of the given type for the
// mode-mode1 unfolding of a tensor with extents dims[0..d-1]; tabs: scratch for the Khatri-Rao
// factors (sum_{m != k} dims[m] * l floats).  kind: 1 uniform, 2 KR-Gaussian, 3 KR-uniform.
cudaError_t sketch_materialize(int kind, uint64_t seed, int mode1, const int64_t* dims, int d, int64_t row0,
                               int64_t rows, int l, float* tabs, float* out, cudaStream_t st);
size_t sketch_tab_floats(const int64_t* dims, int d, int mode1, int l);

}  // namespace rtk
