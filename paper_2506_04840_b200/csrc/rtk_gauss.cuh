// rtk_gauss.cuh -- device implementation of the RTK-GAUSS-1 sketch stream.
//
// Omega_k(j, c) for the standard Gaussian sketch of Alg. 3 / Alg. 4 line 3
// ("standard Gaussian matrix" PAPER.md:96).  Written from
// the DESIGN.md specification, independently of the oracle: Philox4x32-10
// (Salmon et al. 2011) on counter (c/4, lo32(j), hi32(j), k) and key
// (lo32(seed), hi32(seed)), then a Box-Muller pair per two outputs whose ln,
// sin, cos use only correctly rounded, never fused binary64 + - * / sqrt
// (__dadd_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn) in the specified order, and
// a final round-to-nearest to float32.  Bit-identical to the spec by
// construction; tests/test_gpu_omega.py checks it against the oracle.
#pragma once
#include <cstdint>

namespace rtk {

__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    if (r < 9) {
      k.x += 0x9E3779B9u;
      k.y += 0xBB67AE85u;
    }
  }
  return c;
}

// ---- spec constants -------------------------------------------------------
constexpr double kLn2Hi = 0x1.62e42fee00000p-1;
constexpr double kLn2Lo = 0x1.a39ef35793c76p-33;
constexpr double kSqrt2 = 0x1.6a09e667f3bcdp+0;
constexpr double kPiO2 = 0x1.921fb54442d18p+0;

// Spec coefficients, written as correctly rounded quotients of exact integers
// (every factorial below is < 2^53):  ln: c_k = 1/(2k+1), k = 0..11;
// sin: (-1)^k/(2k+1)!, k = 0..8;  cos: (-1)^k/(2k)!, k = 0..9.
__host__ __device__ constexpr double log_c(int k) {
  return k == 0 ? 1.0 : k == 1 ? 1.0 / 3.0 : k == 2 ? 1.0 / 5.0 : k == 3 ? 1.0 / 7.0
       : k == 4 ? 1.0 / 9.0 : k == 5 ? 1.0 / 11.0 : k == 6 ? 1.0 / 13.0 : k == 7 ? 1.0 / 15.0
       : k == 8 ? 1.0 / 17.0 : k == 9 ? 1.0 / 19.0 : k == 10 ? 1.0 / 21.0 : 1.0 / 23.0;
}
__host__ __device__ constexpr double sin_c(int k) {
  return k == 0 ? 1.0 : k == 1 ? -1.0 / 6.0 : k == 2 ? 1.0 / 120.0 : k == 3 ? -1.0 / 5040.0
       : k == 4 ? 1.0 / 362880.0 : k == 5 ? -1.0 / 39916800.0 : k == 6 ? 1.0 / 6227020800.0
       : k == 7 ? -1.0 / 1307674368000.0 : 1.0 / 355687428096000.0;
}
__host__ __device__ constexpr double cos_c(int k) {
  return k == 0 ? 1.0 : k == 1 ? -1.0 / 2.0 : k == 2 ? 1.0 / 24.0 : k == 3 ? -1.0 / 720.0
       : k == 4 ? 1.0 / 40320.0 : k == 5 ? -1.0 / 3628800.0 : k == 6 ? 1.0 / 479001600.0
       : k == 7 ? -1.0 / 87178291200.0 : k == 8 ? 1.0 / 20922789888000.0
       : -1.0 / 6402373705728000.0;
}

// odd integer v = 2(x>>8)+1 in [1, 2^25); u = v * 2^-25
__device__ __forceinline__ uint32_t odd25(uint32_t x) { return ((x >> 8) << 1) | 1u; }

__device__ __forceinline__ double pow2i(int e) {  // exact 2^e for |e| < 1000
  return __longlong_as_double((long long)(1023 + e) << 52);
}

// ln(u), u = ((x>>8)+0.5) 2^-24
__device__ __forceinline__ double log_u(uint32_t x) {
  const uint32_t v = odd25(x);
  int e = 31 - __clz(v);
  double f = __dmul_rn((double)v, pow2i(-e));
  if (f > kSqrt2) {
    f = __dmul_rn(f, 0.5);
    e += 1;
  }
  const double s = __ddiv_rn(__dadd_rn(f, -1.0), __dadd_rn(f, 1.0));
  const double z = __dmul_rn(s, s);
  double p = log_c(11);
#pragma unroll
  for (int k = 10; k >= 0; --k) p = __dadd_rn(__dmul_rn(p, z), log_c(k));
  const double lnf = __dmul_rn(__dmul_rn(2.0, s), p);
  const double n = (double)(e - 25);
  return __dadd_rn(__dmul_rn(n, kLn2Hi), __dadd_rn(__dmul_rn(n, kLn2Lo), lnf));
}

// (sin, cos)(2 pi u)
__device__ __forceinline__ void sincos_2pi_u(uint32_t x, double& so, double& co) {
  const uint32_t w = odd25(x);
  const uint32_t qd = w >> 23;
  const uint32_t rem = w & ((1u << 23) - 1u);
  const double t = __dmul_rn((double)rem, 0x1p-23);
  const bool low = rem < (1u << 22);
  const double xr = __dmul_rn(low ? t : __dadd_rn(1.0, -t), kPiO2);
  const double y = __dmul_rn(xr, xr);
  double ps = sin_c(8);
#pragma unroll
  for (int k = 7; k >= 0; --k) ps = __dadd_rn(__dmul_rn(ps, y), sin_c(k));
  const double sx = __dmul_rn(xr, ps);
  double pc = cos_c(9);
#pragma unroll
  for (int k = 8; k >= 0; --k) pc = __dadd_rn(__dmul_rn(pc, y), cos_c(k));
  const double S = low ? sx : pc;
  const double C = low ? pc : sx;
  switch (qd) {
    case 0: so = S; co = C; break;
    case 1: so = C; co = -S; break;
    case 2: so = -S; co = -C; break;
    default: so = -C; co = S; break;
  }
}

// Box-Muller pair from (xa, xb) -> float32 (z0, z1)
__device__ __forceinline__ float2 box_muller(uint32_t xa, uint32_t xb) {
  const double r = __dsqrt_rn(__dmul_rn(-2.0, log_u(xa)));
  double s, c;
  sincos_2pi_u(xb, s, c);
  return make_float2(__double2float_rn(__dmul_rn(r, c)), __double2float_rn(__dmul_rn(r, s)));
}

// Philox block for (seed, mode, row j, column quad c4): the 4 raw words
__device__ __forceinline__ uint4 omega_bits(uint64_t seed, uint32_t mode, uint64_t j, uint32_t c4) {
  return philox4x32_10(make_uint4(c4, (uint32_t)j, (uint32_t)(j >> 32), mode),
                       make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
}

// Omega(j, 4*c4 + 2*half + {0,1}) : one Box-Muller pair
__device__ __forceinline__ float2 omega_pair(uint64_t seed, uint32_t mode, uint64_t j, uint32_t c4,
                                             int half) {
  const uint4 x = omega_bits(seed, mode, j, c4);
  return half ? box_muller(x.z, x.w) : box_muller(x.x, x.y);
}

// RTK-UNIF-1 value 2u - 1 = (2 (x >> 8) + 1 - 2^24) 2^-24, exact in binary32
__device__ __forceinline__ float unif_sym(uint32_t x) {
  return (float)((int)((x >> 8) << 1) + 1 - (1 << 24)) * 5.9604644775390625e-08f;
}

// Sketch columns (c2, c2 + 1) of row j (c2 even): from a materialised Omega_k ([m][l] row-major,
// the Appendix D types, rtk_omega.cu) or RTK-GAUSS-1 generated in place (om == nullptr)
__device__ __forceinline__ float2 sketch_pair(const float* om, int l, uint64_t seed, uint32_t mode, uint64_t j,
                                              int c2) {
  if (om) {
    const float* p = om + j * (uint64_t)l + c2;
    return make_float2(p[0], c2 + 1 < l ? p[1] : 0.f);
  }
  return omega_pair(seed, mode, j, (uint32_t)(c2 >> 2), (c2 >> 1) & 1);
}

}  // namespace rtk
