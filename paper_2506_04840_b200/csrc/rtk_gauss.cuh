// rtk_gauss.cuh -- device implementation of the RTK-GAUSS-2 sketch stream.
//
// Omega_k(j, c) for the standard Gaussian sketch of Alg. 3 / Alg. 4 line 3
// ("standard Gaussian matrix" PAPER.md:96).  Written from
// the DESIGN.md specification, independently of the oracle: Philox4x32-10
// (Salmon et al. 2011) on counter (c/4, lo32(j), hi32(j), k) and key
// (lo32(seed), hi32(seed)), then a Box-Muller pair per two outputs whose ln,
// sin, cos use only correctly rounded, never fused binary32 + - * / sqrt
// (__fadd_rn / __fmul_rn / __fdiv_rn / __fsqrt_rn) in the specified order.
// Bit-identical to the spec by construction; tests/test_gpu_kernels.py checks
// it against the oracle.
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

// ---- spec constants (binary32 bit patterns, DESIGN.md RTK-GAUSS-2) ------------
__device__ __forceinline__ float f32b(uint32_t b) { return __uint_as_float(b); }
constexpr uint32_t kLn2Hi = 0x3F317200u;   // 0.693145751953125
constexpr uint32_t kLn2Lo = 0x35BFBE8Eu;
constexpr uint32_t kSqrt2 = 0x3FB504F3u;
constexpr uint32_t kPiO2 = 0x3FC90FDBu;
// correctly rounded binary32 of ln: 1/(2k+1), k = 0..4;  sin: (-1)^k/(2k+1)!, k = 0..4;
// cos: (-1)^k/(2k)!, k = 0..5
__device__ __forceinline__ float log_c(int k) {
  return f32b(k == 0 ? 0x3F800000u : k == 1 ? 0x3EAAAAABu : k == 2 ? 0x3E4CCCCDu : k == 3 ? 0x3E124925u : 0x3DE38E39u);
}
__device__ __forceinline__ float sin_c(int k) {
  return f32b(k == 0 ? 0x3F800000u : k == 1 ? 0xBE2AAAABu : k == 2 ? 0x3C088889u : k == 3 ? 0xB9500D01u : 0x3638EF1Du);
}
__device__ __forceinline__ float cos_c(int k) {
  return f32b(k == 0 ? 0x3F800000u : k == 1 ? 0xBF000000u : k == 2 ? 0x3D2AAAABu : k == 3 ? 0xBAB60B61u
              : k == 4 ? 0x37D00D01u : 0xB493F27Eu);
}
// odd integer v = 2(x>>9)+1 in [1, 2^24); u = v * 2^-24 (exact in binary32)
__device__ __forceinline__ uint32_t odd24(uint32_t x) { return ((x >> 9) << 1) | 1u; }
// ln(u), u = (2(x>>9)+1) 2^-24: f = v 2^-e in [1, 2) (halved above sqrt 2), s = (f-1)/(f+1),
// 2 s Horner(z = s^2), ln u = n LN2_HI + (n LN2_LO + lnf), n = e - 24; correctly rounded binary32
// operations in the spec's order, never fused
__device__ __forceinline__ float log_u(uint32_t x) {
  const uint32_t v = odd24(x);
  int e = 31 - __clz(v);
  float f = __fmul_rn((float)v, __int_as_float((127 - e) << 23));   // exact: v < 2^24, 2^-e normal
  if (f > f32b(kSqrt2)) {
    f = __fmul_rn(f, 0.5f);
    e += 1;
  }
  const float s = __fdiv_rn(__fadd_rn(f, -1.0f), __fadd_rn(f, 1.0f));
  const float z = __fmul_rn(s, s);
  float p = log_c(4);
#pragma unroll
  for (int k = 3; k >= 0; --k) p = __fadd_rn(__fmul_rn(p, z), log_c(k));
  const float lnf = __fmul_rn(__fmul_rn(2.0f, s), p);
  const float n = (float)(e - 24);
  return __fadd_rn(__fmul_rn(n, f32b(kLn2Hi)), __fadd_rn(__fmul_rn(n, f32b(kLn2Lo)), lnf));
}
// (sin, cos)(2 pi u): quadrant w >> 22, reduced t = (w mod 2^22) 2^-22, folded at 1/2
__device__ __forceinline__ void sincos_2pi_u(uint32_t x, float& so, float& co) {
  const uint32_t w = odd24(x);
  const uint32_t qd = w >> 22;
  const uint32_t rem = w & ((1u << 22) - 1u);
  const float t = __fmul_rn((float)rem, 0x1p-22f);
  const bool low = rem < (1u << 21);
  const float xr = __fmul_rn(low ? t : __fadd_rn(1.0f, -t), f32b(kPiO2));
  const float y = __fmul_rn(xr, xr);
  float ps = sin_c(4);
#pragma unroll
  for (int k = 3; k >= 0; --k) ps = __fadd_rn(__fmul_rn(ps, y), sin_c(k));
  const float sx = __fmul_rn(xr, ps);
  float pc = cos_c(5);
#pragma unroll
  for (int k = 4; k >= 0; --k) pc = __fadd_rn(__fmul_rn(pc, y), cos_c(k));
  const float S = low ? sx : pc;
  const float C = low ? pc : sx;
  switch (qd) {
    case 0: so = S; co = C; break;
    case 1: so = C; co = -S; break;
    case 2: so = -S; co = -C; break;
    default: so = -C; co = S; break;
  }
}
// Box-Muller pair from (xa, xb): (r cos, r sin), r = sqrt(-2 ln u_a), binary32
__device__ __forceinline__ float2 box_muller(uint32_t xa, uint32_t xb) {
  const float r = __fsqrt_rn(__fmul_rn(-2.0f, log_u(xa)));
  float s, c;
  sincos_2pi_u(xb, s, c);
  return make_float2(__fmul_rn(r, c), __fmul_rn(r, s));
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
// the Appendix D types, rtk_omega.cu) or RTK-GAUSS-2 generated in place (om == nullptr)
__device__ __forceinline__ float2 sketch_pair(const float* om, int l, uint64_t seed, uint32_t mode, uint64_t j,
                                              int c2) {
  if (om) {
    const float* p = om + j * (uint64_t)l + c2;
    return make_float2(p[0], c2 + 1 < l ? p[1] : 0.f);
  }
  return omega_pair(seed, mode, j, (uint32_t)(c2 >> 2), (c2 >> 1) & 1);
}

}  // namespace rtk
