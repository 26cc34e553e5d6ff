// pc_intfp.cuh -- IEEE binary64 companding arithmetic on the integer pipe, bit-identical to
// the FP64 instructions it replaces (round-to-nearest-even products and quotients of positive
// normal doubles, round half away from zero).
//
// Why: on sm_100a the FP64 tensor-core instructions (DMMA) and the FP64 ALU instructions share
// the SM sub-partition's FP64 pipe, and while two warps of a sub-partition issue DMMAs back to
// back, an FP64 instruction of any other warp on it waits until they pause -- measured in the
// persistent kernel (tools/tiled_timeline.py, profiles/r02/): the first FP64 instruction of a
// producer warp (the IEEE division c_s = Q / peak) waited 3.6-9.5 us, while its integer loads,
// maxima and shuffles before it took 0.8 us.  The producer warps' companding (Eq. (2)),
// packing (Eqs. (4)/(7)) and the block's c_s / (c_s c_k)^-1 (Eq. (16)) are
// therefore computed here with integer instructions only.
//
// Every function returns false (and leaves its output unspecified) for operands outside its
// domain -- zeros where not stated, subnormals, infinities, NaNs, results that would not be
// normal -- and the caller then takes the FP64 instruction (never the case for the companding
// of real signals; kept so the result is the FP64 one for every input).
// Host-compilable (tests/test_intfp.py checks every function against the host's FP64
// arithmetic on millions of operands, including exact ties).
#pragma once
#include <cstdint>

#ifndef __CUDACC__
#define PC_HD inline
#else
#define PC_HD __host__ __device__ __forceinline__
#endif

namespace pc {
namespace ifp {

constexpr uint64_t kFrac = 0x000fffffffffffffull, kHid = 0x0010000000000000ull, kSign = 0x8000000000000000ull;

PC_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}
PC_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __clzll((long long)x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}

// Positive normal double -> (biased exponent, 53-bit significand); false for 0, subnormal, inf, NaN.
PC_HD bool split_pos(uint64_t a, int& e, uint64_t& m) {
  e = (int)((a >> 52) & 0x7ff);
  m = (a & kFrac) | kHid;
  return e != 0 && e != 0x7ff && (a >> 63) == 0;
}

// RN(a * b) for positive normal a, b with a normal result.  P = ma mb in [2^104, 2^106): the
// 53 leading bits, ties to even.
PC_HD bool dmul_rn_pos(uint64_t a, uint64_t b, uint64_t& r) {
  int ea, eb;
  uint64_t ma, mb;
  if (!split_pos(a, ea, ma) || !split_pos(b, eb, mb)) return false;
  const uint64_t lo = ma * mb, hi = mulhi64(ma, mb);
  const int top = (int)((hi >> 41) & 1u);             // P >= 2^105
  const int s = 52 + top;
  uint64_t m = (hi << (64 - s)) | (lo >> s);
  const uint64_t rem = lo & ((1ull << s) - 1), half = 1ull << (s - 1);
  m += (rem > half || (rem == half && (m & 1u))) ? 1u : 0u;
  int e = ea + eb - 1023 + top;
  if (m >> 53) {                                      // rounded up to 2^53
    m >>= 1;
    ++e;
  }
  if (e <= 0 || e >= 0x7ff) return false;
  r = ((uint64_t)e << 52) | (m & kFrac);
  return true;
}

// RN(a / b) for positive normal a, b with a normal result.  ma is scaled to [mb, 2 mb); the
// quotient floor(ma 2^52 / mb) comes from a reciprocal R ~ 2^116 / mb (an FP32 seed, two
// integer Newton steps), then the exact remainder corrects it and decides the rounding (ties to
// even).  About a hundred integer instructions with a short dependency chain (a bit-serial
// restoring division took ~1.7 us per call next to the DMMA warps).
PC_HD bool ddiv_rn_pos(uint64_t a, uint64_t b, uint64_t& r) {
  typedef unsigned __int128 u128;
  typedef __int128 i128;
  int ea, eb;
  uint64_t ma, mb;
  if (!split_pos(a, ea, ma) || !split_pos(b, eb, mb)) return false;
  int e = ea - eb + 1023;
  if (ma < mb) {
    ma <<= 1;
    --e;
  }
  uint64_t q;
  if (mb == kHid) {
    q = ma;                                           // mb = 2^52: the quotient is ma itself
  } else {
    // seed: 2^29 / ((mb >> 29) + 1) in FP32 (exact operand <= 2^24; the +1 keeps R0 below 2^64),
    // R0 = seed * 2^87 in (2^62, 2^64)
    const float rf = 1.0f / (float)((uint32_t)(mb >> 29) + 1u);
    uint64_t R;
    {
      // rf = 2^(E - 150) * (2^23 + f): R0 = (2^23 + f) << (E - 150 + 87)
      uint32_t fb;
#if defined(__CUDA_ARCH__)
      fb = (uint32_t)__float_as_int(rf);
#else
      __builtin_memcpy(&fb, &rf, 4);
#endif
      const int E = (int)((fb >> 23) & 0xff);
      const uint64_t mf = (uint64_t)((fb & 0x7fffffu) | 0x800000u);
      const int sh = E - 63;                          // = 87 - 150 + E
      R = sh >= 0 ? mf << sh : mf >> -sh;
    }
#pragma unroll
    for (int it = 0; it < 2; ++it) {                  // R += R (2^116 - mb R) / 2^116
      const i128 err = (i128)((u128)1 << 116) - (i128)((u128)mb * R);   // |err| < 2^96
      const i128 e52 = err >> 52;                     // |e52| < 2^44
      R = (uint64_t)((i128)R + (((i128)R * e52) >> 64));
    }
    q = (uint64_t)(((u128)ma * R) >> 64);            // floor(ma 2^52 / mb) - {0, 1, 2} or + 1
    i128 rem = ((i128)ma << 52) - (i128)((u128)q * mb);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      if (rem < 0) {
        --q;
        rem += mb;
      }
      if (rem >= (i128)mb) {
        ++q;
        rem -= mb;
      }
    }
    const uint64_t r2 = (uint64_t)rem << 1;           // rem < 2^53
    q += (r2 > mb || (r2 == mb && (q & 1u))) ? 1u : 0u;
  }
  if (q >> 53) {
    q >>= 1;
    ++e;
  }
  if (e <= 0 || e >= 0x7ff) return false;
  r = ((uint64_t)e << 52) | (q & kFrac);
  return true;
}

// Eq. (2): n = round(RN(c * x)), round half away from zero (C round()), c positive normal.
// neg0: the FP64 result is -0.0 (x < 0 rounding to zero).  |n| < 2^62.
PC_HD bool compand_int(uint64_t c, uint64_t x, long long& n, bool& neg0) {
  const bool neg = (x >> 63) != 0;
  const uint64_t ax = x & ~kSign;
  if (ax == 0) {
    n = 0;
    neg0 = neg;
    return true;
  }
  uint64_t p;
  if (!dmul_rn_pos(c, ax, p)) return false;
  const uint64_t m = (p & kFrac) | kHid;
  const int sh = 1075 - (int)(p >> 52);               // |RN(c x)| = m / 2^sh
  long long v;
  if (sh <= 0) {
    if (sh < -9) return false;                        // |c x| >= 2^62
    v = (long long)(m << -sh);
  } else if (sh >= 64) {
    v = 0;
  } else {
    v = (long long)((m + (1ull << (sh - 1))) >> sh);
  }
  n = neg ? -v : v;
  neg0 = neg && v == 0;
  return true;
}

// Index of the leading one of 0 < x < 2^23 through the FP32 add pipe (2^23 + x is exact; its
// exponent field minus that of 2^23 is 0 -- the difference 2^23 + x - 2^23 = x is exact and its
// exponent is msb(x)): no FLO / conversion instruction (those queue behind the DMMA warps).
PC_HD int msb23(uint32_t x) {
#if defined(__CUDA_ARCH__)
  const float f = __fsub_rn(__int_as_float(0x4B000000 | (int)x), 8388608.0f);
  return (int)(((uint32_t)__float_as_int(f) >> 23) & 0xff) - 127;
#else
  const uint32_t u = 0x4B000000u | x;
  float f;
  __builtin_memcpy(&f, &u, 4);
  f = f - 8388608.0f;
  uint32_t v;
  __builtin_memcpy(&v, &f, 4);
  return (int)((v >> 23) & 0xff) - 127;
#endif
}
// leading one of 0 < a < 2^69 (three 23-bit limbs)
PC_HD int msb_small(uint64_t a) {
  const uint32_t l2 = (uint32_t)(a >> 46), l1 = (uint32_t)(a >> 23) & 0x7fffffu, l0 = (uint32_t)a & 0x7fffffu;
  return l2 ? 46 + msb23(l2) : (l1 ? 23 + msb23(l1) : msb23(l0));
}
// n * 2^-e2 as binary64 bits, exact for |n| < 2^53 and a normal result; neg0 selects -0.0
// for n == 0 (the sign an FP64 Horner of negative zeros gives).
PC_HD uint64_t i2d_scaled(long long n, int e2, bool neg0) {
  if (n == 0) return neg0 ? kSign : 0ull;
  const uint64_t a = (uint64_t)(n < 0 ? -n : n);
  const int msb = msb_small(a);
  return ((uint64_t)(1023 + msb - e2) << 52) | ((a << (52 - msb)) & kFrac) | (n < 0 ? kSign : 0ull);
}

}  // namespace ifp
}  // namespace pc
