// quant_math.cuh -- per-element quantizer arithmetic for the sm_100a kernels.
//
// Semantics are those of the reference's double-precision scalar path
// (proj/include/lpsim/rounding.hpp, scalar_quant.hpp, quant_ops.cpp:33-115);
// the implementation is different: every element is handled in fp32 and
// 32-bit integer arithmetic that is exact for all finite inputs, so the
// kernels never touch the FP64 pipe or the conversion pipe beyond one FRND.
// Exactness arguments are in DESIGN.md §3 ("element math").
//
// The functions are __host__ __device__ so the same source is compiled for
// the CPU in the test build (tests/test_element_math.py sweeps it against the
// reference over millions of bit patterns). Builds must NOT use fast-math,
// -ftz=true or FMA contraction on float ops here (the kernels use explicit
// __fmul_rn/__fadd_rn on device).
#pragma once

#include <stdint.h>
#include <string.h>
#include <math.h>
#if !defined(__CUDA_ARCH__)
#include <fenv.h>
#endif

#if defined(__CUDACC__)
#define LPQ_HD __host__ __device__ __forceinline__
#else
#define LPQ_HD static inline
#endif

namespace lpq {

// RoundingMode order of proj/include/lpsim/formats.hpp:14-19.
enum Mode : int { kStochastic = 0, kNearestEven = 1, kNearestAway = 2,
                  kNearestZero = 3 };

LPQ_HD uint32_t f2u(float x) {
#if defined(__CUDA_ARCH__)
  return __float_as_uint(x);
#else
  uint32_t u;
  memcpy(&u, &x, 4);
  return u;
#endif
}

LPQ_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
  return __uint_as_float(u);
#else
  float x;
  memcpy(&x, &u, 4);
  return x;
#endif
}

LPQ_HD float fmul(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fmul_rn(a, b);
#else
  volatile float r = a * b;
  return r;
#endif
}

LPQ_HD float fadd(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fadd_rn(a, b);
#else
  volatile float r = a + b;
  return r;
#endif
}

LPQ_HD float fsub(float a, float b) {
#if defined(__CUDA_ARCH__)
  return __fsub_rn(a, b);
#else
  volatile float r = a - b;
  return r;
#endif
}

// u * 2^-24 - r rounded toward -inf, i.e. FFMA.RM(v, 2^-24, -r): one
// directed rounding of the exact value (v * 2^-24 is exact).
LPQ_HD float fma_rd_variate(uint32_t v, float r) {
#if defined(__CUDA_ARCH__)
  return __fmaf_rd(__uint2float_rn(v), 0x1p-24f, -r);
#else
  const int old = fegetround();
  fesetround(FE_DOWNWARD);
  volatile float vf = (float)v;
  volatile float out = fmaf(vf, 0x1p-24f, -r);
  fesetround(old);
  return out;
#endif
}

LPQ_HD float rint_f(float a) {
#if defined(__CUDA_ARCH__)
  return rintf(a);
#else
  return nearbyintf(a);
#endif
}

// Signed integer rounding of r for the two modes the streaming kernels
// specialise (rounding.hpp:27-37, 56-59):
//   NearestEven: rint(r)  (IEEE RNE; -0 may appear, callers add +0)
//   Stochastic : floor(r) + (u < r - floor(r)) == -floor(u - r), and with
//                s = RD(u - r) (a single round-toward-minus-infinity FFMA),
//                floor(s) == floor(u - r) exactly: if u - r lies in
//                (m, m + 1) for an integer m, RD keeps it in [m, m + 1)
//                because m is representable (|r| < 2^24 -- beyond that r is
//                an integer and RD(u - r) == -r).  One FFMA + one FRND
//                replace the fraction/compare sequence.
// r must be exact; flushed-to-zero r is the caller's business (see TINY).
template <int M>
LPQ_HD float round_signed(float r, uint32_t v) {
  if (M == kNearestEven) return rint_f(r);
  return -floorf(fma_rd_variate(v, r));
}

// ---- counter-based RNG: bit-identical to proj/include/lpsim/rng.hpp -------

LPQ_HD uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

LPQ_HD uint64_t stream_key(uint64_t seed, uint64_t call) {
  return mix64(mix64(seed) ^ call);
}

// The reference variate is float(mix64(key ^ i) >> 40) * 2^-24
// (rng.hpp:34-36).  Kernels keep it as the 24-bit integer v, u = v * 2^-24.
// (z ^ (z >> 31)) >> 40 == z >> 40, so the final xor-shift of the splitmix
// finalizer is dropped, and only the high word of the last product is formed.
// z = key ^ index (callers that know index % 4 == 0 form key ^ (index + q)
// as (key ^ index) ^ q without a 64-bit add).
LPQ_HD uint32_t variate24_z(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = z ^ (z >> 27);
  const uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  const uint32_t c_lo = 0x133111EBu, c_hi = 0x94D049BBu;
#if defined(__CUDA_ARCH__)
  const uint32_t top = __umulhi(lo, c_lo) + lo * c_hi + hi * c_lo;
#else
  const uint32_t top =
      (uint32_t)(((uint64_t)lo * c_lo) >> 32) + lo * c_hi + hi * c_lo;
#endif
  return top >> 8;
}

LPQ_HD uint32_t variate24(uint64_t key, uint64_t index) {
  return variate24_z(key ^ index);
}

LPQ_HD uint32_t umulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  return __umulhi(a, b);
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// Pipe-balanced form of variate24_z for the streaming kernels (identical
// result).  ncu showed the stochastic kernels ALU-pipe-bound (shifts, xors,
// compares all issue to the ALU pipe, multiplies to the FMA pipe), so the
// second xor-shift z ^= z >> 27 is formed with IMAD.HI/IMAD against the
// runtime multiplier m32 == 32 (a kernel argument, so ptxas cannot turn the
// multiplies back into shifts):  (z >> 27).lo = hi(lo*32) + hi*32,
// (z >> 27).hi = hi(hi*32).
LPQ_HD uint32_t variate24_zb(uint64_t z, uint32_t m32) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  uint32_t lo = (uint32_t)z, hi = (uint32_t)(z >> 32);
  const uint32_t slo = umulhi32(lo, m32) + hi * m32;
  const uint32_t shi = umulhi32(hi, m32);
  lo ^= slo;
  hi ^= shi;
  const uint32_t top = umulhi32(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu;
  return top >> 8;
}

LPQ_HD float variate_float(uint32_t v) { return (float)v * 0x1p-24f; }

// Runtime multipliers for the FMA-pipe forms of shifts/adds (kernel
// arguments, so ptxas cannot fold the multiplies back into SHF/IADD on the
// ALU pipe).
struct RngMul {
  uint32_t one;   // 1
  uint32_t m4;    // 4      (>> 30 as hi(x * 4))
  uint32_t m32;   // 32     (>> 27 as hi(x * 32))
  uint32_t m24;   // 2^24   (>> 8  as hi(x * 2^24))
  uint32_t m2;    // 2      (>> 31 as hi(x * 2))
  uint32_t neg1;  // 2^32-1 (-x as x * neg1)
};

LPQ_HD RngMul rng_mul() { return RngMul{1u, 4u, 32u, 1u << 24, 2u, 0xFFFFFFFFu}; }

LPQ_HD uint64_t mad_wide_u32(uint32_t a, uint32_t b, uint64_t c) {
#if defined(__CUDA_ARCH__)
  uint64_t d;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
#else
  return (uint64_t)a * b + c;
#endif
}

// FMA-pipe-heavy form of variate24_z for the ALU-bound quantizers (float,
// block): the 64-bit add, both xor-shifts and the final >> 8 run as
// IMAD/IMAD.HI/IMAD.WIDE, leaving 5 ALU ops (xors) per variate.
LPQ_HD uint32_t variate24_zf(uint64_t z, const RngMul& m) {
  // z += C0: (lo * 1 + C0) as a 64-bit IMAD.WIDE, then the high word
  const uint64_t t = mad_wide_u32((uint32_t)z, m.one, 0x9E3779B97F4A7C15ull);
  uint32_t lo = (uint32_t)t;
  uint32_t hi = (uint32_t)(z >> 32) * m.one + (uint32_t)(t >> 32);
  // z ^= z >> 30
  lo ^= umulhi32(lo, m.m4) + hi * m.m4;
  hi ^= umulhi32(hi, m.m4);
  // z *= C1
  const uint64_t w = mad_wide_u32(lo, 0x1CE4E5B9u, 0ull);
  hi = (uint32_t)(w >> 32) + lo * 0xBF58476Du + hi * 0x1CE4E5B9u;
  lo = (uint32_t)w;
  // z ^= z >> 27
  lo ^= umulhi32(lo, m.m32) + hi * m.m32;
  hi ^= umulhi32(hi, m.m32);
  const uint32_t top = umulhi32(lo, 0x133111EBu) + lo * 0x94D049BBu + hi * 0x133111EBu;
  return umulhi32(top, m.m24);  // top >> 8
}

// Four variates for the flat indices idx .. idx+3 with idx % 4 == 0 (the
// four lanes of a float4), sharing the work their hashes have in common.
// z_q = key ^ (idx + q) = (key ^ idx) ^ q, so z_q + C0 = w + j_q with
// w = ((key ^ idx) & ~3) + C0 and j_q = (key & 3) ^ q: unless the low word
// of w is within 3 of 2^32 (then the generic form runs), the four sums share
// their HIGH word.  That makes the high word of z ^= z >> 30 shared, and the
// hi * C1lo term of z *= C1 shared; per lane there remain one add, a funnel
// shift + xor, one IMAD.WIDE + one IMAD, and the unshared tail (>> 27 xor,
// the last product's high word).  Identical to variate24_z(key ^ (idx + q)).
template <int S>
LPQ_HD uint32_t funnel_r(uint32_t lo, uint32_t hi) {  // (hi:lo >> S).lo, one SHF.R.W
#if defined(__CUDA_ARCH__)
  return __funnelshift_r(lo, hi, S);
#else
  return (uint32_t)((((uint64_t)hi << 32) | lo) >> S);
#endif
}

// high word of a * b kept as its own IMAD.HI (no 64-bit addend pair, which
// costs a register move to zero its low half)
LPQ_HD uint32_t mulhi_sep(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
#else
  return (uint32_t)(((uint64_t)a * b) >> 32);
#endif
}

// TOP = true: out[q] is the variate's top word (variate = top >> 8, the low
// 8 bits arbitrary) for quant_float_bits_top, which folds the shift
template <bool TOP = false>
LPQ_HD void variate24_x4(uint64_t key, uint64_t idx, uint32_t m32,
                         uint32_t out[4]) {  // m32: the generic fallback's
  const uint64_t z0 = key ^ idx;
  const uint64_t w = (z0 & ~3ull) + 0x9E3779B97F4A7C15ull;
  const uint32_t wlo = (uint32_t)w, whi = (uint32_t)(w >> 32);
  const uint32_t kl = (uint32_t)key & 3u;
  if ((wlo & 0x3FFFFFFFu) > 0x3FFFFFFCu) {  // w + j_q may carry past bit 29
    for (int q = 0; q < 4; ++q) out[q] = variate24_zb(z0 ^ (uint64_t)q, m32) << (TOP ? 8 : 0);
    return;
  }
  const uint32_t h1 = whi ^ (whi >> 30);                   // shared
  const uint64_t hc = (uint64_t)(h1 * 0x1CE4E5B9u) << 32;  // shared hi*C1lo
  // (z >> 30).lo = (zlo >> 30) | (zhi << 2): with no carry past bit 29,
  // zlo >> 30 = wlo >> 30 for every lane, so the xor-shift word is shared
  const uint32_t c30 = (wlo >> 30) | (whi << 2);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t lo = (wlo + (kl ^ (uint32_t)q)) ^ c30;
    const uint64_t p = (uint64_t)lo * 0x1CE4E5B9u + hc;    // z *= C1
    uint32_t plo = (uint32_t)p;
    uint32_t phi = (uint32_t)(p >> 32) + lo * 0xBF58476Du;
    // z ^= z >> 27 as a funnel shift + shift (4 ALU instructions with the
    // xors; the IMAD.HI form of variate24_zb is one instruction longer, and
    // with the shared work gone this kernel is issue-bound, not ALU-bound:
    // C2 6645 -> 6873 GB/s, C3 stochastic 6101 -> 6409)
    const uint32_t slo = funnel_r<27>(plo, phi);
    const uint32_t shi = phi >> 27;
    plo ^= slo;
    phi ^= shi;
    const uint32_t top = mulhi_sep(plo, 0x133111EBu) + plo * 0x94D049BBu + phi * 0x133111EBu;
    out[q] = TOP ? top : top >> 8;
  }
}

// 3-input maximum that propagates NaN / 3-input minimum (NaN operands
// ignored): one FMNMX3 each
LPQ_HD float fmax3_nan(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
  float d;
  asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
#else
  if (a != a || b != b || c != c) return a + b + c;
  return fmaxf(fmaxf(a, b), c);
#endif
}
LPQ_HD float fmin3(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
  float d;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
#else
  return fminf(fminf(a, b), c);
#endif
}

// mad.lo.u32 against a runtime multiplier (RngMul::one): an add that issues
// on the FMA pipe as an IMAD instead of an ALU IADD3
LPQ_HD uint32_t mad_lo(uint32_t a, uint32_t b, uint32_t c) {
#if defined(__CUDA_ARCH__)
  uint32_t d;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
#else
  return a * b + c;
#endif
}

// variate24_x4 for the elementwise float kernels, returning the TOP words of
// the last product (variate = top >> 8; the low 8 bits are hash bits the
// caller ignores; quant_float_bits_top folds the >> 8 into its own shift).
// The xor-shifts are funnel shifts and the lane add a plain add; an
// FMA-leaning form (lane add as IMAD, >> 27 as IMAD.HI / IMAD against m.m32)
// measured slower once the >> 30 word was shared: C1 5030 -> 5300 GB/s with
// these, log-uniform 3840 -> 3990.  Identical variates to variate24_z.
LPQ_HD void variate24_x4_top(uint64_t key, uint64_t idx, const RngMul& m,
                             uint32_t out[4]) {
  const uint64_t z0 = key ^ idx;
  const uint64_t w = (z0 & ~3ull) + 0x9E3779B97F4A7C15ull;
  const uint32_t wlo = (uint32_t)w, whi = (uint32_t)(w >> 32);
  const uint32_t kl = (uint32_t)key & 3u;
  if ((wlo & 0x3FFFFFFFu) > 0x3FFFFFFCu) {  // w + j_q may carry past bit 29
    for (int q = 0; q < 4; ++q) out[q] = variate24_zb(z0 ^ (uint64_t)q, m.m32) << 8;
    return;
  }
  const uint32_t h1 = whi ^ (whi >> 30);                   // shared
  const uint64_t hc = (uint64_t)(h1 * 0x1CE4E5B9u) << 32;  // shared hi*C1lo
  const uint32_t c30 = (wlo >> 30) | (whi << 2);           // shared (variate24_x4)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t lo = (wlo + (kl ^ (uint32_t)q)) ^ c30;
    const uint64_t p = (uint64_t)lo * 0x1CE4E5B9u + hc;    // z *= C1
    uint32_t plo = (uint32_t)p;
    uint32_t phi = (uint32_t)(p >> 32) + lo * 0xBF58476Du;
    const uint32_t slo = funnel_r<27>(plo, phi);
    const uint32_t shi = phi >> 27;
    plo ^= slo;
    phi ^= shi;
    out[q] = mulhi_sep(plo, 0x133111EBu) + plo * 0x94D049BBu + phi * 0x133111EBu;
  }
}

// ---- magnitude rounding ---------------------------------------------------
//
// a = |r| where r = x * 2^s was formed in fp32; a is exact unless it fell
// below 2^-126 (subnormal or flushed to 0), in which case only the decision
// "is the true fraction > u" matters and it is recovered from xnz (x != 0).
// neg = (x < 0): the sign of r (r keeps x's sign even when it underflows).
// Returns |round_mode(r)| as an exact float integer (or a itself once a is
// beyond 2^23, where fp32 holds only integers; inf stays inf).
//
// Stochastic (rounding.hpp:56-59): k = floor(r) + (u < r - floor(r)).  On
// magnitudes: r >= 0 -> |k| = fl(a) + (u < fa);  r < 0 -> |k| = fl(a) +
// (fa > 0 && u >= 1 - fa) = fl(a) + (fa >= 1 - u), since 1 - u > 0.  fa =
// a - floor(a) is exact for a >= 0, and 1 - u is exact (u on the 2^-24 grid),
// so both compares are exact -- unlike r - floor(r) in fp32 for r in (-1,0).
template <int M, bool TINY = true>
LPQ_HD float round_mag(float a, bool neg, bool xnz, uint32_t v) {
  if (M == kNearestEven) {
#if defined(__CUDA_ARCH__)
    return rintf(a);
#else
    return nearbyintf(a);
#endif
  }
  const float qa = floorf(a);
  const float fa = fsub(a, qa);  // NaN when a = inf: every compare false
  bool up;
  if (M == kNearestAway) {
    up = fa >= 0.5f;
  } else if (M == kNearestZero) {
    up = fa > 0.5f;
  } else {
    // branch-free: r >= 0 compares fa > u, r < 0 compares fa >= 1 - u.
    // a == 0 with x != 0 and r > 0: the true fraction is in (0, 2^-150], so
    // u < it iff u == 0.
    const float u = variate_float(v);
    const float thr = neg ? fsub(1.0f, u) : u;
    up = (fa > thr) | (neg & (fa == thr));
    if (TINY) up |= !neg & (a == 0.0f) & xnz & (v == 0u);
  }
  return up ? fadd(qa, 1.0f) : qa;
}

// Sign of an integer result that rounded to zero (Appendix A of SURVEY.md,
// verified against rounding.hpp):  NearestEven/Stochastic -> +0,
// NearestAway -> -0 iff r < 0, NearestTowardZero -> -0 iff r >= 0 (incl. +-0).
template <int M>
LPQ_HD bool zero_negative(bool neg) {
  if (M == kNearestAway) return neg;
  if (M == kNearestZero) return !neg;
  return false;
}

// ---- fixed point (FixedFolder + fused_fixed, scalar_quant.hpp:38-63,
//      quant_ops.cpp:33-50) -------------------------------------------------

struct FixedParams {
  float up;        // 2^fl
  float down;      // 2^-fl
  float kmin, kmax;
  int32_t kmin_i;
  uint32_t mask;   // 2^wl - 1
  int32_t half;    // 2^(wl-1)
  int32_t wl;
  int32_t saturate;
  int32_t tiny;    // fl <= -1: x * 2^fl may flush to zero
};

LPQ_HD FixedParams make_fixed(int wl, int fl, bool symmetric, bool saturate) {
  FixedParams p;
  p.up = u2f((uint32_t)(127 + fl) << 23);
  p.down = u2f((uint32_t)(127 - fl) << 23);
  const int32_t kmax = (1 << (wl - 1)) - 1;
  p.kmin_i = symmetric ? -kmax : -(1 << (wl - 1));
  p.kmin = (float)p.kmin_i;
  p.kmax = (float)kmax;
  p.mask = (wl >= 32) ? 0xFFFFFFFFu : ((1u << wl) - 1u);
  p.half = 1 << (wl - 1);
  p.wl = wl;
  p.saturate = saturate ? 1 : 0;
  p.tiny = fl <= -1 ? 1 : 0;
  return p;
}

// TINY: fl <= -1, where x * 2^fl can flush to zero (make_fixed: p.tiny).
// Two's-complement fold of an integer-valued k = (kneg ? -1 : 1) * kmag into
// the wl-bit code range (FixedFolder::fold, scalar_quant.hpp:50-62, exact
// fmod semantics incl. the sign of a zero remainder, which follows k),
// scaled by `down`.  kmag >= 2^24 is an integer m * 2^t with t >= 1 (inf:
// t >= 105 > wl).
LPQ_HD float fold_wrap(float kmag, bool kneg, const FixedParams& p, float down) {
  uint32_t km;
  if (kmag < 16777216.0f) {
    km = (uint32_t)kmag;
  } else {
    const uint32_t ab = f2u(kmag);
    const int t = (int)(ab >> 23) - 150;
    const uint32_t m = (ab & 0x7FFFFFu) | 0x800000u;
    km = (t >= 32) ? 0u : (m << t);
  }
  const uint32_t ks = kneg ? (0u - km) : km;
  int32_t m = (int32_t)(ks & p.mask);
  if (m >= p.half) m -= (int32_t)(p.mask + 1u);
  if (m < p.kmin_i) m = p.kmin_i;
  if (m == 0) return kneg ? -0.0f : 0.0f;
  return fmul((float)m, down);
}

template <int M, bool SAT, bool TINY = true>
LPQ_HD float quant_fixed(float x, const FixedParams& p, uint32_t v) {
  const float r = fmul(x, p.up);
  const float a = fabsf(r);
  const bool neg = x < 0.0f;
  const bool xnz = x != 0.0f;
  const float kmag = round_mag<M, TINY>(a, neg, xnz, v);
  const bool kneg = (kmag == 0.0f) ? zero_negative<M>(neg) : neg;
  if (SAT) {
    float k = kneg ? -kmag : kmag;
    k = fminf(fmaxf(k, p.kmin), p.kmax);  // +-inf clamp too
    return fmul(k, p.down);
  }
  return fold_wrap(kmag, kneg, p, p.down);
}

LPQ_HD float fma_rn(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
  return __fmaf_rn(a, b, c);
#else
  return fmaf(a, b, c);
#endif
}

// Saturating fixed point with fl >= 0 (x * 2^fl cannot flush to zero), the
// streaming kernels' form.  NearestEven / Stochastic round the signed value
// directly (round_signed); the reference's +0 for a zero result comes from
// k * 2^-fl + 0 in one FFMA.  NearestAway / NearestTowardZero keep the
// magnitude path with the sign applied by a multiply by +-1.  Identical
// results to quant_fixed<M, true, false>.
template <int M>
LPQ_HD float quant_fixed_sat_fast(float x, const FixedParams& p, uint32_t v) {
  const float r = fmul(x, p.up);
  if (M == kNearestEven || M == kStochastic) {
    float k = round_signed<M>(r, v);
    k = fminf(fmaxf(k, p.kmin), p.kmax);  // +-inf clamp too
    return fma_rn(k, p.down, 0.0f);       // exact product; -0 + 0 = +0
  }
  const float a = fabsf(r);
  const bool neg = x < 0.0f;
  const float kmag = round_mag<M, false>(a, neg, true, v);
  float k = fmul(kmag, neg ? -1.0f : 1.0f);  // -0 when kmag == 0 and r < 0
  k = fminf(fmaxf(k, p.kmin), p.kmax);
  float out = fmul(k, p.down);
  if (M == kNearestZero && kmag == 0.0f) out = neg ? 0.0f : -0.0f;
  return out;  // NearestAway: -0 iff r < 0, as the multiply left it
}

// ---- low-width float (FloatQuantizer, scalar_quant.hpp:103-141;
//      fused_float, quant_ops.cpp:52-66) -------------------------------------

struct FloatParams {
  int32_t man;
  int32_t min_exp;
  int32_t max_exp;
  float max_value;   // (2 - 2^-man) * 2^max_exp
  float under_up;    // 2^-min_exp
  float under_down;  // 2^min_exp
  float carry;       // 2^(man+1)
  uint32_t r_exp;    // (man + 127) << 23
  int32_t tiny;      // min_exp >= 1: |x| * 2^-min_exp may flush to zero
  int32_t ef_min;    // min_exp + 127   (scaled form, biased exponents)
  int32_t ef_max;    // max_exp + 127
  int32_t ef_under;  // min_exp + man + 127: underflow grid step 2^min_exp
  int32_t sc_base;   // 254 + man
  int32_t scaled_ok; // 2 <= exp_bits <= 7
  uint32_t m_sh9;    // 2^9   (runtime multipliers, see RngMul)
  uint32_t m_two;    // 2
  uint32_t m_sh8;    // 2^8
  // bit-domain form (quant_float_bits): |x| >= 2^min_exp or x == 0
  int32_t bits_ok;   // man <= 22
  uint32_t rmask;    // the 23 - man mantissa bits that are rounded off
  uint32_t rhalf;    // rmask >> 1 (RNE: half the step, minus one ulp)
  uint32_t rshift;   // 23 - man (RNE: the kept LSB = the parity of k)
  uint32_t rodd;     // 1; 0 for man == 0, where k = 1 is always odd (rhalf
                     // then carries the +1: ties round up to k = 2)
  uint32_t vshift;   // 1 + man (stochastic: R = (~v & 0xFFFFFF) >> vshift)
  uint32_t vshift8;  // vshift + 8 (quant_float_bits_top: v = top >> 8)
  float min_normal;  // 2^min_exp
  uint32_t m_neg23;  // -2^23 (mod 2^32)
  uint32_t m_pos23;  // 2^23
  uint32_t sc_bits;  // (254 + man) << 23
  uint32_t inv_bits; // -man << 23 (mod 2^32)
  uint32_t m_neg1;   // 2^32 - 1 and 1: runtime multipliers that keep the scaled
  uint32_t m_one;    // form's exponent-field adds on the FMA pipe (mad_lo)
};

LPQ_HD FloatParams make_float(int exp_bits, int man_bits) {
  FloatParams p;
  const int bias = (1 << (exp_bits - 1)) - 1;
  p.man = man_bits;
  p.min_exp = 1 - bias;
  const int me = (1 << exp_bits) - 1 - bias;
  p.max_exp = me < 127 ? me : 127;
  // max_value = (2^(man+1) - 1) * 2^(max_exp - man), exact in fp32
  p.max_value = u2f(((uint32_t)(p.max_exp + 127) << 23) |
                    (0x7FFFFFu & ~((1u << (23 - man_bits)) - 1u)));
  p.under_up = u2f((uint32_t)(127 - p.min_exp) << 23);
  p.under_down = u2f((uint32_t)(127 + p.min_exp) << 23);
  p.carry = u2f((uint32_t)(127 + man_bits + 1) << 23);
  p.r_exp = (uint32_t)(man_bits + 127) << 23;
  p.tiny = p.min_exp >= 1 ? 1 : 0;
  p.ef_min = p.min_exp + 127;
  p.ef_max = p.max_exp + 127;
  p.ef_under = p.min_exp + man_bits + 127;
  p.sc_base = 254 + man_bits;
  p.scaled_ok = (exp_bits >= 2 && exp_bits <= 7) ? 1 : 0;
  p.m_sh9 = 1u << 9;
  p.m_two = 2u;
  p.m_sh8 = 1u << 8;
  p.m_neg23 = 0u - (1u << 23);
  p.m_pos23 = 1u << 23;
  p.sc_bits = (uint32_t)(254 + man_bits) << 23;
  p.inv_bits = 0u - ((uint32_t)man_bits << 23);
  p.m_neg1 = 0xFFFFFFFFu;
  p.m_one = 1u;
  p.bits_ok = man_bits <= 22 ? 1 : 0;
  p.rmask = man_bits <= 22 ? (1u << (23 - man_bits)) - 1u : 0u;
  p.rhalf = (p.rmask >> 1) + (man_bits == 0 ? 1u : 0u);
  p.rodd = man_bits == 0 ? 0u : 1u;
  p.rshift = man_bits <= 22 ? (uint32_t)(23 - man_bits) : 0u;
  p.vshift = (uint32_t)(1 + man_bits);
  p.vshift8 = p.vshift + 8u;
  p.min_normal = p.min_exp >= -126 ? u2f((uint32_t)(127 + p.min_exp) << 23) : 0.0f;
  return p;
}

template <int M>
LPQ_HD float quant_float(float x, const FloatParams& p, uint32_t v) {
  // Branch-free: one rounding of either the in-range significand
  // r = |x| * 2^(man - e) in [2^man, 2^(man+1)) (same mantissa bits, new
  // exponent) or, below 2^min_exp, of |x| * 2^-min_exp < 1 over {0, 1}.
  const uint32_t xb = f2u(x);
  const uint32_t ab = xb & 0x7FFFFFFFu;
  const bool neg = (int32_t)xb < 0;
  const int e = (int)(ab >> 23) - 127;  // denormals give -127 < min_exp
  const bool under = e < p.min_exp;
  const float r_in = u2f((ab & 0x7FFFFFu) | p.r_exp);
  const float r_un = fmul(u2f(ab), p.under_up);
  const float k = round_mag<M>(under ? r_un : r_in, neg, true, v);
  // q = k * 2^(e - man) (or k * 2^min_exp): exponent-field add, k >= 1
  const int sh = under ? p.min_exp : e - p.man;
  uint32_t qb = f2u(k) + ((uint32_t)sh << 23);
  const bool kz = k == 0.0f;
  if (kz) qb = 0u;
  // saturation: beyond the top binade, or a carry out of it
  const bool sat = (e > p.max_exp) | ((e == p.max_exp) & (k >= p.carry));
  if (sat) qb = f2u(p.max_value);
  const bool kneg = kz ? zero_negative<M>(neg) : neg;
  if (kneg) qb |= 0x80000000u;
  return ab == 0u ? x : u2f(qb);  // zero passes through with its sign
}

// Float quantizer, streaming form for NearestEven / Stochastic when
// |x| * 2^-min_exp cannot flush to zero (min_exp <= 0, i.e. exp_bits >= 2):
// the signed significand r = +-|x| * 2^(man - e) (or x * 2^-min_exp below the
// normal range) is rounded once with round_signed; identical results to
// quant_float<M>.
template <int M>
LPQ_HD float quant_float_fast(float x, const FloatParams& p, uint32_t v) {
  const uint32_t xb = f2u(x);
  const uint32_t ab = xb & 0x7FFFFFFFu;
  const uint32_t sign = xb & 0x80000000u;
  const int e = (int)(ab >> 23) - 127;
  const bool under = e < p.min_exp;
  const float r_in = u2f((xb & 0x807FFFFFu) | p.r_exp);
  const float r_un = fmul(x, p.under_up);
  const float k = fabsf(round_signed<M>(under ? r_un : r_in, v));
  const int sh = under ? p.min_exp : e - p.man;
  uint32_t qb = (f2u(k) + ((uint32_t)sh << 23)) | sign;
  const bool sat = (e > p.max_exp) | ((e == p.max_exp) & (k >= p.carry));
  if (sat) qb = f2u(p.max_value) | sign;
  if (k == 0.0f) qb = 0u;  // +0 for both modes
  return ab == 0u ? x : u2f(qb);
}

// Float quantizer, scaled form for NearestEven / Stochastic and
// 2 <= exp_bits <= 7 (so every scale below is a normal fp32 power of two).
// x is first clamped to [-max_value, max_value]: max_value is the top grid
// point, so every rounding of a clamped value stays within it and every x
// beyond it saturates to it in all modes (stochastic rounding past max_value
// lands on the next grid point 2^(max_exp+1), which saturates back) -- no
// clamp of the exponent from above and none of the result.  The binade
// exponent E = e (or min_exp + man below the normal range, which makes the
// grid step 2^min_exp as in the reference's two-point underflow rule) gives
// r = x * 2^(man - E) exactly, one rounding, q = k * 2^(E - man) + 0 in one
// FFMA (exact; -0 -> +0).  Zero results are +0 except x == -0 itself, which
// passes through.  Identical results to quant_float<M>.
template <int M>
LPQ_HD float quant_float_scaled(float x, const FloatParams& p, uint32_t v) {
  const float xc = fminf(fmaxf(x, -p.max_value), p.max_value);
  // the exponent field of |xc| in place (no shifts): 2^(man - E) and
  // 2^(E - man) are one integer add each on it
  uint32_t eb = f2u(xc) & 0x7F800000u;
  eb = eb < ((uint32_t)p.ef_min << 23) ? ((uint32_t)p.ef_under << 23) : eb;
  // sc_bits - eb and eb + inv_bits as IMADs (FMA pipe): the per-element
  // path is ALU-bound (log-uniform C1: ALU 77 %)
  const float sc = u2f(mad_lo(eb, p.m_neg1, p.sc_bits));
  const float inv = u2f(mad_lo(eb, p.m_one, p.inv_bits));
  const float k = round_signed<M>(fmul(xc, sc), v);
  const float q = fma_rn(k, inv, 0.0f);
  return x == 0.0f ? x : q;
}

// Float quantizer in the bit domain for |x| >= 2^min_exp (and x == +-0),
// NearestEven / Stochastic, man <= 22, x already clamped to +-max_value.
// In that range the grid is x's own binade with man fraction bits, so the
// rounding is integer arithmetic on the IEEE bits: add to the magnitude and
// clear the 23 - man dropped bits (a carry out of the mantissa steps to the
// next binade exactly as k = 2^(man+1) does; max_value is on the grid, so no
// clamped value rounds past it; +-0 stay +-0 as the reference returns x).
//  * NearestEven: + (half step - 1 ulp) + the kept LSB (ties to even).
//  * Stochastic: the reference rounds the SIGNED r = x * 2^(man-E) up
//    (toward +inf) iff u < r - floor(r), u = v * 2^-24.  With L the dropped
//    bits of |x| and s = 23 - man, frac|r| = L * 2^-s, so the magnitude goes
//    up iff  x > 0: v < L * 2^(1+man)    x < 0: v >= 2^24 - L * 2^(1+man).
//    Adding R to the magnitude and truncating carries iff L + R >= 2^s:
//    x > 0: R = (2^24 - 1 - v) >> (1+man):  L + R >= 2^s <=> v < L * 2^(1+man)
//    x < 0: R = v >> (1+man):               L + R >= 2^s <=> v >= 2^24 - L * 2^(1+man)
//    (all integers) -- the same decision, bit for bit.
// Values below 2^min_exp (the two-point underflow grid) take
// quant_float_scaled.  Identical results to quant_float<M>.
template <int M>
LPQ_HD float quant_float_bits(float xc, const FloatParams& p, uint32_t v) {
  uint32_t b = f2u(xc);
  if (M == kStochastic) {
#if defined(__CUDA_ARCH__)
    uint32_t neg;  // all ones iff x < 0 (one SHF.R.S32)
    asm("shr.s32 %0, %1, 31;" : "=r"(neg) : "r"(b));
#else
    const uint32_t neg = (uint32_t)((int32_t)b >> 31);
#endif
    b += (v ^ (~neg & 0xFFFFFFu)) >> p.vshift;
  } else {
    b += p.rhalf + ((b >> p.rshift) & p.rodd);
  }
  return u2f(b & ~p.rmask);
}

// quant_float_bits<kStochastic> from the variate's top word (v = top >> 8,
// the low 8 bits of top arbitrary):
// (top ^ (~neg & 0xFFFFFF00)) >> (8 + vshift) == (v ^ (~neg & 0xFFFFFF)) >> vshift.
// FMA = true: the sign spread as IMAD.HI.S32 and the carry add as IMAD against
// the runtime one, on the FMA pipe (the per-op GEMM's bits kernel, whose hash
// holds the ALU pipe); false: SHF.R.S32 and IADD3 (the elementwise kernel:
// C1 5304 -> 5369 GB/s).
template <bool FMA = false>
LPQ_HD float quant_float_bits_top(float xc, const FloatParams& p, uint32_t top,
                                  uint32_t one) {
  uint32_t b = f2u(xc);
  int32_t neg;  // all ones iff x < 0
#if defined(__CUDA_ARCH__)
  if (FMA)  // the high word of b * 1, signed
    asm("mul.hi.s32 %0, %1, %2;" : "=r"(neg) : "r"((int32_t)b), "r"((int32_t)one));
  else
    asm("shr.s32 %0, %1, 31;" : "=r"(neg) : "r"((int32_t)b));
#else
  neg = (int32_t)b >> 31;
#endif
  const uint32_t r = (top ^ (~(uint32_t)neg & 0xFFFFFF00u)) >> p.vshift8;
  b = FMA ? mad_lo(r, one, b) : b + r;
  return u2f(b & ~p.rmask);
}

// One element, NearestEven / Stochastic, any float format: the bit-domain
// form for zero and the normal range, else the streaming forms (identical
// results to quant_float<M>).
template <int M>
LPQ_HD float quant_float_stream(float x, const FloatParams& p, uint32_t v) {
  if (p.bits_ok && (p.scaled_ok || !p.tiny)) {
    const float xc = fminf(fmaxf(x, -p.max_value), p.max_value);
    if (!(fabsf(xc) < p.min_normal && xc != 0.0f)) return quant_float_bits<M>(xc, p, v);
  }
  if (p.scaled_ok) return quant_float_scaled<M>(x, p, v);
  if (!p.tiny) return quant_float_fast<M>(x, p, v);
  return quant_float<M>(x, p, v);
}

// ---- block floating point (block_quant_one_m, scalar_quant.hpp:80-87;
//      fused_block, quant_ops.cpp:68-115) ------------------------------------

struct BlockScale {
  float s1, s2;   // r = (x * s1) * s2 == x * 2^-shift, exact
  float o1, o2;   // q = (k * o1) * o2 == RN(k * 2^shift)
  int32_t zero;   // all-zero block: every output is +0
  int32_t bad;    // block maximum >= 2^127 (check_block_range)
};

LPQ_HD float pow2f(int e) {  // 2^e for e in [-126, 127]
  return u2f((uint32_t)(127 + e) << 23);
}

// floor(log2 m) of a nonzero finite |x| from its bits (float_exponent,
// scalar_quant.hpp:26-33), subnormals included.
LPQ_HD int float_exponent_bits(uint32_t m) {
  const int field = (int)(m >> 23);
  if (field != 0) return field - 127;
#if defined(__CUDA_ARCH__)
  return -118 - __clz((int)m);
#else
  return -118 - __builtin_clz(m);
#endif
}

// From the bits of the block maximum |x| (NaN already excluded).
LPQ_HD BlockScale make_block_scale(uint32_t max_bits, int wl) {
  BlockScale s;
  s.zero = max_bits == 0u;
  s.bad = 0;
  if (s.zero) {
    s.s1 = s.s2 = s.o1 = s.o2 = 0.0f;
    return s;
  }
  int E;
  const int field = (int)(max_bits >> 23);
  if (field != 0) {
    E = field - 127;
  } else {
#if defined(__CUDA_ARCH__)
    E = -118 - __clz((int)max_bits);
#else
    E = -118 - __builtin_clz(max_bits);
#endif
  }
  s.bad = E > 126;
  if (s.bad) E = 126;
  const int shift = E - (wl - 2);  // in [-171, 126]
  const int ns = -shift;           // in [-126, 171]
  if (ns <= 127) { s.s1 = pow2f(ns); s.s2 = 1.0f; }
  else { s.s1 = pow2f(127); s.s2 = pow2f(ns - 127); }
  if (shift >= -126) { s.o1 = pow2f(shift); s.o2 = 1.0f; }
  else { s.o1 = pow2f(-126); s.o2 = pow2f(shift + 126); }
  return s;
}

template <int M>
LPQ_HD float quant_block(float x, const BlockScale& s, float kmin, float kmax,
                         uint32_t v) {
  if (s.zero) return 0.0f;
  const float r = fmul(fmul(x, s.s1), s.s2);
  const bool neg = x < 0.0f;
  const float kmag = round_mag<M>(fabsf(r), neg, x != 0.0f, v);
  const bool kneg = (kmag == 0.0f) ? zero_negative<M>(neg) : neg;
  float k = kneg ? -kmag : kmag;
  k = fminf(fmaxf(k, kmin), kmax);
  return fmul(fmul(k, s.o1), s.o2);
}

// Block element, streaming form for NearestEven / Stochastic: signed
// rounding (round_signed), k * delta + 0 in one FFMA (-0 -> +0, and a single
// rounding of the exact k * 2^shift).  TWO: the scales needed two factors
// (block maxima near the fp32 range ends).  All-zero blocks have zero scales
// and produce +0.  Identical results to quant_block<M>.
//  * No lower clamp: |x| <= max < 2^(E+1), so |r| < 2^(wl-1) and every
//    rounding of r is >= -2^(wl-1) = kmin; only k = 2^(wl-1) needs clamping.
//  * Stochastic: a positive x whose r flushed to +0 takes the smallest
//    denormal, which gives the exact decision (k = 1 iff u == 0).  A negative
//    flushed r gives k = 0 for every u, as the exact r would.  The guard is
//    r_bits = max(r_bits, t) with t = (-x_bits) >> 31 (1 for x > +0, and for
//    x = -0 whose r_bits 0x80000000 it leaves unchanged), formed with IMADs
//    against runtime multipliers (neg1 = 2^32-1, m2 = 2) so it issues on the
//    FMA pipe; one integer max on the ALU pipe.
//  * GUARD = false skips the guard for blocks with s1 >= 1 (no product can
//    flush: |r| >= |x| >= 2^-149), and for two-factor scales (s1 = 2^127).
template <int M, bool TWO, bool GUARD = true>
LPQ_HD float quant_block_fast(float x, const BlockScale& s, float kmin,
                              float kmax, uint32_t v, uint32_t m2 = 2u,
                              uint32_t neg1 = 0xFFFFFFFFu) {
  (void)kmin;
  float r = fmul(x, s.s1);
  if (TWO) r = fmul(r, s.s2);
  if (M == kStochastic && GUARD) {
    const uint32_t t = umulhi32(f2u(x) * neg1, m2);
    const uint32_t rb = f2u(r);
    r = u2f(rb > t ? rb : t);
  }
  float k = round_signed<M>(r, v);
  k = fminf(k, kmax);
  if (TWO) return fma_rn(fmul(k, s.o1), s.o2, 0.0f);
  return fma_rn(k, s.o1, 0.0f);
}

LPQ_HD bool nonfinite(float x) { return (f2u(x) & 0x7F800000u) == 0x7F800000u; }

// |x| bits for the block maximum; NaN is ignored like `a > m` in
// reduce_max_abs (tensor.cpp:320-353); +inf stays (-> block range error).
LPQ_HD uint32_t absbits_for_max(float x) {
  const uint32_t ab = f2u(x) & 0x7FFFFFFFu;
  return ab > 0x7F800000u ? 0u : ab;
}

}  // namespace lpq
