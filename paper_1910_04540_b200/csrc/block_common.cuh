// block_common.cuh -- device helpers shared by the block-floating-point
// kernels (block.cu, block_cluster.cu).
#pragma once

#include "kernels.cuh"

namespace lpq {
namespace blk {

constexpr uint32_t kFull = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t max4(const float4& v) {
  return max(max(absbits_for_max(v.x), absbits_for_max(v.y)),
             max(absbits_for_max(v.z), absbits_for_max(v.w)));
}
__device__ __forceinline__ uint32_t nf4(const float4& v) {
  return (nonfinite(v.x) | nonfinite(v.y) | nonfinite(v.z) | nonfinite(v.w))
             ? 1u : 0u;
}

// TWO: the block's scales need two factors (maxima near the fp32 range
// ends); uniform per block, so kernels branch once per block/row.
// z = key ^ flat index; m32 == 32 (runtime, see variate24_zb).
// GUARD: see quant_block_fast (stochastic flush guard; needs_guard()).
// v: the element's 24-bit variate (stochastic), else unused
template <int M, bool TWO, bool GUARD = true>
__device__ __forceinline__ float qbv(float x, const BlockScale& s, float kmin,
                                     float kmax, uint32_t v, const RngMul& rm) {
  if (M == kNearestEven || M == kStochastic)
    return quant_block_fast<M == kNearestEven ? kNearestEven : kStochastic, TWO,
                            GUARD>(x, s, kmin, kmax, v, rm.m2, rm.neg1);
  return quant_block<M>(x, s, kmin, kmax, v);
}

template <int M, bool TWO, bool GUARD = true>
__device__ __forceinline__ float qb(float x, const BlockScale& s, float kmin,
                                    float kmax, uint64_t z, const RngMul& rm) {
  uint32_t v = 0;
  if (M == kStochastic) v = variate24_zb(z, rm.m32);
  return qbv<M, TWO, GUARD>(x, s, kmin, kmax, v, rm);
}

// IDX4: idx % 4 == 0, so key ^ (idx + q) == (key ^ idx) ^ q, and the four
// variates come from variate24_x4
template <int M, bool TWO, bool IDX4, bool GUARD = true>
__device__ __forceinline__ float4 qb4(const float4& x, const BlockScale& s,
                                      float kmin, float kmax, uint64_t key,
                                      uint64_t idx, const RngMul& m32) {
  float4 o;
  if (M == kStochastic && IDX4) {
    uint32_t v[4];
    variate24_x4(key, idx, m32.m32, v);
    o.x = qbv<M, TWO, GUARD>(x.x, s, kmin, kmax, v[0], m32);
    o.y = qbv<M, TWO, GUARD>(x.y, s, kmin, kmax, v[1], m32);
    o.z = qbv<M, TWO, GUARD>(x.z, s, kmin, kmax, v[2], m32);
    o.w = qbv<M, TWO, GUARD>(x.w, s, kmin, kmax, v[3], m32);
    return o;
  }
  const uint64_t z0 = key ^ idx;
  o.x = qb<M, TWO, GUARD>(x.x, s, kmin, kmax, z0, m32);
  o.y = qb<M, TWO, GUARD>(x.y, s, kmin, kmax, IDX4 ? z0 ^ 1u : key ^ (idx + 1), m32);
  o.z = qb<M, TWO, GUARD>(x.z, s, kmin, kmax, IDX4 ? z0 ^ 2u : key ^ (idx + 2), m32);
  o.w = qb<M, TWO, GUARD>(x.w, s, kmin, kmax, IDX4 ? z0 ^ 3u : key ^ (idx + 3), m32);
  return o;
}

// single-factor scales with s1 < 1: a product x * s1 can flush to zero
__device__ __forceinline__ bool needs_guard(const BlockScale& s) {
  return s.s1 < 1.0f;
}

// |x| maximum that PROPAGATES NaN (FMNMX3.NAN, 0.5 instructions per
// element, fmax3_nan in quant_math.cuh); a NaN row maximum sends the row
// down absmax_nf's slow path.
__device__ __forceinline__ void absmax_nan(const float4& v, float& m) {
  m = fmax3_nan(m, fabsf(v.x), fabsf(v.y));
  m = fmax3_nan(m, fabsf(v.z), fabsf(v.w));
}

// |x| maximum with NaN ignored (fmaxf returns the non-NaN operand, like
// `a > m` in reduce_max_abs); nf = x * 0 + nf turns NaN on any non-finite x.
__device__ __forceinline__ void absmax_nf(const float4& v, float& m, float& nf) {
  m = fmaxf(fmaxf(m, fabsf(v.x)), fmaxf(fabsf(v.y), fmaxf(fabsf(v.z), fabsf(v.w))));
  nf = __fmaf_rn(v.x, 0.0f, nf);
  nf = __fmaf_rn(v.y, 0.0f, nf);
  nf = __fmaf_rn(v.z, 0.0f, nf);
  nf = __fmaf_rn(v.w, 0.0f, nf);
}

__device__ __forceinline__ bool two_factor(const BlockScale& s) {
  return s.s2 != 1.0f || s.o2 != 1.0f;
}

__device__ __forceinline__ void flag(uint32_t* status, uint32_t bits) {
  if (bits) atomicOr(status, bits);
}


}  // namespace blk
}  // namespace lpq
