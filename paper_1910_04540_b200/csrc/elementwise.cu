// elementwise.cu -- single-pass float / fixed quantizers and the device-side
// generators (random_uniform, variate_tensor).
//
// Replaces the per-element CPU loops fused_fixed / fused_float
// (proj/src/quant_ops.cpp:33-66) driven by quant_pass/parallel_for
// (quant_ops.cpp:13-31, tensor.cpp:118-136).  HBM-bound: 8 algorithmic bytes
// per element.  Each thread moves U float4 with the loads issued before any
// arithmetic (U*16 B in flight per thread) and streaming cache hints
// (ld.global.cs / st.global.cs); the grid covers the tensor in one trip per
// thread (launch_ew: U = 8 for large tensors, 4-7 below 2^26 elements so the
// last wave of 4 CTAs/SM fills well), the kernel loops grid-stride only when
// the grid would exceed the launch limit.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "kernels.cuh"

// Threads per CTA of the small-tensor (< 2^26 elements) elementwise kernels:
// one-warp CTAs for stochastic and four-warp CTAs for nearest, at the same
// warps per SM as the 256-thread CTAs, retire at a finer grain, which
// shortens the last wave: C1 stochastic 5163-5359 -> 5400-5502 GB/s (with
// 64 / 128 threads: 5375-5454 / 5384-5416), C1 log-uniform nearest 5707 ->
// 5800-5900 (64 threads: 5917-5934, but the C5 sweep's many small nearest
// tensors 6268 -> 6250; 128: 6264); tensors >= 2^26 keep 256 (128 / 64
// there: C2 7021 -> 6937-6949 GB/s, float stochastic 2^30 +0.8 %).
#ifndef LPQ_SMALL_TPB_RN
#define LPQ_SMALL_TPB_RN 128
#endif
#ifndef LPQ_SMALL_TPB
#define LPQ_SMALL_TPB 32
#endif

namespace lpq {

namespace {

constexpr int kThreads = 256;
constexpr int kUnrollBig = 8;    // 8 float4 = 128 B in flight per thread
// tensors below 2^26 elements: a finer last wave (graph-captured
// back-to-back 2^24 launches, scripts/time_b2b.py: nearest best at 4 float4
// per thread, stochastic at 6 -- float(5,2) 4869 -> 4969 GB/s, fixed(8,4)
// 5683 -> 5874)
template <int M>
constexpr int unroll_small() { return M == kStochastic ? 6 : 4; }

template <bool TINY>
struct FixedSatOp {
  static constexpr bool kFmaRng = false;  // FMA-pipe-bound already
  static constexpr bool kBits = false;
  __device__ __forceinline__ bool in_range4(const float4&) const { return false; }
  template <int M>
  __device__ __forceinline__ float4 bits4(const float4& x, const uint32_t (&)[4], uint32_t) const {
    return x;
  }
  FixedParams p;
  template <int M>
  __device__ __forceinline__ float apply(float x, uint32_t v) const {
    if (TINY) return quant_fixed<M, true, true>(x, p, v);
    return quant_fixed_sat_fast<M>(x, p, v);
  }
};
struct FixedWrapOp {
  static constexpr bool kFmaRng = true;
  static constexpr bool kBits = false;
  __device__ __forceinline__ bool in_range4(const float4&) const { return false; }
  template <int M>
  __device__ __forceinline__ float4 bits4(const float4& x, const uint32_t (&)[4], uint32_t) const {
    return x;
  }
  FixedParams p;
  template <int M>
  __device__ __forceinline__ float apply(float x, uint32_t v) const {
    return quant_fixed<M, false>(x, p, v);
  }
};
// V: 2 = scaled form (even/stochastic, 2 <= exp_bits <= 7), 1 = bit-surgery
// streaming form (even/stochastic, exp_bits == 8), 0 = general
template <int V>
struct FloatOp {
  static constexpr bool kFmaRng = V != 2;  // the scaled form is FMA-heavy
  static constexpr bool kBits = V != 0;   // apply4: the bit-domain form
  FloatParams p;
  // Four elements take the bit-domain form (bits4) when every |x| <=
  // max_value (no clamp; NaN and inf fail the max.NaN test, so that path
  // needs no non-finite probe) and every element is zero or >= 2^min_exp --
  // the common case, tested with two 3-input max/min per float4, the exact
  // per-element underflow test only when the minimum falls below 2^min_exp
  // (a zero, or an underflow candidate).
  __device__ __forceinline__ bool in_range4(const float4& x) const {
    if (!p.bits_ok) return false;
    const float ax = fabsf(x.x), ay = fabsf(x.y), az = fabsf(x.z), aw = fabsf(x.w);
    if (!(fmax3_nan(fmax3_nan(ax, ay, az), aw, aw) <= p.max_value)) return false;
    return !(fmin3(fmin3(ax, ay, az), aw, aw) < p.min_normal &&
             ((ax < p.min_normal && ax != 0.0f) | (ay < p.min_normal && ay != 0.0f) |
              (az < p.min_normal && az != 0.0f) | (aw < p.min_normal && aw != 0.0f)));
  }
  // M: NearestEven or Stochastic; t: the variates' top words
  // (variate24_x4_top)
  template <int M>
  __device__ __forceinline__ float4 bits4(const float4& x, const uint32_t (&t)[4],
                                          uint32_t one) const {
    if (M == kStochastic)
      return make_float4(quant_float_bits_top(x.x, p, t[0], one),
                         quant_float_bits_top(x.y, p, t[1], one),
                         quant_float_bits_top(x.z, p, t[2], one),
                         quant_float_bits_top(x.w, p, t[3], one));
    return make_float4(quant_float_bits<kNearestEven>(x.x, p, 0u),
                       quant_float_bits<kNearestEven>(x.y, p, 0u),
                       quant_float_bits<kNearestEven>(x.z, p, 0u),
                       quant_float_bits<kNearestEven>(x.w, p, 0u));
  }
  template <int M>
  __device__ __forceinline__ float apply(float x, uint32_t v) const {
    constexpr int MF = M == kNearestEven ? kNearestEven : kStochastic;
    if (V == 2 && (M == kNearestEven || M == kStochastic))
      return quant_float_scaled<MF>(x, p, v);
    if (V == 1 && (M == kNearestEven || M == kStochastic))
      return quant_float_fast<MF>(x, p, v);
    return quant_float<M>(x, p, v);
  }
};

// z = key ^ flat_index.  Non-finite inputs are not special-cased per
// element: the kernel folds |x| bits into a running maximum and flags the
// call (the reference throws and discards the whole output,
// quant_ops.cpp:21-29), so the output of such a call is unspecified.
// nf accumulates x * 0 + nf on the FMA pipe: it stays +0 for finite x and
// turns NaN for any +-inf or NaN.
template <int M, class Op>
__device__ __forceinline__ float qelem(const Op& op, float x, uint64_t z,
                                       const RngMul& rm, float& nf) {
  uint32_t v = 0;
  if (M == kStochastic)
    v = Op::kFmaRng ? variate24_zf(z, rm) : variate24_zb(z, rm.m32);
  nf = __fmaf_rn(x, 0.0f, nf);
  return op.template apply<M>(x, v);
}

template <int M, class Op>
__device__ __forceinline__ float qelem_v(const Op& op, float x, uint32_t v,
                                         float& nf) {
  nf = __fmaf_rn(x, 0.0f, nf);
  return op.template apply<M>(x, v);
}

// IDX4: (base + head) % 4 == 0, so the four flat indices of a float4 differ
// from the first only in their two low bits: key ^ (i + q) == (key ^ i) ^ q.
template <int M, class Op, bool IDX4, int kUnroll, int TPB = kThreads>
// (float ops with the bit-domain form: <= 64 registers, 4 CTAs per SM --
// the inlined fallback path would otherwise cost one CTA per SM; 5 for the
// small-tensor nearest kernel: C1 nearest 5971 -> 6096 GB/s)
__global__ void __launch_bounds__(TPB, (!Op::kBits ? 0 : (kUnroll == 8 || M == kStochastic ? 4 : 5)) * (kThreads / TPB))
    k_elementwise(const float* __restrict__ x, float* __restrict__ y,
                  int64_t n, int64_t head, uint64_t base, uint64_t key, Op op,
                  RngMul rm, uint32_t* __restrict__ status) {
  // programmatic dependent launch: the next kernel of the stream may be
  // scheduled once every CTA of this one has started (so only into the SM
  // slots our last wave frees), and this one reads nothing before the
  // previous kernel's writes are visible
  pdl_trigger();
  const int64_t n4 = (n - head) >> 2;
  const float4* __restrict__ x4 = reinterpret_cast<const float4*>(x + head);
  float4* __restrict__ y4 = reinterpret_cast<float4*>(y + head);
  float nf = 0.0f;
  const int64_t hi = n4;
  const int64_t step = (int64_t)gridDim.x * TPB * kUnroll;
  // (hashing the first trip's variates before the wait, to overlap the
  // previous kernel's tail, delays this kernel's loads: C1 5406 -> 5054-5113
  // GB/s with two float4s' variates, 4346 with all seven)
  pdl_wait();
  const int64_t i_first = (int64_t)blockIdx.x * TPB * kUnroll + threadIdx.x;
  for (int64_t i0 = i_first; i0 < hi; i0 += step) {
    float4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t j = i0 + (int64_t)u * TPB;
      if (j < hi) v[u] = __ldcs(x4 + j);  // (.L2::256B: C2 7012 -> 6993, C1 -2 %)
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t j = i0 + (int64_t)u * TPB;
      if (j < hi) {
        const uint64_t idx = base + (uint64_t)(head + 4 * j);
        if (Op::kBits && (M == kNearestEven || (M == kStochastic && IDX4))) {
          // the variates' top words (variate24_x4_top); the per-element
          // forms take top >> 8.  (Testing
          // the range first and hashing per path inlines two hashes per
          // float4: C1 5095 -> 4874 GB/s, log-uniform 3506 -> 2720.)
          uint32_t tt[4] = {0u, 0u, 0u, 0u};
          if (M == kStochastic) variate24_x4_top(key, idx, rm, tt);
          float4 o;
          // warp-uniform choice: a warp whose float4s are not all in range
          // runs the per-element forms for every lane, instead of diverging
          // into both paths (mixed warps, e.g. log-uniform magnitudes, paid
          // for both): C1 log-uniform stochastic 3492 -> 3806 GB/s, nearest
          // 5061 -> 5595, at ~1 % on uniform stochastic (the vote; a
          // full-mask vote for warps wholly inside the tensor, behind a
          // warp-uniform test, was slower: C1 4662, log-uniform 3612; so
          // was deferring the per-element float4s to a cold second loop to
          // keep the hot code contiguous: C1 4568-4809 vs 5005-5011; and the
          // scaled form two elements at a time with FMUL2 / FFMA2.RM / FFMA2:
          // ~7 instructions fewer per float4, log-uniform 3967 -> 3988-4005,
          // C1 and nearest no better)
          if (__all_sync(__activemask(), op.in_range4(v[u]))) {
            o = op.template bits4<M>(v[u], tt, rm.one);
          } else {
            // v = top >> 8 as hi(top * 2^24): an IMAD.HI on the FMA pipe
            const uint32_t m = M == kStochastic ? rm.m24 : 0u;
            o.x = qelem_v<M>(op, v[u].x, umulhi32(tt[0], m), nf);
            o.y = qelem_v<M>(op, v[u].y, umulhi32(tt[1], m), nf);
            o.z = qelem_v<M>(op, v[u].z, umulhi32(tt[2], m), nf);
            o.w = qelem_v<M>(op, v[u].w, umulhi32(tt[3], m), nf);
          }
          __stcs(y4 + j, o);
          continue;
        }
        if (M == kStochastic && IDX4) {  // the float4's variates together
          uint32_t vv[4];
          variate24_x4(key, idx, rm.m32, vv);
          float4 o;
          o.x = qelem_v<M>(op, v[u].x, vv[0], nf);
          o.y = qelem_v<M>(op, v[u].y, vv[1], nf);
          o.z = qelem_v<M>(op, v[u].z, vv[2], nf);
          o.w = qelem_v<M>(op, v[u].w, vv[3], nf);
          __stcs(y4 + j, o);
          continue;
        }
        uint64_t z0, z1, z2, z3;
        if (IDX4) {
          z0 = key ^ idx;
          z1 = z0 ^ 1u;
          z2 = z0 ^ 2u;
          z3 = z0 ^ 3u;
        } else {
          z0 = key ^ idx;
          z1 = key ^ (idx + 1);
          z2 = key ^ (idx + 2);
          z3 = key ^ (idx + 3);
        }
        float4 o;
        o.x = qelem<M>(op, v[u].x, z0, rm, nf);
        o.y = qelem<M>(op, v[u].y, z1, rm, nf);
        o.z = qelem<M>(op, v[u].z, z2, rm, nf);
        o.w = qelem<M>(op, v[u].w, z3, rm, nf);
        __stcs(y4 + j, o);
      }
    }
  }
  // scalar head (before 16-byte alignment) and tail (after the last float4)
  const int64_t tail0 = head + 4 * n4;
  const int64_t extra = head + (n - tail0);
  for (int64_t t = (int64_t)blockIdx.x * TPB + threadIdx.x; t < extra;
       t += (int64_t)gridDim.x * TPB) {
    const int64_t e = t < head ? t : tail0 + (t - head);
    y[e] = qelem<M>(op, x[e], key ^ (base + (uint64_t)e), rm, nf);
  }
  if (__any_sync(0xFFFFFFFFu, nf != nf) && (threadIdx.x & 31) == 0)
    atomicOr(status, kStatusNonFinite);
}

// k_elementwise launches under programmatic dependent launch (kernels.cuh
// launch_pdl): C1 5350 -> 5390 GB/s, C1 nearest 6057 -> 6080-6170, C5 6243
// -> 6293
template <int TPB = kThreads, typename... KArgs, typename... Args>
cudaError_t launch_ew_kernel(void (*k)(KArgs...), int grid, cudaStream_t s, Args... args) {
  return launch_pdl(k, dim3((unsigned)grid), dim3(TPB), s, args...);
}

int64_t vector_head(const float* x, const float* y, int64_t n) {
  const uintptr_t ax = reinterpret_cast<uintptr_t>(x);
  const uintptr_t ay = reinterpret_cast<uintptr_t>(y);
  if (((ax ^ ay) & 15u) != 0) return n;  // different misalignment: scalar
  const int64_t h = (int64_t)(((16u - (ax & 15u)) & 15u) >> 2);
  return std::min(h, n);
}

template <int M, class Op>
cudaError_t launch_ew(const float* x, float* y, int64_t n, uint64_t base,
                      uint64_t key, const Op& op, uint32_t* status,
                      cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t head = vector_head(x, y, n);
  const int64_t n4 = (n - head) >> 2;
  const int64_t work = std::max<int64_t>(n4, n - 4 * n4);
  const bool idx4 = ((base + (uint64_t)head) & 3u) == 0;
  // (A TMA variant -- one cp.async.bulk of a 32 KB tile into shared memory
  // per CTA, quantize there, one bulk store -- measured slower on C2: 6880
  // GB/s at 6 CTAs/SM, 6695 with 16 KB tiles at 8, vs 6984-7022.)
  // One trip per thread over the whole tensor (not a persistent grid): CTAs
  // retire and launch in address order, which keeps the DRAM pages in use
  // compact.  Measured on B200 (scripts/ew_variants.cu, 2^30 elements):
  // persistent grid-stride 5.85 TB/s vs one-trip 8 x float4 6.59 TB/s.
  // tensors below 2^26 elements: fewer float4 per thread (unroll_small), a
  // finer last wave (2^24 float(5,2) nearest 6082 -> 6319 GB/s with 4, 2^20
  // stochastic 1764 -> 2032)
  const bool small = idx4 && n < (int64_t(1) << 26);
  constexpr int kUnrollSmall = unroll_small<M>();
  if constexpr (M == kStochastic) if (small) {  // (not instantiated for other modes)
    // stochastic (issue-heavier) small tensors: 5, 6 or 7 float4 per thread,
    // whichever fills the last wave of 4 CTAs/SM best (2^24 float(5,2): 7,
    // 3.96 waves, 4864 -> 4947 GB/s vs 6 at 4.61 waves)
    const int64_t slots = 4 * (kThreads / LPQ_SMALL_TPB) * (int64_t)device_info().sm_count;
    int u = 6;
    double best = 0.0;
    for (int c : {6, 7, 5}) {
      const int64_t ctas = (work + (int64_t)LPQ_SMALL_TPB * c - 1) / ((int64_t)LPQ_SMALL_TPB * c);
      const int64_t waves = (ctas + slots - 1) / slots;
      const double fill = (double)ctas / (double)(waves * slots);
      if (fill > best + 0.02) { best = fill; u = c; }
    }
    // (a resident grid with equal contiguous shares per CTA, so every SM
    // finishes together, measured slower: C1 5187 -> 4945 GB/s; 5 / 6 / 4
    // float4 per thread at 5 / 5 / 6 CTAs per SM and 8 at 4: 4933 / 5095 /
    // 5026 / 5121 vs 5057, within run-to-run noise or worse; with one-warp
    // CTAs, forcing 5 / 6 / 8 float4 per thread at 2^24: 4761 / 5090-5128 /
    // 5434-5440 vs 5427-5455 for the 7 chosen here)
    constexpr int kT = LPQ_SMALL_TPB;
    const int64_t want = (work + (int64_t)kT * u - 1) / ((int64_t)kT * u);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, 0x7FFFFFFF));
    cudaError_t e;
    if (u == 5)
      e = launch_ew_kernel<kT>(k_elementwise<M, Op, true, 5, kT>, grid, s, x, y, n, head, base, key, op,
                           rng_mul(), status);
    else if (u == 7)
      e = launch_ew_kernel<kT>(k_elementwise<M, Op, true, 7, kT>, grid, s, x, y, n, head, base, key, op,
                           rng_mul(), status);
    else
      e = launch_ew_kernel<kT>(k_elementwise<M, Op, true, 6, kT>, grid, s, x, y, n, head, base, key, op,
                           rng_mul(), status);
    note_launch();
    return e;
  }
  const int unroll = small ? kUnrollSmall : kUnrollBig;
  const int64_t tpb = small ? LPQ_SMALL_TPB_RN : kThreads;
  const int64_t want = (work + tpb * unroll - 1) / (tpb * unroll);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, 0x7FFFFFFF));
  cudaError_t e;
  if (small)
    e = launch_ew_kernel<LPQ_SMALL_TPB_RN>(k_elementwise<M, Op, true, kUnrollSmall, LPQ_SMALL_TPB_RN>,
                                           grid, s, x, y, n, head, base, key, op, rng_mul(), status);
  else if (idx4)
    e = launch_ew_kernel(k_elementwise<M, Op, true, kUnrollBig>, grid, s, x, y, n, head, base,
                         key, op, rng_mul(), status);
  else
    e = launch_ew_kernel(k_elementwise<M, Op, false, kUnrollBig>, grid, s, x, y, n, head, base,
                         key, op, rng_mul(), status);
  note_launch();
  return e;
}

template <class Op>
cudaError_t dispatch_mode(const float* x, float* y, int64_t n, uint64_t base,
                          uint64_t key, const Op& op, int mode,
                          uint32_t* status, cudaStream_t s) {
  switch (mode) {
    case kStochastic: return launch_ew<kStochastic>(x, y, n, base, key, op, status, s);
    case kNearestAway: return launch_ew<kNearestAway>(x, y, n, base, key, op, status, s);
    case kNearestZero: return launch_ew<kNearestZero>(x, y, n, base, key, op, status, s);
    default: return launch_ew<kNearestEven>(x, y, n, base, key, op, status, s);
  }
}

// ---- byte codes of quantized values (host-path device->host copy) -----------

__device__ __forceinline__ uint8_t encode8(float q, const ByteCode& bc) {
  if (bc.kind == 1) return (uint8_t)__float2int_rn(__fmul_rn(q, bc.scale));  // exact k
  const uint32_t b = f2u(q);
  const uint32_t sign = (b >> 31) << 7;
  const uint32_t ab = b & 0x7FFFFFFFu;
  if (ab == 0u) return (uint8_t)sign;
  const int e = (int)(ab >> 23) - 127;  // quantized values are normal
  const uint32_t ei = (uint32_t)(e - bc.min_exp + 1);
  const uint32_t mt = (ab >> (23 - bc.man)) & ((1u << bc.man) - 1u);
  return (uint8_t)(sign | (ei << bc.man) | mt);
}

__global__ void __launch_bounds__(kThreads)
    k_encode8(const float* __restrict__ q, uint8_t* __restrict__ c, int64_t n,
              ByteCode bc) {
  const int64_t i0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * 16;
  if (i0 + 16 <= n && (reinterpret_cast<uintptr_t>(q + i0) & 15u) == 0 &&
      (reinterpret_cast<uintptr_t>(c + i0) & 15u) == 0) {
    uint32_t w[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(q + i0) + g);
      w[g] = (uint32_t)encode8(v.x, bc) | ((uint32_t)encode8(v.y, bc) << 8) |
             ((uint32_t)encode8(v.z, bc) << 16) | ((uint32_t)encode8(v.w, bc) << 24);
    }
    __stcs(reinterpret_cast<uint4*>(c + i0), make_uint4(w[0], w[1], w[2], w[3]));
  } else {
    for (int64_t i = i0; i < n && i < i0 + 16; ++i) c[i] = encode8(q[i], bc);
  }
}

// Block byte codes: k = q * 2^-(E_b - (wl - 2)) in double (exact: a power-of-
// two scale of an fp32 value), checked to be an int8 whose decode
// float(double(k) * delta_b) gives q back bit for bit.
__global__ void __launch_bounds__(kThreads)
    k_encode_block8(const float* __restrict__ q, uint8_t* __restrict__ c, int64_t n,
                    int64_t extent, int64_t stride, const uint32_t* __restrict__ maxima,
                    int wl, uint32_t* __restrict__ not_exact) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kThreads) {
    const int64_t b = (i / stride) % extent;
    const uint32_t mb = maxima[b];
    const float v = q[i];
    int k = 0;
    if (mb != 0u) {
      const int E = float_exponent_bits(mb);
      const double inv = ldexp(1.0, -(E - (wl - 2)));
      const double kd = (double)v * inv;
      k = (int)kd;
      bad |= (double)k != kd || k < -128 || k > 127 ||
             f2u((float)((double)k * ldexp(1.0, E - (wl - 2)))) != f2u(v);
    } else {
      bad |= f2u(v) != 0u;  // an all-zero block quantizes to +0
    }
    c[i] = (uint8_t)(int8_t)k;
  }
  if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(not_exact, 1u);
}

// ---- generators -------------------------------------------------------------

__global__ void __launch_bounds__(kThreads)
    k_uniform(float* __restrict__ y, int64_t n, uint64_t base, uint64_t key,
              double lo, double span) {
  // tensor.cpp:430-440: float(lo + (hi - lo) * u) in double; (hi-lo)*u is
  // exact (24 x 24 bits), so contraction into DFMA cannot change the result.
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kThreads) {
    const double u = (double)variate24(key, base + (uint64_t)i) * 0x1p-24;
    y[i] = __double2float_rn(__dadd_rn(lo, __dmul_rn(span, u)));
  }
}

__global__ void __launch_bounds__(kThreads)
    k_variates(float* __restrict__ y, int64_t n, uint64_t base, uint64_t key) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kThreads)
    y[i] = variate_float(variate24(key, base + (uint64_t)i));
}

int gen_grid(int64_t n) {
  const int64_t cap = (int64_t)device_info().sm_count * 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(cap, (n + kThreads - 1) / kThreads));
}

}  // namespace

cudaError_t launch_fixed(const float* x, float* y, int64_t n, uint64_t base,
                         uint64_t key, const FixedParams& p, int mode,
                         uint32_t* status, cudaStream_t s) {
  if (p.saturate && !p.tiny)
    return dispatch_mode(x, y, n, base, key, FixedSatOp<false>{p}, mode, status, s);
  if (p.saturate)
    return dispatch_mode(x, y, n, base, key, FixedSatOp<true>{p}, mode, status, s);
  return dispatch_mode(x, y, n, base, key, FixedWrapOp{p}, mode, status, s);
}

cudaError_t launch_float(const float* x, float* y, int64_t n, uint64_t base,
                         uint64_t key, const FloatParams& p, int mode,
                         uint32_t* status, cudaStream_t s) {
  if (p.scaled_ok)
    return dispatch_mode(x, y, n, base, key, FloatOp<2>{p}, mode, status, s);
  if (!p.tiny)
    return dispatch_mode(x, y, n, base, key, FloatOp<1>{p}, mode, status, s);
  return dispatch_mode(x, y, n, base, key, FloatOp<0>{p}, mode, status, s);
}

cudaError_t launch_encode8(const float* q, uint8_t* c, int64_t n, const ByteCode& bc,
                           cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t per = (int64_t)kThreads * 16;
  k_encode8<<<(unsigned)((n + per - 1) / per), kThreads, 0, s>>>(q, c, n, bc);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_uniform(float* y, int64_t n, uint64_t base, uint64_t key,
                           float lo, float hi, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const double l = lo, h = hi;
  k_uniform<<<gen_grid(n), kThreads, 0, s>>>(y, n, base, key, l, h - l);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_variates(float* y, int64_t n, uint64_t base, uint64_t key,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_variates<<<gen_grid(n), kThreads, 0, s>>>(y, n, base, key);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_encode_block8(const float* q, uint8_t* c, const BlockGeom& g,
                                 const uint32_t* maxima, int wl, uint32_t* not_exact,
                                 cudaStream_t s) {
  const int64_t n = g.outer * g.extent * g.stride;
  if (n <= 0) return cudaSuccess;
  const int64_t grid = std::min<int64_t>((n + kThreads - 1) / kThreads,
                                         (int64_t)device_info().sm_count * 16);
  k_encode_block8<<<(unsigned)grid, kThreads, 0, s>>>(q, c, n, g.extent, g.stride, maxima,
                                                      wl, not_exact);
  note_launch();
  return cudaGetLastError();
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("LPQ_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace lpq
