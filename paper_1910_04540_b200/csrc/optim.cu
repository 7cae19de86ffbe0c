// optim.cu -- the low-precision optimizer step, fused (SURVEY.md §8(f) row 2:
// the training-loop caller of the quantizers).
//
// Reference: LowPrecisionOptimizer::step (proj/src/train.cpp:148-178).  Per
// parameter tensor it makes four quantize_fused calls (gradient, velocity,
// accumulator, weight) and four elementwise tensor ops (scale, add, scale,
// sub), each a full pass with its own temporary.  Here the whole update of
// one parameter is ONE kernel pass: read g, vel, acc once, write vel, acc, w
// once (24 algorithmic bytes per element), with the reference's per-op fp32
// arithmetic (`float(double(a) op double(b))` == fp32 RN) and its four
// quantizers (each with its own seed and call id, flat-index variates):
//
//   g   = Qg(g)
//   v   = Qa1(fl32(fl32(momentum * vel) + g));   vel = v
//   a   = Qa2(fl32(acc - fl32(lr * v)));         acc = a
//   w   = Qw(a)
//
// Block formats need a whole-tensor maximum of an intermediate and cannot be
// fused; they are rejected (LPQ_ERR_UNSUPPORTED) -- run the unfused sequence.
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/lpq.h"
#include "kernels.cuh"
#include "runtime.h"

namespace lpq {

namespace {

constexpr int kT = 256;

struct Slot {
  int32_t enabled;
  int32_t kind;  // LPQ_FLOAT / LPQ_FIXED
  int32_t mode;
  int32_t saturate;
  uint64_t key;
  FloatParams fp;
  FixedParams xp;
};

// The element forms the streaming quantizers use (elementwise.cu launch_*),
// picked by the slot's (uniform) parameters.
template <int M>
__device__ __forceinline__ float q_mode(float x, const Slot& s, uint32_t v) {
  constexpr bool kFast = M == kNearestEven || M == kStochastic;
  if (s.kind == LPQ_FLOAT) {
    constexpr int MF = kFast ? M : kNearestEven;
    if (kFast && s.fp.bits_ok && (s.fp.scaled_ok || !s.fp.tiny)) {
      // the bit-domain form for zero and the normal range (quant_float_bits)
      const float xc = fminf(fmaxf(x, -s.fp.max_value), s.fp.max_value);
      if (!(fabsf(xc) < s.fp.min_normal && xc != 0.0f))
        return quant_float_bits<MF>(xc, s.fp, v);
    }
    if (kFast && s.fp.scaled_ok) return quant_float_scaled<kFast ? M : kNearestEven>(x, s.fp, v);
    if (kFast && !s.fp.tiny) return quant_float_fast<kFast ? M : kNearestEven>(x, s.fp, v);
    return quant_float<M>(x, s.fp, v);
  }
  if (s.saturate) {
    if (s.xp.tiny) return quant_fixed<M, true, true>(x, s.xp, v);
    return quant_fixed_sat_fast<M>(x, s.xp, v);
  }
  return quant_fixed<M, false>(x, s.xp, v);
}

// grid-uniform dispatch on the slot's mode (no divergence)
__device__ __forceinline__ float q_slot_key(float x, const Slot& s, uint64_t key,
                                            uint64_t idx, uint32_t& flags) {
  if (!s.enabled) return x;
  if (nonfinite(x)) flags |= kStatusNonFinite;
  switch (s.mode) {
    case kStochastic: return q_mode<kStochastic>(x, s, variate24(key, idx));
    case kNearestAway: return q_mode<kNearestAway>(x, s, 0u);
    case kNearestZero: return q_mode<kNearestZero>(x, s, 0u);
    default: return q_mode<kNearestEven>(x, s, 0u);
  }
}

__device__ __forceinline__ float q_slot(float x, const Slot& s, uint64_t idx,
                                        uint32_t& flags) {
  return q_slot_key(x, s, s.key, idx, flags);
}

// LowPrecisionOptimizer::step (train.cpp:148-178) for one element
__device__ __forceinline__ void sgd_element(float gin, float& vel, float& acc,
                                            float& w, float momentum, float lr,
                                            const Slot* q, const uint64_t* key,
                                            uint64_t idx, uint32_t& flags) {
  const float g = q_slot_key(gin, q[0], key[0], idx, flags);
  float v = __fadd_rn(__fmul_rn(momentum, vel), g);  // add(scale(vel, m), g)
  if (nonfinite(v)) flags |= kStatusInvalidValue;    // map_elements check
  v = q_slot_key(v, q[1], key[1], idx, flags);
  vel = v;
  const float lv = __fmul_rn(v, lr);                  // scale(v, lr)
  float a = __fsub_rn(acc, lv);                       // sub(acc, .)
  if (nonfinite(lv) || nonfinite(a)) flags |= kStatusInvalidValue;
  a = q_slot_key(a, q[2], key[2], idx, flags);
  acc = a;
  w = q_slot_key(a, q[3], key[3], idx, flags);
}

__global__ void __launch_bounds__(kT)
    k_sgd_step(const float* __restrict__ grad, float* __restrict__ vel,
               float* __restrict__ acc, float* __restrict__ w, int64_t n,
               float momentum, float lr, Slot qg, Slot qa1, Slot qa2, Slot qw,
               uint64_t base, uint32_t* __restrict__ status) {
  uint32_t flags = 0;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kT) {
    const uint64_t idx = base + (uint64_t)i;
    const float g = q_slot(grad[i], qg, idx, flags);
    float v = __fadd_rn(__fmul_rn(momentum, vel[i]), g);  // add(scale(vel, m), g)
    if (nonfinite(v)) flags |= kStatusInvalidValue;        // map_elements check
    v = q_slot(v, qa1, idx, flags);
    vel[i] = v;
    const float lv = __fmul_rn(v, lr);                      // scale(v, lr)
    float a = __fsub_rn(acc[i], lv);                        // sub(acc, .)
    if (nonfinite(lv) || nonfinite(a)) flags |= kStatusInvalidValue;
    a = q_slot(a, qa2, idx, flags);
    acc[i] = a;
    w[i] = q_slot(a, qw, idx, flags);
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(status, flags);
}

// ---- grouped step: many parameter tensors per launch ----------------------
constexpr int kMaxSgd = 64;
constexpr int kSgdPer = 4;                 // elements per thread
constexpr int64_t kSgdTile = (int64_t)kT * kSgdPer;

struct SgdEntry {
  const float* g;
  float* v;
  float* a;
  float* w;
  int64_t n;
  uint64_t base;
  uint64_t key[4];
  int64_t first;  // first CTA of this tensor
};

struct SgdTable {
  SgdEntry e[kMaxSgd];
  Slot q[4];
  int count;
  int64_t ctas;
};

__global__ void __launch_bounds__(kT)
    k_sgd_grouped(const __grid_constant__ SgdTable t, float momentum, float lr,
                  uint32_t* __restrict__ status) {
  int lo = 0, hi = t.count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.e[mid].first <= (int64_t)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const SgdEntry& e = t.e[lo];
  const int64_t t0 = ((int64_t)blockIdx.x - e.first) * kSgdTile;
  uint32_t flags = 0;
  float gv[kSgdPer], vv[kSgdPer], av[kSgdPer];
#pragma unroll
  for (int k = 0; k < kSgdPer; ++k) {  // all loads first (coalesced)
    const int64_t i = t0 + threadIdx.x + (int64_t)k * kT;
    if (i < e.n) {
      gv[k] = __ldcs(e.g + i);
      vv[k] = __ldcs(e.v + i);
      av[k] = __ldcs(e.a + i);
    }
  }
#pragma unroll
  for (int k = 0; k < kSgdPer; ++k) {
    const int64_t i = t0 + threadIdx.x + (int64_t)k * kT;
    if (i < e.n) {
      float w;
      sgd_element(gv[k], vv[k], av[k], w, momentum, lr, t.q, e.key,
                  e.base + (uint64_t)i, flags);
      __stcs(e.v + i, vv[k]);
      __stcs(e.a + i, av[k]);
      __stcs(e.w + i, w);
    }
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(status, flags);
}

// Specialised form for the common slot modes (each slot off, NearestEven or
// Stochastic -- compile-time), 4 consecutive parameters per thread (float4
// loads and stores when the tensor's arrays are 16-byte aligned) and the
// float4-shared variates.  Same per-element semantics as sgd_element.
constexpr int kOff = -1;
constexpr int kSgdV = 4;  // parameters per thread (consecutive)
constexpr int64_t kSgdTileV = (int64_t)kT * kSgdV;

template <int MS>
__device__ __forceinline__ void quant4(float (&x)[kSgdV], const Slot& s, uint64_t key,
                                       uint64_t idx, bool idx4, uint32_t& flags) {
  if (MS == kOff) return;
  uint32_t v[kSgdV] = {0u, 0u, 0u, 0u};
  if (MS == kStochastic) {
    if (idx4) {
      variate24_x4(key, idx, 32u, v);
    } else {
#pragma unroll
      for (int q = 0; q < kSgdV; ++q) v[q] = variate24(key, idx + q);
    }
  }
  constexpr int MF = MS == kOff ? kNearestEven : MS;
#pragma unroll
  for (int q = 0; q < kSgdV; ++q)
    if (nonfinite(x[q])) flags |= kStatusNonFinite;
  // the slot's format dispatch once per 4 elements (uniform), not per
  // element; float slots take the bit-domain form when none of the 4 is in
  // the underflow range (as FloatOp::apply4 in elementwise.cu), same results
  // as q_mode per element
  if (s.kind == LPQ_FLOAT) {
    const FloatParams& p = s.fp;
    if (p.bits_ok && (p.scaled_ok || !p.tiny)) {
      float c[kSgdV];
      bool under = false;
#pragma unroll
      for (int q = 0; q < kSgdV; ++q) {
        c[q] = fminf(fmaxf(x[q], -p.max_value), p.max_value);
        under |= fabsf(c[q]) < p.min_normal && c[q] != 0.0f;
      }
      if (!under) {
#pragma unroll
        for (int q = 0; q < kSgdV; ++q) x[q] = quant_float_bits<MF>(c[q], p, v[q]);
        return;
      }
    }
#pragma unroll
    for (int q = 0; q < kSgdV; ++q) {
      if (p.scaled_ok) x[q] = quant_float_scaled<MF>(x[q], p, v[q]);
      else if (!p.tiny) x[q] = quant_float_fast<MF>(x[q], p, v[q]);
      else x[q] = quant_float<MF>(x[q], p, v[q]);
    }
    return;
  }
  if (s.saturate) {
    if (s.xp.tiny) {
#pragma unroll
      for (int q = 0; q < kSgdV; ++q) x[q] = quant_fixed<MF, true, true>(x[q], s.xp, v[q]);
    } else {
#pragma unroll
      for (int q = 0; q < kSgdV; ++q) x[q] = quant_fixed_sat_fast<MF>(x[q], s.xp, v[q]);
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < kSgdV; ++q) x[q] = quant_fixed<MF, false>(x[q], s.xp, v[q]);
}

template <int MG, int MA, int MW>
__global__ void __launch_bounds__(kT)
    k_sgd_grouped_t(const __grid_constant__ SgdTable t, float momentum, float lr,
                    uint32_t* __restrict__ status) {
  int lo = 0, hi = t.count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.e[mid].first <= (int64_t)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const SgdEntry& e = t.e[lo];
  const int64_t i0 = ((int64_t)blockIdx.x - e.first) * kSgdTileV + (int64_t)threadIdx.x * kSgdV;
  if (i0 >= e.n) return;
  const bool vec = i0 + kSgdV <= e.n &&
      ((reinterpret_cast<uintptr_t>(e.g) | reinterpret_cast<uintptr_t>(e.v) |
        reinterpret_cast<uintptr_t>(e.a) | reinterpret_cast<uintptr_t>(e.w)) & 15u) == 0;
  const int cnt = (int)min((int64_t)kSgdV, e.n - i0);
  float g[kSgdV], v[kSgdV], a[kSgdV];
  if (vec) {
    const float4 g4 = __ldcs(reinterpret_cast<const float4*>(e.g + i0));
    const float4 v4 = __ldcs(reinterpret_cast<const float4*>(e.v + i0));
    const float4 a4 = __ldcs(reinterpret_cast<const float4*>(e.a + i0));
    g[0] = g4.x; g[1] = g4.y; g[2] = g4.z; g[3] = g4.w;
    v[0] = v4.x; v[1] = v4.y; v[2] = v4.z; v[3] = v4.w;
    a[0] = a4.x; a[1] = a4.y; a[2] = a4.z; a[3] = a4.w;
  } else {
#pragma unroll
    for (int q = 0; q < kSgdV; ++q) {
      g[q] = q < cnt ? e.g[i0 + q] : 0.0f;
      v[q] = q < cnt ? e.v[i0 + q] : 0.0f;
      a[q] = q < cnt ? e.a[i0 + q] : 0.0f;
    }
  }
  const uint64_t idx = e.base + (uint64_t)i0;
  const bool idx4 = (idx & 3u) == 0;
  uint32_t flags = 0;
  quant4<MG>(g, t.q[0], e.key[0], idx, idx4, flags);         // g = Qg(grad)
#pragma unroll
  for (int q = 0; q < kSgdV; ++q) {
    v[q] = __fadd_rn(__fmul_rn(momentum, v[q]), g[q]);      // add(scale(vel, m), g)
    if (q < cnt && nonfinite(v[q])) flags |= kStatusInvalidValue;
  }
  quant4<MA>(v, t.q[1], e.key[1], idx, idx4, flags);         // vel = Qa(v)
  float w[kSgdV];
#pragma unroll
  for (int q = 0; q < kSgdV; ++q) {
    const float lv = __fmul_rn(v[q], lr);                   // scale(v, lr)
    a[q] = __fsub_rn(a[q], lv);                             // sub(acc, .)
    if (q < cnt && (nonfinite(lv) || nonfinite(a[q]))) flags |= kStatusInvalidValue;
  }
  quant4<MA>(a, t.q[2], e.key[2], idx, idx4, flags);         // acc = Qa(a)
#pragma unroll
  for (int q = 0; q < kSgdV; ++q) w[q] = a[q];
  quant4<MW>(w, t.q[3], e.key[3], idx, idx4, flags);         // w = Qw(acc)
  if (vec) {
    __stcs(reinterpret_cast<float4*>(e.v + i0), make_float4(v[0], v[1], v[2], v[3]));
    __stcs(reinterpret_cast<float4*>(e.a + i0), make_float4(a[0], a[1], a[2], a[3]));
    __stcs(reinterpret_cast<float4*>(e.w + i0), make_float4(w[0], w[1], w[2], w[3]));
  } else {
#pragma unroll
    for (int q = 0; q < kSgdV; ++q)
      if (q < cnt) {
        e.v[i0 + q] = v[q];
        e.a[i0 + q] = a[q];
        e.w[i0 + q] = w[q];
      }
  }
  // (padding lanes q >= cnt hold zeros: finite, results discarded)
  flags = __reduce_or_sync(__activemask(), flags);
  if (flags) atomicOr(status, flags);
}

// slot mode as a template value: kOff, NearestEven, Stochastic; -2 = other
__host__ inline int fast_mode(const Slot& s) {
  if (!s.enabled) return kOff;
  if (s.mode == kNearestEven || s.mode == kStochastic) return s.mode;
  return -2;
}

template <int MG, int MA>
cudaError_t launch_sgd_w(int mw, const SgdTable& t, float m, float lr,
                         uint32_t* st, cudaStream_t s) {
  const unsigned grid = (unsigned)t.ctas;
  switch (mw) {
    case kOff: k_sgd_grouped_t<MG, MA, kOff><<<grid, kT, 0, s>>>(t, m, lr, st); break;
    case kNearestEven: k_sgd_grouped_t<MG, MA, kNearestEven><<<grid, kT, 0, s>>>(t, m, lr, st); break;
    default: k_sgd_grouped_t<MG, MA, kStochastic><<<grid, kT, 0, s>>>(t, m, lr, st); break;
  }
  return cudaGetLastError();
}
template <int MG>
cudaError_t launch_sgd_a(int ma, int mw, const SgdTable& t, float m, float lr,
                         uint32_t* st, cudaStream_t s) {
  switch (ma) {
    case kOff: return launch_sgd_w<MG, kOff>(mw, t, m, lr, st, s);
    case kNearestEven: return launch_sgd_w<MG, kNearestEven>(mw, t, m, lr, st, s);
    default: return launch_sgd_w<MG, kStochastic>(mw, t, m, lr, st, s);
  }
}
cudaError_t launch_sgd_fast(int mg, int ma, int mw, const SgdTable& t, float m,
                            float lr, uint32_t* st, cudaStream_t s) {
  switch (mg) {
    case kOff: return launch_sgd_a<kOff>(ma, mw, t, m, lr, st, s);
    case kNearestEven: return launch_sgd_a<kNearestEven>(ma, mw, t, m, lr, st, s);
    default: return launch_sgd_a<kStochastic>(ma, mw, t, m, lr, st, s);
  }
}

lpq_status make_slot(const lpq_quant_slot* in, Slot* out) {
  *out = Slot{};
  if (!in || !in->enabled) return LPQ_OK;
  lpq_status st = check_format(&in->format);
  if (st != LPQ_OK) return st;
  if (in->format.kind == LPQ_BLOCK) return LPQ_ERR_UNSUPPORTED;
  if (in->mode < 0 || in->mode > 3) return LPQ_ERR_ARGUMENT;
  out->enabled = 1;
  out->kind = in->format.kind;
  out->mode = in->mode;
  out->saturate = in->format.saturate;
  out->key = stream_key(in->seed, in->call);
  if (in->format.kind == LPQ_FLOAT)
    out->fp = make_float(in->format.exp_bits, in->format.man_bits);
  else
    out->xp = make_fixed(in->format.wl, in->format.fl, in->format.symmetric != 0,
                         in->format.saturate != 0);
  return LPQ_OK;
}

}  // namespace

}  // namespace lpq

using namespace lpq;

extern "C" lpq_status lpq_sgd_step(const float* grad, float* vel, float* acc,
                                   float* weight, int64_t n, float momentum,
                                   float lr, const lpq_quant_slot* grad_q,
                                   const lpq_quant_slot* acc_q_vel,
                                   const lpq_quant_slot* acc_q_acc,
                                   const lpq_quant_slot* weight_q,
                                   uint64_t index_base, uint32_t* d_status,
                                   void* stream) {
  if (n < 0) return LPQ_ERR_ARGUMENT;
  Slot s[4];
  const lpq_quant_slot* in[4] = {grad_q, acc_q_vel, acc_q_acc, weight_q};
  for (int k = 0; k < 4; ++k) {
    lpq_status st = make_slot(in[k], &s[k]);
    if (st != LPQ_OK) return st;
  }
  if (n == 0) return LPQ_OK;
  if (!grad || !vel || !acc || !weight || !d_status) return LPQ_ERR_ARGUMENT;
  const int64_t cap = (int64_t)device_info().sm_count * 8;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cap, (n + kT - 1) / kT));
  k_sgd_step<<<grid, kT, 0, static_cast<cudaStream_t>(stream)>>>(
      grad, vel, acc, weight, n, momentum, lr, s[0], s[1], s[2], s[3], index_base,
      d_status);
  note_launch();
  note_passes(1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

extern "C" lpq_status lpq_sgd_step_grouped(const lpq_sgd_tensor* tensors,
                                           int count, float momentum, float lr,
                                           const lpq_quant_slot* grad_q,
                                           const lpq_quant_slot* acc_q_vel,
                                           const lpq_quant_slot* acc_q_acc,
                                           const lpq_quant_slot* weight_q,
                                           uint32_t* d_status, void* stream) {
  if (count < 0 || (count > 0 && !tensors)) return LPQ_ERR_ARGUMENT;
  SgdTable t{};
  const lpq_quant_slot* in[4] = {grad_q, acc_q_vel, acc_q_acc, weight_q};
  for (int k = 0; k < 4; ++k) {
    lpq_status st = make_slot(in[k], &t.q[k]);
    if (st != LPQ_OK) return st;
  }
  for (int i = 0; i < count; ++i) {
    const lpq_sgd_tensor& d = tensors[i];
    if (d.n < 0) return LPQ_ERR_ARGUMENT;
    if (d.n > 0 && (!d.grad || !d.vel || !d.acc || !d.weight)) return LPQ_ERR_ARGUMENT;
  }
  if (!d_status) return LPQ_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // the two accumulator slots share the spec; both must match for the
  // specialised kernel
  const int mg = fast_mode(t.q[0]), ma = fast_mode(t.q[1]), mw = fast_mode(t.q[3]);
  const bool fast = mg != -2 && ma != -2 && mw != -2 && fast_mode(t.q[2]) == ma;
  const int64_t tile = fast ? kSgdTileV : kSgdTile;
  auto flush = [&]() -> cudaError_t {
    if (t.count == 0) return cudaSuccess;
    cudaError_t e;
    if (fast) {
      e = launch_sgd_fast(mg, ma, mw, t, momentum, lr, d_status, s);
    } else {
      k_sgd_grouped<<<(unsigned)t.ctas, kT, 0, s>>>(t, momentum, lr, d_status);
      e = cudaGetLastError();
    }
    note_launch();
    note_passes(1);
    t.count = 0;
    t.ctas = 0;
    return e;
  };
  for (int i = 0; i < count; ++i) {
    const lpq_sgd_tensor& d = tensors[i];
    if (d.n == 0) continue;
    if (t.count == kMaxSgd) {
      const cudaError_t e = flush();
      if (e != cudaSuccess) return cuda_fail(e);
    }
    SgdEntry& e = t.e[t.count++];
    e.g = d.grad;
    e.v = d.vel;
    e.a = d.acc;
    e.w = d.weight;
    e.n = d.n;
    e.base = d.index_base;
    const uint64_t calls[4] = {d.call_grad, d.call_vel, d.call_acc, d.call_weight};
    for (int k = 0; k < 4; ++k)
      e.key[k] = t.q[k].enabled ? stream_key(in[k]->seed, calls[k]) : 0u;
    e.first = t.ctas;
    t.ctas += (d.n + tile - 1) / tile;
  }
  const cudaError_t e = flush();
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}
