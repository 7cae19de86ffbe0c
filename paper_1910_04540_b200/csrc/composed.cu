// composed.cu -- the many-kernel quantizer (the paper's baseline, PAPER.md:
// 135-147; the reference's quantize_composed, proj/src/quant_ops.cpp:117-150).
//
// The same quantization expressed as a chain of generic tensor operations,
// each its own kernel and full HBM pass with its own temporary -- scale,
// round, clamp/wrap, scale for fixed point; abs, reduce, block_shift,
// broadcast, ldexp, round, clamp, ldexp for block floating point -- with the
// per-op fp32 semantics of proj/src/tensor.cpp (map_elements validation:
// non-finite results raise invalid_value_error).  It exists to reproduce the
// paper's fused-vs-many-kernel comparison on B200 and to back the drop-in's
// quantize_composed; it is bit-identical to the fused kernels on finite,
// in-range inputs (the reference's own fused == composed property).
#include <cuda_runtime.h>

#include <algorithm>

#include "../../include/lpq.h"
#include "kernels.cuh"
#include "runtime.h"

namespace lpq {

namespace {

constexpr int kT = 256;
constexpr uint32_t kInvalidValue = kStatusInvalidValue;  // map_elements

int grid_for(int64_t n) {
  const int64_t cap = (int64_t)device_info().sm_count * 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(cap, (n + kT - 1) / kT));
}

// y[i] = op(a[i], b[i], i, flags); flags OR-ed into *status.
template <class Op>
__global__ void __launch_bounds__(kT)
    k_map(const float* __restrict__ a, const float* __restrict__ b,
          float* __restrict__ y, int64_t n, Op op,
          uint32_t* __restrict__ status) {
  uint32_t flags = 0;
  for (int64_t i = (int64_t)blockIdx.x * kT + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kT)
    y[i] = op(a[i], b ? b[i] : 0.0f, i, flags);
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(status, flags);
}

template <class Op>
void map(const float* a, const float* b, float* y, int64_t n, const Op& op,
         uint32_t* status, cudaStream_t s) {
  if (n <= 0) return;
  k_map<Op><<<grid_for(n), kT, 0, s>>>(a, b, y, n, op, status);
  note_launch();
  note_passes(1);
}

__device__ __forceinline__ uint32_t result_flag(float v) {
  return nonfinite(v) ? kInvalidValue : 0u;
}

struct ScaleOp {  // tensor.cpp:169-175: float(double(x) * double(s))
  float s;
  __device__ float operator()(float x, float, int64_t, uint32_t& f) const {
    const float v = __fmul_rn(x, s);  // one rounding of the exact product
    f |= result_flag(v);
    return v;
  }
};

template <int M>
struct RoundNearestOp {  // tensor.cpp:208-224 (round_integer_m in double)
  __device__ float operator()(float x, float, int64_t, uint32_t& f) const {
    if (nonfinite(x)) {
      f |= kStatusNonFinite;
      return 0.0f;
    }
    const bool neg = x < 0.0f;
    const float kmag = round_mag<M, false>(fabsf(x), neg, x != 0.0f, 0u);
    const bool kneg = kmag == 0.0f ? zero_negative<M>(neg) : neg;
    return kneg ? -kmag : kmag;
  }
};

struct StochasticRoundOp {  // tensor.cpp:226-239: floor(r) + (u < r - floor(r))
  __device__ float operator()(float x, float u, int64_t, uint32_t& f) const {
    if (nonfinite(x)) {
      f |= kStatusNonFinite;
      return 0.0f;
    }
    const uint32_t v = (uint32_t)(u * 16777216.0f);  // u is on the 2^-24 grid
    return __fadd_rn(round_signed<kStochastic>(x, v), 0.0f);  // -0 -> +0
  }
};

struct ClampOp {  // tensor.cpp:198-206
  float lo, hi;
  __device__ float operator()(float x, float, int64_t, uint32_t& f) const {
    float v = x;
    if (v > hi) v = hi;
    if (v < lo) v = lo;
    f |= result_flag(v);
    return v;
  }
};

struct WrapOp {  // tensor.cpp:241-251: fixed_fold with wl, fl = 0
  FixedParams p;
  __device__ float operator()(float x, float, int64_t, uint32_t& f) const {
    if (nonfinite(x)) {
      f |= kStatusNonFinite;
      return 0.0f;
    }
    return fold_wrap(fabsf(x), signbit(x) != 0, p, 1.0f);
  }
};

struct AbsOp {  // tensor.cpp:191-196
  __device__ float operator()(float x, float, int64_t, uint32_t& f) const {
    const float v = fabsf(x);
    f |= result_flag(v);
    return v;
  }
};

struct VariateOp {  // variate_tensor, tensor.cpp:281-290
  uint64_t key, base;
  __device__ float operator()(float, float, int64_t i, uint32_t&) const {
    return variate_float(variate24(key, base + (uint64_t)i));
  }
};

struct BlockShiftOp {  // tensor.cpp:263-279
  int wl;
  __device__ float operator()(float m, float, int64_t, uint32_t& f) const {
    if (nonfinite(m)) {
      f |= kStatusNonFinite;
      return 0.0f;
    }
    if (m == 0.0f) return 0.0f;
    const uint32_t b = f2u(m) & 0x7FFFFFFFu;
    const int field = (int)(b >> 23);
    const int E = field ? field - 127 : -118 - __clz((int)b);
    if (E > 126) {
      f |= kStatusBlockRange;
      return 0.0f;
    }
    return (float)((wl - 2) - E);
  }
};

struct BroadcastOp {  // tensor.cpp:292-318: out[i] = v[(i / stride) % extent]
  const float* v;
  int64_t stride, extent;
  __device__ float operator()(float, float, int64_t i, uint32_t&) const {
    return v[(i / stride) % extent];
  }
};

struct LdexpOp {  // tensor.cpp:253-261: float(ldexp(double(x), dir * int(e)))
  int dir;
  __device__ float operator()(float x, float e, int64_t, uint32_t& f) const {
    const float v = __double2float_rn(scalbn((double)x, dir * (int)e));
    f |= result_flag(v);
    return v;
  }
};

}  // namespace

size_t composed_workspace(const BlockGeom& g, bool block) {
  const int64_t n = g.outer * g.extent * g.stride;
  const size_t full = sizeof(float) * (size_t)std::max<int64_t>(n, 1);
  const size_t small = sizeof(float) * (size_t)std::max<int64_t>(g.extent, 1);
  const size_t pad = 256;
  // three full temporaries (+ maxima and shifts for block formats)
  return 3 * ((full + pad - 1) / pad * pad) +
         (block ? 2 * ((small + pad - 1) / pad * pad) : 0);
}

lpq_status quantize_composed_device(const float* x, float* y,
                                    const int64_t* shape, int rank,
                                    uint64_t index_base, const lpq_format* f,
                                    int mode, uint64_t seed, uint64_t call,
                                    void* ws, size_t ws_bytes,
                                    uint32_t* status, cudaStream_t s) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  if (f->kind == LPQ_FLOAT) return LPQ_ERR_UNSUPPORTED;  // quant_ops.cpp:169-171
  int64_t n = 0;
  st = check_shape(shape, rank, &n);
  if (st != LPQ_OK) return st;
  if (mode < 0 || mode > 3) return LPQ_ERR_ARGUMENT;
  BlockGeom g{1, 1, n};
  if (f->kind == LPQ_BLOCK) {
    st = block_geometry(f, shape, rank, &g);
    if (st != LPQ_OK) return st;
  }
  if (n == 0) return LPQ_OK;
  if (!x || !y || !status) return LPQ_ERR_ARGUMENT;
  const size_t need = composed_workspace(g, f->kind == LPQ_BLOCK);
  if (!ws || ws_bytes < need) return LPQ_ERR_WORKSPACE;
  const size_t full = (sizeof(float) * (size_t)n + 255) / 256 * 256;
  float* t0 = static_cast<float*>(ws);
  float* t1 = reinterpret_cast<float*>(static_cast<char*>(ws) + full);
  float* t2 = reinterpret_cast<float*>(static_cast<char*>(ws) + 2 * full);
  const uint64_t key = stream_key(seed, call);
  auto round_into = [&](const float* in, float* out) {
    if (mode == kStochastic) {
      map(nullptr, nullptr, t2, n, VariateOp{key, index_base}, status, s);
      map(in, t2, out, n, StochasticRoundOp{}, status, s);
    } else if (mode == kNearestAway) {
      map(in, nullptr, out, n, RoundNearestOp<kNearestAway>{}, status, s);
    } else if (mode == kNearestZero) {
      map(in, nullptr, out, n, RoundNearestOp<kNearestZero>{}, status, s);
    } else {
      map(in, nullptr, out, n, RoundNearestOp<kNearestEven>{}, status, s);
    }
  };
  if (f->kind == LPQ_FIXED) {  // composed_fixed, quant_ops.cpp:117-131
    const float up = u2f((uint32_t)(127 + f->fl) << 23);
    const float down = u2f((uint32_t)(127 - f->fl) << 23);
    map(x, nullptr, t0, n, ScaleOp{up}, status, s);
    round_into(t0, t1);
    const FixedParams p = make_fixed(f->wl, 0, f->symmetric != 0, false);
    if (f->saturate)
      map(t1, nullptr, t0, n, ClampOp{p.kmin, p.kmax}, status, s);
    else
      map(t1, nullptr, t0, n, WrapOp{p}, status, s);
    map(t0, nullptr, y, n, ScaleOp{down}, status, s);
    return LPQ_OK;
  }
  // composed_block, quant_ops.cpp:133-150
  const size_t small = (sizeof(float) * (size_t)g.extent + 255) / 256 * 256;
  uint32_t* maxima = reinterpret_cast<uint32_t*>(static_cast<char*>(ws) + 3 * full);
  float* shifts = reinterpret_cast<float*>(static_cast<char*>(ws) + 3 * full + small);
  map(x, nullptr, t0, n, AbsOp{}, status, s);                    // magnitudes
  cudaError_t e = launch_block_reduce(t0, g, maxima, s);       // maxima
  if (e != cudaSuccess) return cuda_fail(e);
  note_passes(1);
  map(reinterpret_cast<const float*>(maxima), nullptr, shifts, g.extent,
      BlockShiftOp{f->wl}, status, s);
  map(nullptr, nullptr, t1, n, BroadcastOp{shifts, g.stride, g.extent}, status, s);
  map(x, t1, t0, n, LdexpOp{+1}, status, s);                     // scaled
  round_into(t0, y);                                             // rounded
  const float kmax = (float)((1 << (f->wl - 1)) - 1);
  const float kmin = -(float)(1 << (f->wl - 1));
  map(y, nullptr, t0, n, ClampOp{kmin, kmax}, status, s);         // clamped
  map(t0, t1, y, n, LdexpOp{-1}, status, s);
  return cudaGetLastError() == cudaSuccess ? LPQ_OK : LPQ_ERR_CUDA;
}

}  // namespace lpq

using namespace lpq;

extern "C" {

size_t lpq_composed_workspace_size(const lpq_format* f, const int64_t* shape,
                                   int rank) {
  if (!f || check_format(f) != LPQ_OK) return 0;
  int64_t n = 0;
  if (check_shape(shape, rank, &n) != LPQ_OK) return 0;
  BlockGeom g{1, 1, n};
  if (f->kind == LPQ_BLOCK && block_geometry(f, shape, rank, &g) != LPQ_OK) return 0;
  return composed_workspace(g, f->kind == LPQ_BLOCK);
}

lpq_status lpq_quantize_composed(const float* x, float* y, const int64_t* shape,
                                 int rank, uint64_t index_base,
                                 const lpq_format* f, int mode, uint64_t seed,
                                 uint64_t call, void* ws, size_t ws_bytes,
                                 uint32_t* d_status, void* stream) {
  return quantize_composed_device(x, y, shape, rank, index_base, f, mode, seed,
                                  call, ws, ws_bytes, d_status,
                                  static_cast<cudaStream_t>(stream));
}

}  // extern "C"
