// group.cu -- grouped (multi-tensor) quantization: many tensors, one launch.
//
// A training step quantizes every parameter and gradient tensor (ResNet-50:
// 54 + 54 tensors of 9K-2.4M elements); one launch per
// tensor costs more in launch latency than the small tensors cost in HBM
// time.  lpq_quantize_grouped quantizes up to kMaxGroup tensors per launch:
// the tensor table travels in the kernel parameters (so the call is
// graph-capturable and needs no device copy), the grid is the concatenation
// of every tensor's tiles (elementwise formats) or rows (block format along
// dim 0), and each CTA finds its tensor by a binary search over the prefix
// table.  Each tensor i is quantize_fused_at(t_i, {format, mode, seed},
// call_i) with flat-index variates from index_base_i (quant_ops.cpp:154-164).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "../../include/lpq.h"
#include "block_common.cuh"
#include "kernels.cuh"
#include "runtime.h"

namespace lpq {

namespace {

using namespace blk;

constexpr int kMaxGroup = 64;
constexpr int kT = 256;
constexpr int kEwU = 8;                        // float4 per thread (elementwise)
constexpr int64_t kTile = (int64_t)kT * kEwU * 4;  // elements per CTA
constexpr int kRowV = 32;                      // floats per thread (block rows)
constexpr int64_t kMaxRow = (int64_t)kT * kRowV;   // 8192

struct Entry {
  const float* x;
  float* y;
  int64_t n;       // elements
  int64_t len;     // block row length (block formats)
  uint64_t base;   // flat index of x[0]
  uint64_t key;    // stream_key(seed, call_i)
  int64_t first;   // first CTA of this tensor
};

struct Table {
  Entry e[kMaxGroup];
  int count;
  int64_t ctas;
};

__device__ __forceinline__ int find_entry(const Table& t, int64_t b) {
  int lo = 0, hi = t.count - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.e[mid].first <= b) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// the streaming element forms of elementwise.cu, picked by the (uniform)
// format parameters
struct FixOp {
  FixedParams p;
  template <int M> __device__ __forceinline__ float apply(float x, uint32_t v) const {
    if (p.saturate) {
      if (p.tiny) return quant_fixed<M, true, true>(x, p, v);
      return quant_fixed_sat_fast<M>(x, p, v);
    }
    return quant_fixed<M, false>(x, p, v);
  }
};
struct FltOp {
  FloatParams p;
  template <int M> __device__ __forceinline__ float apply(float x, uint32_t v) const {
    constexpr bool kFast = M == kNearestEven || M == kStochastic;
    constexpr int MF = kFast ? M : kNearestEven;
    if (kFast) return quant_float_stream<MF>(x, p, v);
    return quant_float<M>(x, p, v);
  }
};

template <int M, class Op>
__global__ void __launch_bounds__(kT)
    k_group_elementwise(const __grid_constant__ Table t, Op op,
                        uint32_t* __restrict__ status) {
  const Entry& e = t.e[find_entry(t, blockIdx.x)];
  const int64_t t0 = (blockIdx.x - e.first) * kTile;
  const int64_t len = min(kTile, e.n - t0);
  const float* __restrict__ x = e.x + t0;
  float* __restrict__ y = e.y + t0;
  float nf = 0.0f;
  const bool vec = len == kTile &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u) == 0;
  if (vec) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    float4* y4 = reinterpret_cast<float4*>(y);
    float4 v[kEwU];
#pragma unroll
    for (int u = 0; u < kEwU; ++u) v[u] = __ldcs(x4 + threadIdx.x + u * kT);
    const bool idx4 = (e.base & 3u) == 0;  // uniform per tensor
#pragma unroll
    for (int u = 0; u < kEwU; ++u) {
      const int64_t j = threadIdx.x + u * kT;
      const uint64_t idx = e.base + (uint64_t)(t0 + 4 * j);
      float4 o;
      const float* vi = reinterpret_cast<const float*>(&v[u]);
      float* oi = reinterpret_cast<float*>(&o);
      uint32_t r[4] = {0u, 0u, 0u, 0u};
      if (M == kStochastic) {
        if (idx4) {
          variate24_x4(e.key, idx, 32u, r);
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) r[q] = variate24(e.key, idx + q);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        nf = __fmaf_rn(vi[q], 0.0f, nf);
        oi[q] = op.template apply<M>(vi[q], r[q]);
      }
      __stcs(y4 + j, o);
    }
  } else {
    for (int64_t j = threadIdx.x; j < len; j += kT) {
      const float xv = x[j];
      uint32_t r = 0;
      if (M == kStochastic) r = variate24(e.key, e.base + (uint64_t)(t0 + j));
      nf = __fmaf_rn(xv, 0.0f, nf);
      y[j] = op.template apply<M>(xv, r);
    }
  }
  if (__any_sync(0xFFFFFFFFu, nf != nf) && (threadIdx.x & 31) == 0)
    atomicOr(status, kStatusNonFinite);
}

// block format along dim 0: one CTA per row (row length <= kMaxRow floats)
template <int M>
__global__ void __launch_bounds__(kT)
    k_group_block_rows(const __grid_constant__ Table t, int wl,
                       uint32_t* __restrict__ status) {
  __shared__ uint32_t red[kT / 32];
  __shared__ uint32_t row_max;
  const Entry& e = t.e[find_entry(t, blockIdx.x)];
  const int64_t r = blockIdx.x - e.first;
  const float* __restrict__ x = e.x + r * e.len;
  float* __restrict__ y = e.y + r * e.len;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float v[kRowV];
  float mf = 0.0f, nf = 0.0f;
#pragma unroll
  for (int k = 0; k < kRowV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * kT;
    v[k] = j < e.len ? __ldcs(x + j) : 0.0f;
    mf = fmaxf(mf, fabsf(v[k]));
    nf = __fmaf_rn(v[k], 0.0f, nf);
  }
  uint32_t m = __reduce_max_sync(kFull, f2u(mf));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (warp == 0) {
    uint32_t tt = lane < kT / 32 ? red[lane] : 0u;
    tt = __reduce_max_sync(kFull, tt);
    if (lane == 0) row_max = tt;
  }
  __syncthreads();
  const BlockScale sc = make_block_scale(row_max, wl);
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const uint64_t rb = e.base + (uint64_t)(r * e.len);
  const RngMul rm = rng_mul();
#pragma unroll
  for (int k = 0; k < kRowV; ++k) {
    const int64_t j = threadIdx.x + (int64_t)k * kT;
    if (j < e.len)
      y[j] = two_factor(sc) ? qb<M, true>(v[k], sc, kmin, kmax, e.key ^ (rb + j), rm)
                            : qb<M, false>(v[k], sc, kmin, kmax, e.key ^ (rb + j), rm);
  }
  uint32_t bad = (sc.bad ? 2u : 0u) | (nf != nf ? 1u : 0u);
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0 && bad) atomicOr(status, bad);
}

template <int M>
cudaError_t launch_group_m(const Table& t, const lpq_format* f, uint32_t* st,
                           cudaStream_t s) {
  const unsigned grid = (unsigned)t.ctas;
  if (f->kind == LPQ_BLOCK) {
    k_group_block_rows<M><<<grid, kT, 0, s>>>(t, f->wl, st);
  } else if (f->kind == LPQ_FIXED) {
    const FixOp op{make_fixed(f->wl, f->fl, f->symmetric != 0, f->saturate != 0)};
    k_group_elementwise<M, FixOp><<<grid, kT, 0, s>>>(t, op, st);
  } else {
    const FltOp op{make_float(f->exp_bits, f->man_bits)};
    k_group_elementwise<M, FltOp><<<grid, kT, 0, s>>>(t, op, st);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_group(const Table& t, const lpq_format* f, int mode,
                         uint32_t* st, cudaStream_t s) {
  switch (mode) {
    case kStochastic: return launch_group_m<kStochastic>(t, f, st, s);
    case kNearestAway: return launch_group_m<kNearestAway>(t, f, st, s);
    case kNearestZero: return launch_group_m<kNearestZero>(t, f, st, s);
    default: return launch_group_m<kNearestEven>(t, f, st, s);
  }
}

}  // namespace

}  // namespace lpq

using namespace lpq;

extern "C" lpq_status lpq_quantize_grouped(const lpq_tensor_desc* tensors,
                                           int count, const lpq_format* f,
                                           int mode, uint64_t seed, void* ws,
                                           size_t ws_bytes, uint32_t* d_status,
                                           void* stream) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  if (count < 0 || (count > 0 && !tensors) || mode < 0 || mode > 3 || !d_status)
    return LPQ_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const bool groupable = f->kind != LPQ_BLOCK || f->block_dim == 0;
  Table t{};
  auto flush = [&]() -> lpq_status {
    if (t.count == 0) return LPQ_OK;
    const cudaError_t e = launch_group(t, f, mode, d_status, s);
    note_passes(1);
    t = Table{};
    return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
  };
  for (int i = 0; i < count; ++i) {
    const lpq_tensor_desc& d = tensors[i];
    int64_t n = 0;
    st = check_shape(d.shape, d.rank, &n);
    if (st != LPQ_OK) return st;
    BlockGeom g{1, 1, n};
    if (f->kind == LPQ_BLOCK) {
      st = block_geometry(f, d.shape, d.rank, &g);
      if (st != LPQ_OK) return st;
    }
    if (n == 0) continue;
    if (!d.x || !d.y || ((reinterpret_cast<uintptr_t>(d.x) | reinterpret_cast<uintptr_t>(d.y)) & 3u))
      return LPQ_ERR_ARGUMENT;
    const bool rows_ok = f->kind != LPQ_BLOCK || (g.outer == 1 && g.stride <= kMaxRow);
    if (!groupable || !rows_ok) {
      // outside the grouped kernels' reach: the single-tensor path
      st = quantize_device(d.x, d.y, d.shape, d.rank, d.index_base, f, mode,
                           seed, d.call, ws, ws_bytes, d_status, s);
      if (st != LPQ_OK) return st;
      continue;
    }
    if (t.count == kMaxGroup) {
      st = flush();
      if (st != LPQ_OK) return st;
    }
    Entry& e = t.e[t.count++];
    e.x = d.x;
    e.y = d.y;
    e.n = n;
    e.len = f->kind == LPQ_BLOCK ? g.stride : 0;
    e.base = d.index_base;
    e.key = stream_key(seed, d.call);
    e.first = t.ctas;
    t.ctas += f->kind == LPQ_BLOCK ? g.extent : (n + kTile - 1) / kTile;
  }
  return flush();
}
