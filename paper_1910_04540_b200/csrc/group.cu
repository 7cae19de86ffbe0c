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
#include <type_traits>
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
constexpr int64_t kMaxRow = 8192;              // longest grouped block row (floats)

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

// Block format along dim 0 (rows of <= kMaxRow floats): one WARP per row,
// 8 rows per CTA.  Pass 1 streams the row (float4 when the rows are 16-byte
// aligned) and reduces max|x| over the warp; pass 2 re-reads it -- 36 KB at
// most per CTA, an L1 / L2 hit, so HBM sees one read and one write -- and
// quantizes with the float4-shared variates.  (One 256-thread CTA per row
// holding 32 floats per thread in registers issued all 32 predicated slots
// for the 64-576-float rows of the ResNet-50 weights: 786 GB/s,
// profiles/r02_group_block_rows_r50w.raw.csv.)
constexpr int kRowsPerCta = kT / 32;

template <int M>
__global__ void __launch_bounds__(kT)
    k_group_block_rows(const __grid_constant__ Table t, int wl,
                       uint32_t* __restrict__ status) {
  const Entry& e = t.e[find_entry(t, blockIdx.x)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r = (blockIdx.x - e.first) * kRowsPerCta + warp;
  const int64_t rows = e.n / e.len;
  if (r >= rows) return;  // (no CTA-wide barriers below)
  const float* __restrict__ x = e.x + r * e.len;
  float* __restrict__ y = e.y + r * e.len;
  const uint64_t rb = e.base + (uint64_t)(r * e.len);
  const bool vec = (e.len & 3) == 0 &&
      ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15u) == 0;
  const int64_t len4 = e.len >> 2;
  float mf = 0.0f, nf = 0.0f;
  if (vec) {
    const float4* __restrict__ x4 = reinterpret_cast<const float4*>(x);
    for (int64_t j = lane; j < len4; j += 32) {
      const float4 v = __ldg(x4 + j);
      absmax_nf(v, mf, nf);
    }
  } else {
    for (int64_t j = lane; j < e.len; j += 32) {
      const float v = __ldg(x + j);
      mf = fmaxf(mf, fabsf(v));
      nf = __fmaf_rn(v, 0.0f, nf);
    }
  }
  const uint32_t m = __reduce_max_sync(kFull, f2u(mf));
  const BlockScale sc = make_block_scale(m, wl);
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const RngMul rm = rng_mul();
  auto run = [&](auto two_t) {
    constexpr bool TWO = decltype(two_t)::value;
    if (vec) {
      const float4* __restrict__ x4 = reinterpret_cast<const float4*>(x);
      float4* __restrict__ y4 = reinterpret_cast<float4*>(y);
      if ((rb & 3u) == 0) {
        for (int64_t j = lane; j < len4; j += 32)
          __stcs(y4 + j, qb4<M, TWO, true>(__ldcs(x4 + j), sc, kmin, kmax, e.key,
                                           rb + 4 * j, rm));
      } else {
        for (int64_t j = lane; j < len4; j += 32)
          __stcs(y4 + j, qb4<M, TWO, false>(__ldcs(x4 + j), sc, kmin, kmax, e.key,
                                            rb + 4 * j, rm));
      }
    } else {
      for (int64_t j = lane; j < e.len; j += 32)
        y[j] = qb<M, TWO>(__ldcs(x + j), sc, kmin, kmax, e.key ^ (rb + j), rm);
    }
  };
  if (two_factor(sc)) run(std::true_type{});
  else run(std::false_type{});
  const uint32_t bad = __reduce_or_sync(kFull, (sc.bad ? 2u : 0u) | (nf != nf ? 1u : 0u));
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
    t.ctas += f->kind == LPQ_BLOCK ? (g.extent + kRowsPerCta - 1) / kRowsPerCta
                                   : (n + kTile - 1) / kTile;
  }
  return flush();
}
