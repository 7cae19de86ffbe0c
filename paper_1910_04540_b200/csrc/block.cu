// block.cu -- block-floating-point quantizers (shared exponent per block).
//
// Replaces fused_block (proj/src/quant_ops.cpp:68-115) and the block-maximum
// reduction it calls, reduce_max_abs (proj/src/tensor.cpp:320-353).  The
// tensor is viewed as [outer, extent, stride]; block b is the slice at index
// b along `extent` (formats.hpp:69-78).  Three plans:
//
//  * kRowsInRegisters (outer == 1, contiguous block <= 32768 floats, aligned):
//    ONE HBM pass.  Rows <= 512 floats: a group of <= 32 lanes per row, several
//    rows per warp.  Longer rows: one CTA per block ("row"): the row is loaded into
//    registers with 128-bit loads, max-reduced with warp REDUX + shared
//    memory, the shared exponent derived in registers, the row quantized and
//    stored.  8 algorithmic bytes per element.  (BASELINE config C3.)
//  * kTwoPassSegments (stride >= 1024): pass 1 reduces 4096-element pieces
//    of each contiguous segment to one atomicMax on the block's maximum;
//    pass 2 re-reads and quantizes with one shared scale per piece.
//  * kTwoPassColumns (stride < 1024): the tensor as a [outer, extent*stride]
//    matrix; each thread owns 4 columns for a chunk of rows and keeps their
//    maxima in registers (shared-memory atomics once per column, global
//    atomics once per block touched); pass 2 derives each column's scale once
//    and streams the rows.
//  Two-pass plans move 12 algorithmic bytes per element.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "block_common.cuh"
#include "kernels.cuh"

namespace lpq {

namespace {
using namespace blk;

// ---------------------------------------------------------------------------
// Plan 1: one row per CTA, held in registers (single HBM pass).
// T threads, VPT float4 per thread; row length L (multiple of 4, <= 4*T*VPT).
// FULL: L == 4*T*VPT (no bounds tests).  The row maximum propagates NaN
// (absmax_nan); a NaN row recomputes the NaN-ignoring maximum of
// reduce_max_abs and flags the non-finite input.  Three element loops per
// block class: two-factor scales, single factor with the stochastic flush
// guard (s1 < 1), single factor without.
template <int T>
__device__ __forceinline__ uint32_t cta_max(uint32_t m, uint32_t* red,
                                            uint32_t* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  m = __reduce_max_sync(kFull, m);  // non-negative floats: uint order
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < T / 32 ? red[lane] : 0u;
    t = __reduce_max_sync(kFull, t);
    if (lane == 0) *out = t;
  }
  __syncthreads();
  return *out;
}

template <int M, int T, int VPT, bool IDX4, bool FULL>
__global__ void __launch_bounds__(T)
    k_block_rows(const float* __restrict__ x, float* __restrict__ y, int64_t L,
                 int64_t nrows, uint64_t base, uint64_t key, int wl,
                 RngMul m32, uint32_t* __restrict__ status) {
  __shared__ uint32_t red[T / 32];
  __shared__ uint32_t row_max;
  const int lane = threadIdx.x & 31;
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const int64_t L4 = L >> 2;
  uint32_t bad = 0;
  for (int64_t r = blockIdx.x; r < nrows; r += gridDim.x) {
    const float4* __restrict__ xr = reinterpret_cast<const float4*>(x + r * L);
    float4* __restrict__ yr = reinterpret_cast<float4*>(y + r * L);
    float4 v[VPT];
    float mf = 0.0f;
#pragma unroll
    for (int k = 0; k < VPT; ++k) {
      const int64_t j = threadIdx.x + (int64_t)k * T;
      if (FULL || j < L4) {
        v[k] = __ldcs(xr + j);
        absmax_nan(v[k], mf);
      }
    }
    uint32_t m = cta_max<T>(f2u(mf), red, &row_max);
    if (m > 0x7F800000u) {  // NaN in the row (uniform): slow path
      bad |= 1u;
      float nf = 0.0f;
      mf = 0.0f;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int64_t j = threadIdx.x + (int64_t)k * T;
        if (FULL || j < L4) absmax_nf(v[k], mf, nf);
      }
      __syncthreads();  // row_max is rewritten
      m = cta_max<T>(f2u(mf), red, &row_max);
    }
    const BlockScale sc = make_block_scale(m, wl);
    if (sc.bad) bad |= 2u;
    const uint64_t row_base = base + (uint64_t)(r * L);
    auto run = [&](auto two_t, auto guard_t) {
      constexpr bool TWO = decltype(two_t)::value;
      constexpr bool GUARD = decltype(guard_t)::value;
#pragma unroll
      for (int k = 0; k < VPT; ++k) {
        const int64_t j = threadIdx.x + (int64_t)k * T;
        if (FULL || j < L4)
          __stcs(yr + j, qb4<M, TWO, IDX4, GUARD>(v[k], sc, kmin, kmax, key,
                                                  row_base + 4 * j, m32));
      }
    };
    if (two_factor(sc)) run(std::true_type{}, std::false_type{});
    else if (M == kStochastic && needs_guard(sc)) run(std::false_type{}, std::true_type{});
    else run(std::false_type{}, std::false_type{});
    __syncthreads();  // red/row_max are reused by the next row
  }
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0) flag(status, bad);
}

// Short rows (L <= 512 floats): G lanes per row (G a power of two <= 32),
// V float4 per lane, R rows per lane group (their loads all in flight
// together), 32/G groups per warp, 8 warps per CTA; the row maximum is a
// butterfly over the row's G lanes.  (One CTA per 64-float row would leave
// most of each CTA idle and make the launch CTA-rate-bound.)  Iteration i
// of a warp covers 32/G consecutive rows, so its loads are contiguous.
template <int M, int G, int V, int R, bool IDX4>
__global__ void __launch_bounds__(256)
    k_block_rows_small(const float* __restrict__ x, float* __restrict__ y,
                       int64_t L, int64_t nrows, uint64_t base, uint64_t key,
                       int wl, RngMul m32, uint32_t* __restrict__ status) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane % G;
  const int64_t L4 = L >> 2;
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + warp) * R * (32 / G) + lane / G;
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  float4 v[R][V];
  float nf = 0.0f;
  uint32_t m[R];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t r = r0 + (int64_t)i * (32 / G);
    const float4* __restrict__ xr = reinterpret_cast<const float4*>(x + r * L);
    float mf = 0.0f;
#pragma unroll
    for (int k = 0; k < V; ++k) {
      const int64_t j = g + (int64_t)k * G;
      v[i][k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < nrows && j < L4) {
        v[i][k] = __ldcs(xr + j);
        absmax_nf(v[i][k], mf, nf);
      }
    }
    m[i] = f2u(mf);
  }
  uint32_t bad = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int64_t r = r0 + (int64_t)i * (32 / G);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) m[i] = max(m[i], __shfl_xor_sync(kFull, m[i], o));
    if (r >= nrows) continue;
    const BlockScale sc = make_block_scale(m[i], wl);
    if (sc.bad) bad |= 2u;
    float4* __restrict__ yr = reinterpret_cast<float4*>(y + r * L);
    const uint64_t row_base = base + (uint64_t)(r * L);
    // block-class loops (see k_block_rows); the class is per row, so it may
    // differ between the rows of a warp
    auto run = [&](auto two_t, auto guard_t) {
      constexpr bool TWO = decltype(two_t)::value;
      constexpr bool GUARD = decltype(guard_t)::value;
#pragma unroll
      for (int k = 0; k < V; ++k) {
        const int64_t j = g + (int64_t)k * G;
        if (j < L4)
          __stcs(yr + j, qb4<M, TWO, IDX4, GUARD>(v[i][k], sc, kmin, kmax, key,
                                                  row_base + 4 * j, m32));
      }
    };
    if (two_factor(sc)) run(std::true_type{}, std::false_type{});
    else if (M == kStochastic && needs_guard(sc)) run(std::false_type{}, std::true_type{});
    else run(std::false_type{}, std::false_type{});
  }
  if (nf != nf) bad |= 1u;
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0) flag(status, bad);
}

template <int M, int G, int V>
void launch_rows_small_t(const float* x, float* y, int64_t L, int64_t nrows,
                         uint64_t base, uint64_t key, int wl, uint32_t* st,
                         cudaStream_t s) {
  // several rows per lane group pays for nearest rounding (more loads in
  // flight: [2^22, 64] 0.365 -> 0.353 ms) but not for stochastic, which is
  // issue-bound (0.504 -> 0.533 ms)
  constexpr int R = M == kStochastic ? 1 : (V == 1 ? 4 : (V == 2 ? 2 : 1));
  const int64_t per_cta = 8 * R * (32 / G);
  const int grid = (int)std::max<int64_t>(
      1, std::min<int64_t>((nrows + per_cta - 1) / per_cta, 0x7FFFFFFF));
  if ((base & 3u) == 0)
    k_block_rows_small<M, G, V, R, true><<<grid, 256, 0, s>>>(x, y, L, nrows, base, key, wl, rng_mul(), st);
  else
    k_block_rows_small<M, G, V, R, false><<<grid, 256, 0, s>>>(x, y, L, nrows, base, key, wl, rng_mul(), st);
  note_launch();
}

template <int M, int T, int VPT>
void launch_rows_t(const float* x, float* y, int64_t L, int64_t nrows,
                   uint64_t base, uint64_t key, int wl, uint32_t* st,
                   cudaStream_t s) {
  // one CTA per row, all rows launched (CTAs retire in address order)
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nrows, 0x7FFFFFFF));
  const bool full = (L >> 2) == (int64_t)T * VPT;
  if ((base & 3u) == 0 && full)
    k_block_rows<M, T, VPT, true, true><<<grid, T, 0, s>>>(x, y, L, nrows, base, key, wl, rng_mul(), st);
  else if ((base & 3u) == 0)
    k_block_rows<M, T, VPT, true, false><<<grid, T, 0, s>>>(x, y, L, nrows, base, key, wl, rng_mul(), st);
  else
    k_block_rows<M, T, VPT, false, false><<<grid, T, 0, s>>>(x, y, L, nrows, base, key, wl, rng_mul(), st);
  note_launch();
}

template <int M>
void launch_rows(const float* x, float* y, int64_t L, int64_t nrows,
                 uint64_t base, uint64_t key, int wl, uint32_t* st,
                 cudaStream_t s) {
  const int64_t L4 = L >> 2;
  if (M == kStochastic && L4 <= 64) {
    // issue-bound: 4 float4 per lane, so the per-row work (butterfly, scale)
    // is shared by 16 elements per thread rather than 4
    if (L4 <= 4) launch_rows_small_t<M, 1, 4>(x, y, L, nrows, base, key, wl, st, s);
    else if (L4 <= 8) launch_rows_small_t<M, 2, 4>(x, y, L, nrows, base, key, wl, st, s);
    else if (L4 <= 16) launch_rows_small_t<M, 4, 4>(x, y, L, nrows, base, key, wl, st, s);
    else if (L4 <= 32) launch_rows_small_t<M, 8, 4>(x, y, L, nrows, base, key, wl, st, s);
    else launch_rows_small_t<M, 16, 4>(x, y, L, nrows, base, key, wl, st, s);
    return;
  }
  if (L4 <= 1) launch_rows_small_t<M, 1, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 2) launch_rows_small_t<M, 2, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 4) launch_rows_small_t<M, 4, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 8) launch_rows_small_t<M, 8, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 16) launch_rows_small_t<M, 16, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 32) launch_rows_small_t<M, 32, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 64) launch_rows_small_t<M, 32, 2>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 128) launch_rows_small_t<M, 32, 4>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 256) launch_rows_t<M, 256, 1>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 512) launch_rows_t<M, 256, 2>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 1024) launch_rows_t<M, 128, 8>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 2048) launch_rows_t<M, 512, 4>(x, y, L, nrows, base, key, wl, st, s);
  else if (L4 <= 4096) launch_rows_t<M, 1024, 4>(x, y, L, nrows, base, key, wl, st, s);
  else launch_rows_t<M, 1024, 8>(x, y, L, nrows, base, key, wl, st, s);
}

// ---------------------------------------------------------------------------
// Plan 2: long contiguous segments (stride >= 1024).  Work item = a piece of
// kPiece elements inside one segment; every element of a piece shares b.
constexpr int kSegT = 256;
constexpr int kPiece = kSegT * 4 * 4;  // 4096 elements, 4 float4 per thread

template <bool VEC>
__global__ void __launch_bounds__(kSegT)
    k_seg_reduce(const float* __restrict__ x, int64_t nseg, int64_t stride,
                 int64_t extent, int64_t pieces, uint32_t* __restrict__ maxima) {
  __shared__ uint32_t red[kSegT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t items = nseg * pieces;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t seg = it / pieces, pc = it - seg * pieces;
    const int64_t off = pc * kPiece;
    const int64_t len = min((int64_t)kPiece, stride - off);
    const float* xs = x + seg * stride + off;
    uint32_t m = 0;
    if (VEC) {
      const float4* x4 = reinterpret_cast<const float4*>(xs);
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = threadIdx.x + k * kSegT;
        if (4 * j < len) v[k] = __ldcs(x4 + j);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (4 * (threadIdx.x + k * kSegT) < len) m = max(m, max4(v[k]));
    } else {
      for (int j = threadIdx.x; j < len; j += kSegT)
        m = max(m, absbits_for_max(xs[j]));
    }
    m = __reduce_max_sync(kFull, m);
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (warp == 0) {
      uint32_t t = lane < kSegT / 32 ? red[lane] : 0u;
      t = __reduce_max_sync(kFull, t);
      if (lane == 0 && t) atomicMax(maxima + (seg % extent), t);
    }
    __syncthreads();
  }
}

template <int M, bool VEC>
__global__ void __launch_bounds__(kSegT)
    k_seg_apply(const float* __restrict__ x, float* __restrict__ y,
                int64_t nseg, int64_t stride, int64_t extent, int64_t pieces,
                const uint32_t* __restrict__ maxima, uint64_t base,
                uint64_t key, int wl, uint32_t* __restrict__ status) {
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const int64_t items = nseg * pieces;
  uint32_t bad = 0;
  for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const int64_t seg = it / pieces, pc = it - seg * pieces;
    const int64_t off = pc * kPiece;
    const int64_t len = min((int64_t)kPiece, stride - off);
    const int64_t e0 = seg * stride + off;
    const BlockScale sc = make_block_scale(__ldg(maxima + (seg % extent)), wl);
    if (sc.bad) bad |= 2u;
    if (VEC) {
      const float4* x4 = reinterpret_cast<const float4*>(x + e0);
      float4* y4 = reinterpret_cast<float4*>(y + e0);
      float4 v[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = threadIdx.x + k * kSegT;
        if (4 * j < len) v[k] = __ldcs(x4 + j);
      }
      // the block-class loops of k_block_rows: two-factor scales, single
      // factor with / without the stochastic flush guard; float4-shared
      // variates when the flat indices are 4-aligned (base % 4 == 0)
      const bool idx4 = (base & 3u) == 0;  // uniform
      auto run = [&](auto two_t, auto guard_t, auto idx4_t) {
        constexpr bool TWO = decltype(two_t)::value;
        constexpr bool GUARD = decltype(guard_t)::value;
        constexpr bool I4 = decltype(idx4_t)::value;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int j = threadIdx.x + k * kSegT;
          if (4 * j < len) {
            bad |= nf4(v[k]);
            const uint64_t idx = base + (uint64_t)(e0 + 4 * j);
            __stcs(y4 + j, qb4<M, TWO, I4, GUARD>(v[k], sc, kmin, kmax, key, idx, rng_mul()));
          }
        }
      };
      if (two_factor(sc)) {
        if (idx4) run(std::true_type{}, std::false_type{}, std::true_type{});
        else run(std::true_type{}, std::false_type{}, std::false_type{});
      } else if (M == kStochastic && needs_guard(sc)) {
        if (idx4) run(std::false_type{}, std::true_type{}, std::true_type{});
        else run(std::false_type{}, std::true_type{}, std::false_type{});
      } else {
        if (idx4) run(std::false_type{}, std::false_type{}, std::true_type{});
        else run(std::false_type{}, std::false_type{}, std::false_type{});
      }
    } else {
      for (int j = threadIdx.x; j < len; j += kSegT) {
        const float xv = x[e0 + j];
        bad |= nonfinite(xv) ? 1u : 0u;
        y[e0 + j] = qb<M, true>(xv, sc, kmin, kmax, key ^ (base + (uint64_t)(e0 + j)), rng_mul());
      }
    }
  }
  bad = __reduce_or_sync(kFull, bad);
  if ((threadIdx.x & 31) == 0) flag(status, bad);
}

// ---------------------------------------------------------------------------
// Plan 3: short segments (stride < 1024): [outer, W = extent*stride] matrix,
// 4 columns per thread (a float4 when W % 4 == 0 and aligned), row chunks.
constexpr int kColT = 256;
constexpr int kColTile = kColT * 4;  // columns per CTA

template <bool VEC>
__device__ __forceinline__ float4 load4(const float* __restrict__ row, int64_t c,
                                        int64_t W) {
  if (VEC) return __ldcs(reinterpret_cast<const float4*>(row + c));
  float4 v;
  v.x = c < W ? row[c] : 0.0f;
  v.y = c + 1 < W ? row[c + 1] : 0.0f;
  v.z = c + 2 < W ? row[c + 2] : 0.0f;
  v.w = c + 3 < W ? row[c + 3] : 0.0f;
  return v;
}

// Column plans: a CTA covers a tile of tw = ceil(min(W, kColTile) / 4)
// float4 columns and runs kColT / tw row lanes over its row chunk, so narrow
// tensors ([outer, W] with W < 1024, e.g. per-channel blocks of NHWC data)
// keep every thread busy instead of one thread per 4 columns.
struct ColLanes {
  int tw, lanes, lane, ct;
  __device__ __forceinline__ explicit ColLanes(int64_t W) {
    tw = (int)((min(W, (int64_t)kColTile) + 3) / 4);
    lanes = kColT / tw;
    lane = threadIdx.x / tw;
    ct = threadIdx.x - lane * tw;
  }
};

template <bool VEC>
__global__ void __launch_bounds__(kColT)
    k_col_reduce(const float* __restrict__ x, int64_t outer, int64_t W,
                 int64_t stride, int64_t rows_per_chunk,
                 uint32_t* __restrict__ maxima) {
  __shared__ uint32_t smax[kColTile];  // indexed by b - b0 (<= kColTile)
  const ColLanes L(W);
  const int64_t c0 = (int64_t)blockIdx.x * kColTile;
  const int64_t c = c0 + 4 * L.ct;
  const int64_t b0 = c0 / stride;
  for (int i = threadIdx.x; i < kColTile; i += kColT) smax[i] = 0u;
  __syncthreads();
  if (c < W && L.lane < L.lanes) {
    uint32_t m0 = 0, m1 = 0, m2 = 0, m3 = 0;
    // grid.y is capped at 65535: chunks beyond it are taken grid-stride
    const int64_t rstep = (int64_t)gridDim.y * rows_per_chunk;
    for (int64_t rc = (int64_t)blockIdx.y * rows_per_chunk; rc < outer; rc += rstep)
      for (int64_t r = rc + L.lane, r1 = min(outer, rc + rows_per_chunk); r < r1;
           r += L.lanes) {
        const float4 v = load4<VEC>(x + r * W, c, W);
        m0 = max(m0, absbits_for_max(v.x));
        m1 = max(m1, absbits_for_max(v.y));
        m2 = max(m2, absbits_for_max(v.z));
        m3 = max(m3, absbits_for_max(v.w));
      }
    atomicMax(&smax[c / stride - b0], m0);
    if (c + 1 < W) atomicMax(&smax[(c + 1) / stride - b0], m1);
    if (c + 2 < W) atomicMax(&smax[(c + 2) / stride - b0], m2);
    if (c + 3 < W) atomicMax(&smax[(c + 3) / stride - b0], m3);
  }
  __syncthreads();
  const int64_t cend = min(W, c0 + kColTile);
  const int64_t nb = (cend - 1) / stride - b0 + 1;
  for (int64_t i = threadIdx.x; i < nb; i += kColT)
    if (smax[i]) atomicMax(maxima + b0 + i, smax[i]);
}

template <int M, bool VEC>
__global__ void __launch_bounds__(kColT)
    k_col_apply(const float* __restrict__ x, float* __restrict__ y,
                int64_t outer, int64_t W, int64_t stride,
                int64_t rows_per_chunk, const uint32_t* __restrict__ maxima,
                uint64_t base, uint64_t key, int wl,
                uint32_t* __restrict__ status) {
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const ColLanes L(W);
  const int64_t c = (int64_t)blockIdx.x * kColTile + 4 * L.ct;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_chunk;
  uint32_t bad = 0;
  if (c < W && L.lane < L.lanes) {
    BlockScale s[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t cq = min(c + q, W - 1);
      s[q] = make_block_scale(__ldg(maxima + cq / stride), wl);
      if (s[q].bad) bad |= 2u;
    }
    // grid.y is capped at 65535: chunks beyond it are taken grid-stride
    const int64_t rstep = (int64_t)gridDim.y * rows_per_chunk;
    for (int64_t rc = r0; rc < outer; rc += rstep)
    for (int64_t r = rc + L.lane, r1 = min(outer, rc + rows_per_chunk); r < r1;
         r += L.lanes) {
      const float4 v = load4<VEC>(x + r * W, c, W);
      const uint64_t idx = base + (uint64_t)(r * W + c);
      float4 o;
      o.x = qb<M, true>(v.x, s[0], kmin, kmax, key ^ idx, rng_mul());
      o.y = qb<M, true>(v.y, s[1], kmin, kmax, key ^ (idx + 1), rng_mul());
      o.z = qb<M, true>(v.z, s[2], kmin, kmax, key ^ (idx + 2), rng_mul());
      o.w = qb<M, true>(v.w, s[3], kmin, kmax, key ^ (idx + 3), rng_mul());
      if (VEC) {
        bad |= nf4(v);
        __stcs(reinterpret_cast<float4*>(y + r * W + c), o);
      } else {
        float* yr = y + r * W;
        bad |= nonfinite(v.x) ? 1u : 0u;
        yr[c] = o.x;
        if (c + 1 < W) { bad |= nonfinite(v.y) ? 1u : 0u; yr[c + 1] = o.y; }
        if (c + 2 < W) { bad |= nonfinite(v.z) ? 1u : 0u; yr[c + 2] = o.z; }
        if (c + 3 < W) { bad |= nonfinite(v.w) ? 1u : 0u; yr[c + 3] = o.w; }
      }
    }
  }
  bad = __reduce_or_sync(kFull, bad);
  if ((threadIdx.x & 31) == 0) flag(status, bad);
}

bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

int64_t col_rows_per_chunk(int64_t outer, int64_t W) {
  // aim at >= ~16K elements per CTA so register maxima amortise the atomics,
  // while keeping >= ~8 CTAs per SM when the tensor is large.
  const int64_t tiles = (W + kColTile - 1) / kColTile;
  const int64_t tile_w = std::min<int64_t>(W, kColTile);
  const int64_t lanes = kColT / ((tile_w + 3) / 4);
  const int64_t floor_r = lanes;  // at least one row per lane
  int64_t r = std::max<int64_t>(floor_r, 16384 / tile_w);
  const int64_t target_ctas = (int64_t)device_info().sm_count * 8;
  while (r > floor_r && tiles * ((outer + r - 1) / r) < target_ctas) r /= 2;
  return std::max<int64_t>(1, std::min(std::max(r, floor_r), outer));
}

// grid for the column plans: grid.y is capped at 65535 (the kernels take
// row chunks beyond it grid-stride)
dim3 col_grid(int64_t outer, int64_t W, int64_t rpc) {
  return dim3((unsigned)((W + kColTile - 1) / kColTile),
              (unsigned)std::min<int64_t>(65535, (outer + rpc - 1) / rpc));
}

template <int M>
cudaError_t launch_two_pass_m(const float* x, float* y, const BlockGeom& g,
                              bool segments, bool reduce, uint32_t* maxima,
                              uint64_t base, uint64_t key, int wl,
                              uint32_t* status, cudaStream_t s);

template <int M>
cudaError_t launch_block_m(const float* x, float* y, const BlockGeom& g,
                           BlockPlan plan, uint64_t base, uint64_t key, int wl,
                           void* ws, uint32_t* status, cudaStream_t s) {
  const int64_t n = g.outer * g.extent * g.stride;
  if (n <= 0) return cudaSuccess;
  if (plan == BlockPlan::kRowsInRegisters) {
    launch_rows<M>(x, y, g.stride, g.extent, base, key, wl, status, s);
    return cudaGetLastError();
  }
  if (plan == BlockPlan::kRowsChunked) {
    const cudaError_t e = launch_block_chunks(x, y, g.stride, g.extent, base, key, wl, M, ws,
                                              status, s);
    if (e != cudaErrorCooperativeLaunchTooLarge) return e;
    // fewer SMs than the occupancy query saw (MPS / green contexts): the
    // two-pass segment plan (its maxima fit the chunk plan's workspace)
    cudaGetLastError();
    plan = BlockPlan::kTwoPassSegments;
  }
  if (plan == BlockPlan::kRowsCluster)
    return launch_block_cluster(x, y, g.stride, g.extent, base, key, wl, M,
                                status, s);
  uint32_t* maxima = static_cast<uint32_t*>(ws);
  cudaError_t e = cudaMemsetAsync(maxima, 0, sizeof(uint32_t) * g.extent, s);
  if (e != cudaSuccess) return e;
  return launch_two_pass_m<M>(x, y, g, plan == BlockPlan::kTwoPassSegments, true,
                              maxima, base, key, wl, status, s);
}

// The two-pass plans; reduce == false: maxima[extent] is given (already
// reduced, e.g. across shards: lpq_quantize_block_apply) and only the
// quantize pass runs.
template <int M>
cudaError_t launch_two_pass_m(const float* x, float* y, const BlockGeom& g,
                              bool segments, bool reduce, uint32_t* maxima,
                              uint64_t base, uint64_t key, int wl,
                              uint32_t* status, cudaStream_t s) {
  const int sms = device_info().sm_count;
  if (segments) {
    const int64_t nseg = g.outer * g.extent;
    const int64_t pieces = (g.stride + kPiece - 1) / kPiece;
    const bool vec = (g.stride % 4 == 0) && aligned16(x) && aligned16(y);
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)sms * 8, nseg * pieces));
    if (vec) {
      if (reduce)
        k_seg_reduce<true><<<grid, kSegT, 0, s>>>(x, nseg, g.stride, g.extent, pieces, maxima);
      k_seg_apply<M, true><<<grid, kSegT, 0, s>>>(x, y, nseg, g.stride, g.extent, pieces,
                                                  maxima, base, key, wl, status);
    } else {
      if (reduce)
        k_seg_reduce<false><<<grid, kSegT, 0, s>>>(x, nseg, g.stride, g.extent, pieces, maxima);
      k_seg_apply<M, false><<<grid, kSegT, 0, s>>>(x, y, nseg, g.stride, g.extent, pieces,
                                                   maxima, base, key, wl, status);
    }
    note_launch(reduce ? 2 : 1);
    return cudaGetLastError();
  }
  const int64_t W = g.extent * g.stride;
  const bool vec = (W % 4 == 0) && aligned16(x) && aligned16(y);
  const int64_t rpc = col_rows_per_chunk(g.outer, W);
  const dim3 grid = col_grid(g.outer, W, rpc);
  if (vec) {
    if (reduce)
      k_col_reduce<true><<<grid, kColT, 0, s>>>(x, g.outer, W, g.stride, rpc, maxima);
    k_col_apply<M, true><<<grid, kColT, 0, s>>>(x, y, g.outer, W, g.stride, rpc, maxima,
                                                base, key, wl, status);
  } else {
    if (reduce)
      k_col_reduce<false><<<grid, kColT, 0, s>>>(x, g.outer, W, g.stride, rpc, maxima);
    k_col_apply<M, false><<<grid, kColT, 0, s>>>(x, y, g.outer, W, g.stride, rpc, maxima,
                                                 base, key, wl, status);
  }
  note_launch(reduce ? 2 : 1);
  return cudaGetLastError();
}

}  // namespace

// Per-block max|x| (as uint bits) into maxima[extent] with the two-pass
// plans' reduction kernels (used by the many-kernel baseline in composed.cu).
cudaError_t launch_block_reduce(const float* x, const BlockGeom& g,
                                uint32_t* maxima, cudaStream_t s) {
  const int64_t n = g.outer * g.extent * g.stride;
  cudaError_t e = cudaMemsetAsync(maxima, 0, sizeof(uint32_t) * g.extent, s);
  if (e != cudaSuccess || n <= 0) return e;
  if (g.stride >= 1024) {
    const int64_t nseg = g.outer * g.extent;
    const int64_t pieces = (g.stride + kPiece - 1) / kPiece;
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((int64_t)device_info().sm_count * 8, nseg * pieces));
    if ((g.stride % 4 == 0) && aligned16(x))
      k_seg_reduce<true><<<grid, kSegT, 0, s>>>(x, nseg, g.stride, g.extent, pieces, maxima);
    else
      k_seg_reduce<false><<<grid, kSegT, 0, s>>>(x, nseg, g.stride, g.extent, pieces, maxima);
  } else {
    const int64_t W = g.extent * g.stride;
    const int64_t rpc = col_rows_per_chunk(g.outer, W);
    const dim3 grid = col_grid(g.outer, W, rpc);
    if ((W % 4 == 0) && aligned16(x))
      k_col_reduce<true><<<grid, kColT, 0, s>>>(x, g.outer, W, g.stride, rpc, maxima);
    else
      k_col_reduce<false><<<grid, kColT, 0, s>>>(x, g.outer, W, g.stride, rpc, maxima);
  }
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_block_apply(const float* x, float* y, const BlockGeom& g,
                               const uint32_t* maxima, uint64_t base, uint64_t key,
                               int wl, int mode, uint32_t* status, cudaStream_t s) {
  if (g.outer * g.extent * g.stride <= 0) return cudaSuccess;
  uint32_t* mx = const_cast<uint32_t*>(maxima);  // read only when reduce == false
  const bool seg = g.stride >= 1024;
  switch (mode) {
    case kStochastic: return launch_two_pass_m<kStochastic>(x, y, g, seg, false, mx, base, key, wl, status, s);
    case kNearestAway: return launch_two_pass_m<kNearestAway>(x, y, g, seg, false, mx, base, key, wl, status, s);
    case kNearestZero: return launch_two_pass_m<kNearestZero>(x, y, g, seg, false, mx, base, key, wl, status, s);
    default: return launch_two_pass_m<kNearestEven>(x, y, g, seg, false, mx, base, key, wl, status, s);
  }
}

bool block_cluster_ok(const BlockGeom& g, const float* x, const float* y) {
  return g.outer == 1 && g.stride % 4 == 0 && aligned16(x) && aligned16(y) &&
         g.stride > 32768 && g.stride <= (int64_t(1) << 20);
}

BlockPlan block_plan(const BlockGeom& g, const float* x, const float* y) {
  const bool rows = g.outer == 1 && g.stride % 4 == 0 && aligned16(x) && aligned16(y);
  if (rows && g.stride <= 32768 && g.stride >= 4) return BlockPlan::kRowsInRegisters;
  // rows of 32K-75K floats: 2-CTA clusters ([256, 50176]: 5169 GB/s nearest
  // vs 3847 on the chunk plan, whose 7 chunks per row leave a fourth round
  // of 16 CTAs; at 100352 the two are even), when they fill the GPU
  if (block_cluster_ok(g, x, y) && g.stride <= 75000 &&
      g.extent * cluster_size_for(g.stride) >= 2 * (int64_t)device_info().sm_count)
    return BlockPlan::kRowsCluster;
  // longer rows of up to ~2.4M floats: chunk rendezvous (one HBM pass, every
  // SM busy; needs the workspace -- quantize_device takes the cluster plan
  // when the caller supplied none)
  if (rows && block_chunks_ok(g.stride, g.extent)) return BlockPlan::kRowsChunked;
  // cluster plan: rows of at most 1M floats (L2-resident second read) and
  // enough (row, CTA) pairs to fill the SMs; a few huge rows stream through
  // every SM with the two-pass segment plan instead (quantize_device still
  // takes the cluster plan when the caller supplied no workspace)
  if (block_cluster_ok(g, x, y) &&
      g.extent * cluster_size_for(g.stride) >= 2 * (int64_t)device_info().sm_count)
    return BlockPlan::kRowsCluster;
  if (g.stride >= 1024) return BlockPlan::kTwoPassSegments;
  return BlockPlan::kTwoPassColumns;
}

size_t block_workspace(const BlockGeom& g, BlockPlan p) {
  if (p == BlockPlan::kRowsChunked) return block_chunks_workspace(g.extent);
  if (block_plan_single_pass(p)) return 0;
  return (size_t)(((g.extent * 4) + 255) / 256 * 256);
}

cudaError_t launch_block(const float* x, float* y, const BlockGeom& g,
                         BlockPlan plan, uint64_t base, uint64_t key, int wl,
                         int mode, void* ws, uint32_t* status, cudaStream_t s) {
  switch (mode) {
    case kStochastic: return launch_block_m<kStochastic>(x, y, g, plan, base, key, wl, ws, status, s);
    case kNearestAway: return launch_block_m<kNearestAway>(x, y, g, plan, base, key, wl, ws, status, s);
    case kNearestZero: return launch_block_m<kNearestZero>(x, y, g, plan, base, key, wl, ws, status, s);
    default: return launch_block_m<kNearestEven>(x, y, g, plan, base, key, wl, ws, status, s);
  }
}

}  // namespace lpq
