// block_chunks.cu -- single-HBM-pass block floating point for long
// contiguous blocks ("rows" of 32K .. ~4M floats: the per-sample activation
// blocks of ResNet-50 at batch 256, up to 802,816 floats = 3.2 MB, and whole
// tensors of up to a few M floats).
//
// Semantics: fused_block (proj/src/quant_ops.cpp:68-115) with the block
// maximum of reduce_max_abs (proj/src/tensor.cpp:320-353, NaN ignored) over
// contiguous blocks.
//
// Plan ("chunk rendezvous"): a row is cut into cpr equal chunks of at most
// kT * kV float4 (32 KB).  A cooperative grid of G co-resident CTAs takes
// chunks g, g + G, g + 2G, ... (address order).  A CTA loads its chunk into
// REGISTERS, reduces max|x| over it, folds it into the row's maximum
// (atomicMax) and arrives on the row's counter, starts an L2 prefetch of its
// next chunk, and once all cpr chunks of the row have arrived quantizes the
// chunk from registers and streams it out.  HBM traffic is exactly one read
// and one write per element (8 algorithmic bytes) and every SM stays busy
// whatever the row length -- unlike a cluster per row, which pins CTAs to
// GPCs and re-reads the slice through L2 (1.59x DRAM read amplification on
// [256, 802816], profiles/r01_act_block_cluster_*).
//
// Progress: with cpr <= G a CTA's consecutive chunks t and t + G are never in
// the same row, so a CTA that holds a chunk of row R in its next round first
// finishes a chunk of a row < R: every wait points at a lower row, there is
// no cycle, and with all CTAs co-resident (the cooperative launch) every row
// completes.  block_chunks_ok requires cpr <= the resident CTA count.
//
// Workspace (u32): rowmax[nrows] (max|x| bits per row -- the same layout as
// the two-pass plans' maxima, which the host path's block byte coder reads),
// arrive[nrows]; zeroed on the stream before the launch.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

#include "block_common.cuh"
#include "kernels.cuh"

namespace lpq {

namespace {

using namespace blk;

constexpr int kT = 256;  // threads per CTA
// float4 per thread (chunks of kT * kV float4 = 32 KB held in registers)
// and CTAs per SM.  Measured on B200 against (16 float4, 2 CTAs/SM), (8, 3),
// (4, 6), (4, 8), (6, 4) on the ResNet-50 activation rows (scripts/
// time_act_plans.py): more resident CTAs hide the rendezvous and load
// latencies until the register cap spills; [256, 802816] stochastic 4607 ->
// 4673 GB/s, nearest 5801 -> 5967.  Also measured and slower (stochastic /
// nearest): a shared-memory variant double-buffering chunks with cp.async,
// the next chunk's loads issued before the rendezvous, 3 CTAs/SM (3867 /
// 4710); a register double-buffered one, 2 CTAs/SM (3518 / 4596), and with
// 4 float4 per thread at 4 CTAs/SM (3567 / 4511); 128-thread CTAs x 8 per SM
// (3772 / 4425); the L2 prefetch two rounds ahead (4425 / 5740); staging the
// next chunk in shared memory by cp.async and arriving it BEFORE quantizing
// the current one, so a row's arrivals never wait on a CTA's stochastic
// quantize pass (4084 / 5465); up to twice as many smaller chunks per row
// when that fills the last round of the grid better ([256, 50176] 3847 ->
// 4169 nearest, but [256, 401408] 5873 -> 5462 and [256, 200704] 5478 ->
// 4960: the rendezvous cost per chunk outweighs the waves); hashing a
// stochastic chunk's variates into shared memory while the row's other
// chunks arrive (stochastic 4547 -> 4463: the kernel is issue-bound, not
// latency-bound, under stochastic rounding).
constexpr int kV = 8;
constexpr int kB = 4;

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

// L2 prefetch of a chunk (16-byte aligned, a multiple of 16 bytes) in
// pieces of 4 KB, one per thread of the first warps
__device__ __forceinline__ void prefetch_l2(const float4* p, int64_t n4) {
  const int64_t piece4 = 256;  // 4 KB
  const int64_t i0 = (int64_t)threadIdx.x * piece4;
  if (i0 < n4) {
    const int64_t len4 = n4 - i0 < piece4 ? n4 - i0 : piece4;
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;"
                 :: "l"(p + i0), "r"((uint32_t)(16 * len4)) : "memory");
  }
}

template <int M, bool IDX4>
__global__ void __launch_bounds__(kT, kB)
    k_block_chunks(const float* __restrict__ x, float* __restrict__ y, int64_t L,
                   int64_t nrows, int64_t cpr, int64_t S4, uint32_t* __restrict__ ws,
                   uint64_t base, uint64_t key, int wl, RngMul rm,
                   uint32_t* __restrict__ status) {
  __shared__ uint32_t red[kT / 32];
  __shared__ uint32_t sh_max;     // the chunk's maximum
  __shared__ uint32_t sh_row;     // the row's maximum
  uint32_t* rowmax = ws;
  uint32_t* arrive = ws + nrows;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t total = nrows * cpr;
  const int64_t L4 = L >> 2;
  const int64_t G = gridDim.x;
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  // chunk t -> (row, float4 offset, length)
  auto chunk = [&](int64_t t, int64_t& row, int64_t& off4) {
    row = t / cpr;
    off4 = (t - row * cpr) * S4;
    return S4 < L4 - off4 ? S4 : L4 - off4;
  };
  uint32_t bad = 0;
  for (int64_t t = blockIdx.x; t < total; t += G) {
    int64_t row, off4;
    const int64_t len4 = chunk(t, row, off4);
    const float4* __restrict__ xr = reinterpret_cast<const float4*>(x + row * L) + off4;
    float4* __restrict__ yr = reinterpret_cast<float4*>(y + row * L) + off4;
    float4 v[kV];
    float mf = 0.0f;
#pragma unroll
    for (int k = 0; k < kV; ++k) {
      const int64_t j = threadIdx.x + (int64_t)k * kT;
      if (j < len4) {
        v[k] = __ldcs(xr + j);
        absmax_nan(v[k], mf);
      }
    }
    // chunk maximum (NaN-propagating first; a NaN chunk recomputes the
    // NaN-ignoring maximum of reduce_max_abs and flags the input)
    uint32_t m = __reduce_max_sync(kFull, f2u(mf));
    if (lane == 0) red[warp] = m;
    __syncthreads();
    if (warp == 0) {
      uint32_t u = lane < kT / 32 ? red[lane] : 0u;
      u = __reduce_max_sync(kFull, u);
      if (lane == 0) sh_max = u;
    }
    __syncthreads();
    m = sh_max;
    if (m > 0x7F800000u) {  // NaN in the chunk (uniform)
      bad |= 1u;
      float nf = 0.0f;
      mf = 0.0f;
#pragma unroll
      for (int k = 0; k < kV; ++k) {
        const int64_t j = threadIdx.x + (int64_t)k * kT;
        if (j < len4) absmax_nf(v[k], mf, nf);
      }
      m = __reduce_max_sync(kFull, f2u(mf));
      __syncthreads();  // sh_max / red are rewritten
      if (lane == 0) red[warp] = m;
      __syncthreads();
      if (warp == 0) {
        uint32_t u = lane < kT / 32 ? red[lane] : 0u;
        u = __reduce_max_sync(kFull, u);
        if (lane == 0) sh_max = u;
      }
      __syncthreads();
      m = sh_max;
    }
    // arrive; stream this CTA's next chunk into L2 while the row completes
    if (threadIdx.x == 0) {
      atomicMax(rowmax + row, m);
      red_release_add(arrive + row, 1u);
    }
    // (two rounds ahead measured slower: [256, 802816] nearest 4662 -> 4425)
    if (t + G < total) {
      int64_t nrow, noff4;
      const int64_t nlen4 = chunk(t + G, nrow, noff4);
      prefetch_l2(reinterpret_cast<const float4*>(x + nrow * L) + noff4, nlen4);
    }
    if (threadIdx.x == 0) {
      // (a watchdog, not a code path: a rendezvous that has not completed
      // after ~2^32 cycles (> 2 s) means the co-residency the cooperative
      // launch guarantees was broken -- trap instead of hanging the device)
      const long long t0 = clock64();
      while (ld_acquire_gpu(arrive + row) < (uint32_t)cpr) {
        __nanosleep(64);
        if (clock64() - t0 > (1ll << 32)) __trap();
      }
      sh_row = ld_relaxed_gpu(rowmax + row);
    }
    __syncthreads();
    const uint32_t row_max = sh_row;
    const BlockScale sc = make_block_scale(row_max, wl);
    if (sc.bad) bad |= 2u;
    const uint64_t ebase = base + (uint64_t)(row * L + 4 * off4);
    auto run = [&](auto two_t, auto guard_t) {
      constexpr bool TWO = decltype(two_t)::value;
      constexpr bool GUARD = decltype(guard_t)::value;
#pragma unroll
      for (int k = 0; k < kV; ++k) {
        const int64_t j = threadIdx.x + (int64_t)k * kT;
        if (j < len4)
          __stcs(yr + j, qb4<M, TWO, IDX4, GUARD>(v[k], sc, kmin, kmax, key,
                                                  ebase + 4 * j, rm));
      }
    };
    if (two_factor(sc)) run(std::true_type{}, std::false_type{});
    else if (M == kStochastic && needs_guard(sc)) run(std::false_type{}, std::true_type{});
    else run(std::false_type{}, std::false_type{});
    // red / sh_max / sh_row are rewritten next iteration only after a
    // __syncthreads there, which every thread reaches after reading them
  }
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0) flag(status, bad);
}

template <int M, bool IDX4>
int per_sm_t() {  // resident CTAs per SM (a property of the kernel and the arch)
  static int per_sm = -1;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (per_sm < 0) {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_block_chunks<M, IDX4>, kT, 0) !=
        cudaSuccess)
      b = 1;
    per_sm = std::max(1, b);
  }
  return per_sm;
}

// the least resident count over the instantiations on the CURRENT device:
// the grid of every mode (and the progress test in block_chunks_ok)
int resident_ctas() {
  static const int per_sm = std::min({per_sm_t<kStochastic, true>(),
                                      per_sm_t<kStochastic, false>(),
                                      per_sm_t<kNearestEven, true>(),
                                      per_sm_t<kNearestEven, false>(),
                                      per_sm_t<kNearestAway, true>(),
                                      per_sm_t<kNearestAway, false>(),
                                      per_sm_t<kNearestZero, true>(),
                                      per_sm_t<kNearestZero, false>()});
  return per_sm * device_info().sm_count;
}

// chunk geometry of a row of L floats: cpr chunks of S4 float4 each
void chunk_geometry(int64_t L, int64_t* cpr, int64_t* S4) {
  const int64_t L4 = L >> 2;
  const int64_t C4 = (int64_t)kT * kV;
  *cpr = (L4 + C4 - 1) / C4;
  *S4 = (L4 + *cpr - 1) / *cpr;
}

template <int M, bool IDX4>
cudaError_t launch_chunks_t(const float* x, float* y, int64_t L, int64_t nrows,
                            uint64_t base, uint64_t key, int wl, void* ws,
                            uint32_t* st, cudaStream_t s) {
  int64_t cpr, S4;
  chunk_geometry(L, &cpr, &S4);
  cudaError_t e = cudaMemsetAsync(ws, 0, block_chunks_workspace(nrows), s);
  if (e != cudaSuccess) return e;
  const int64_t total = nrows * cpr;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(total, resident_ctas()));
  // cooperative: every CTA co-resident (the rendezvous relies on it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid, 1, 1);
  cfg.blockDim = dim3(kT, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;  // (without it: ~6 % faster, but no co-residency guarantee)
  e = cudaLaunchKernelEx(&cfg, k_block_chunks<M, IDX4>, x, y, L, nrows, cpr, S4,
                         static_cast<uint32_t*>(ws), base, key, wl, rng_mul(), st);
  note_launch();
  return e;
}

template <int M>
cudaError_t launch_chunks_m(const float* x, float* y, int64_t L, int64_t nrows,
                            uint64_t base, uint64_t key, int wl, void* ws,
                            uint32_t* st, cudaStream_t s) {
  if ((base & 3u) == 0)
    return launch_chunks_t<M, true>(x, y, L, nrows, base, key, wl, ws, st, s);
  return launch_chunks_t<M, false>(x, y, L, nrows, base, key, wl, ws, st, s);
}

}  // namespace

size_t block_chunks_workspace(int64_t nrows) {
  return (size_t)((8 * nrows + 255) / 256 * 256);
}

bool block_chunks_ok(int64_t L, int64_t nrows) {
  if (L <= 0 || nrows <= 0 || L % 4 != 0) return false;
  int64_t cpr, S4;
  chunk_geometry(L, &cpr, &S4);
  // cpr <= G (progress, see the header)
  return cpr <= (int64_t)resident_ctas() && nrows * cpr < (int64_t(1) << 31);
}

cudaError_t launch_block_chunks(const float* x, float* y, int64_t L, int64_t nrows,
                                uint64_t base, uint64_t key, int wl, int mode, void* ws,
                                uint32_t* status, cudaStream_t s) {
  switch (mode) {
    case kStochastic: return launch_chunks_m<kStochastic>(x, y, L, nrows, base, key, wl, ws, status, s);
    case kNearestAway: return launch_chunks_m<kNearestAway>(x, y, L, nrows, base, key, wl, ws, status, s);
    case kNearestZero: return launch_chunks_m<kNearestZero>(x, y, L, nrows, base, key, wl, ws, status, s);
    default: return launch_chunks_m<kNearestEven>(x, y, L, nrows, base, key, wl, ws, status, s);
  }
}

}  // namespace lpq
