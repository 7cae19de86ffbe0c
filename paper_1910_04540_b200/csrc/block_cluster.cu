// block_cluster.cu -- single-HBM-pass block floating point for long
// contiguous blocks (> 32K floats, e.g. the per-sample activation blocks of
// ResNet-50 at batch 256, up to 802,816 floats = 3.2 MB).
//
// A row (one block) is spread over a thread-block CLUSTER of up to 16 CTAs.
// Each CTA reduces max|x| over its slice, publishes it in its shared memory,
// and after a cluster barrier reads the other CTAs' maxima through
// distributed shared memory (mapa + ld.shared::cluster) -- no global atomics,
// no second kernel.  It then re-reads its slice, which the residency cap keeps
// in the 126 MB L2, and streams the quantized values out: one HBM read and one
// HBM write per element (8 algorithmic bytes instead of the two-pass plan's
// 12).  (A first version staged the slice in shared memory with TMA bulk
// copies; one 196 KB CTA per SM could not overlap loading with storing and
// reached only 4.3 TB/s -- see DESIGN.md.)
// Semantics: fused_block (proj/src/quant_ops.cpp:68-115) with block_dim such
// that blocks are contiguous rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>

#include "block_common.cuh"
#include "kernels.cuh"

namespace lpq {

namespace {

using namespace blk;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// read a u32 from the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t ld_dsmem(const uint32_t* local, uint32_t rank) {
  uint32_t remote, v;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(remote) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(remote) : "memory");
  return v;
}


// One cluster per row; CTA `rank` owns float4s [rank*S4, min(L4,(rank+1)*S4)).
// Pass 1 streams the slice from HBM (normal L2 policy: it stays in L2),
// reduces max|x| and publishes it in shared memory; after a cluster barrier
// every CTA gathers the CS slice maxima over DSMEM; pass 2 re-reads the slice
// (L2 hits, evict-first) and streams the quantized values out (evict-first).
// HBM traffic: one read + one write per element (8 algorithmic bytes).  The
// dynamic shared-memory request only caps residency at kCtasPerSm CTAs/SM so
// the rows in flight fit in the 126 MB L2.
template <int M, bool IDX4, int kCT, int kU>
__global__ void __launch_bounds__(kCT)
    k_block_rows_cluster(const float* __restrict__ x, float* __restrict__ y,
                         int64_t L, int64_t S4, uint64_t base, uint64_t key,
                         int wl, RngMul rm, uint32_t* __restrict__ status) {
  __shared__ uint32_t red[kCT / 32];
  __shared__ uint32_t cta_max;
  const uint32_t rank = cluster_rank();
  uint32_t cs;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs));
  const int64_t row = blockIdx.x / cs;
  const int64_t L4 = L >> 2;
  const int64_t s0 = (int64_t)rank * S4;
  const int64_t rem4 = L4 - s0;
  const int64_t len4 = rem4 <= 0 ? 0 : (rem4 < S4 ? rem4 : S4);
  const float4* __restrict__ xr = reinterpret_cast<const float4*>(x + row * L) + s0;
  float4* __restrict__ yr = reinterpret_cast<float4*>(y + row * L) + s0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  // pass 1: max|x| (NaN ignored) and the non-finite probe
  float mf = 0.0f, nf = 0.0f;
  for (int64_t j0 = threadIdx.x; j0 < len4; j0 += (int64_t)kCT * kU) {
    float4 v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t j = j0 + (int64_t)u * kCT;
      if (j < len4) v[u] = __ldg(xr + j);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (j0 + (int64_t)u * kCT < len4) absmax_nf(v[u], mf, nf);
  }
  uint32_t m = __reduce_max_sync(kFull, f2u(mf));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < kCT / 32 ? red[lane] : 0u;
    t = __reduce_max_sync(kFull, t);
    if (lane == 0) cta_max = t;
  }
  // publish this CTA's maximum to the cluster, then gather all of them
  cluster_arrive();
  cluster_wait();
  uint32_t row_max = 0;
  for (uint32_t r = 0; r < cs; ++r) row_max = max(row_max, ld_dsmem(&cta_max, r));
  // nobody may exit (and free its shared memory) before every peer has read
  // its maximum: arrive now, wait at the very end
  cluster_arrive();

  // pass 2: quantize (the slice is L2-resident from pass 1)
  const BlockScale sc = make_block_scale(row_max, wl);
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const uint64_t ebase = base + (uint64_t)(row * L + s0 * 4);
  // block-class loops (see k_block_rows in block.cu)
  auto run = [&](auto two_t, auto guard_t) {
    constexpr bool TWO = decltype(two_t)::value;
    constexpr bool GUARD = decltype(guard_t)::value;
    for (int64_t j0 = threadIdx.x; j0 < len4; j0 += (int64_t)kCT * kU) {
      float4 v[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t j = j0 + (int64_t)u * kCT;
        if (j < len4) v[u] = __ldcs(xr + j);
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t j = j0 + (int64_t)u * kCT;
        if (j < len4)
          __stcs(yr + j, qb4<M, TWO, IDX4, GUARD>(v[u], sc, kmin, kmax, key,
                                                  ebase + 4 * j, rm));
      }
    }
  };
  if (two_factor(sc)) run(std::true_type{}, std::false_type{});
  else if (M == kStochastic && needs_guard(sc)) run(std::false_type{}, std::true_type{});
  else run(std::false_type{}, std::false_type{});
  uint32_t bad = (sc.bad ? 2u : 0u) | (nf != nf ? 1u : 0u);
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0 && bad) atomicOr(status, bad);
  cluster_wait();
}

template <int M, bool IDX4, int kCT, int kU>
cudaError_t launch_cluster_v(const float* x, float* y, int64_t L, int64_t nrows,
                             int cs, uint64_t base, uint64_t key, int wl,
                             uint32_t* st, cudaStream_t s, int kCtasPerSm) {
  const int64_t L4 = L >> 2;
  const int64_t S4 = (L4 + cs - 1) / cs;
  auto kern = k_block_rows_cluster<M, IDX4, kCT, kU>;
  // residency cap: request a share of shared memory so that at most
  // kCtasPerSm CTAs are resident per SM
  const int smem = kCtasPerSm > 0 ? device_info().max_smem_optin / kCtasPerSm - 2048 : 0;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nrows * cs), 1, 1);
  cfg.blockDim = dim3(kCT, 1, 1);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  e = cudaLaunchKernelEx(&cfg, kern, x, y, L, S4, base, key, wl, rng_mul(), st);
  note_launch();
  return e;
}

// 512 threads x 8 float4 in flight, residency left to the hardware
// (measured on B200 against 256/4, 256/8, 256/16, 512/8 with 2-4 CTA/SM caps
// and slices of 16K-1M floats: this is the fastest, ~4.45 TB/s on the
// ResNet-50 activation shapes)
template <int M, bool IDX4>
cudaError_t launch_cluster_t(const float* x, float* y, int64_t L, int64_t nrows,
                             int cs, uint64_t base, uint64_t key, int wl,
                             uint32_t* st, cudaStream_t s) {
  return launch_cluster_v<M, IDX4, 512, 8>(x, y, L, nrows, cs, base, key, wl, st, s, 0);
}

template <int M>
cudaError_t launch_cluster_m(const float* x, float* y, int64_t L, int64_t nrows,
                             int cs, uint64_t base, uint64_t key, int wl,
                             uint32_t* st, cudaStream_t s) {
  if ((base & 3u) == 0)
    return launch_cluster_t<M, true>(x, y, L, nrows, cs, base, key, wl, st, s);
  return launch_cluster_t<M, false>(x, y, L, nrows, cs, base, key, wl, st, s);
}

}  // namespace

// Cluster size for a contiguous block of L floats.  Measured on B200
// (scripts/time_act_shapes.py, ResNet-50 per-sample activation rows, every
// cs from 1 to 16): the best sizes are 2 CTAs up to ~100K floats (50176:
// 4215 GB/s vs 2884 with one CTA), 4 up to ~200K, 8 up to 1M (802816: 4901
// vs 4048 with 13).  Cluster sizes that tile a GPC's CTA slots well (2, 4,
// 8: cudaOccupancyMaxActiveClusters, scripts/cluster_probe.cu) beat the
// "one ~64K-float slice per CTA" rule; longer rows take 128K-float slices.
int cluster_size_for(int64_t L) {
  if (L <= 110000) return 2;
  if (L <= 220000) return 4;
  if (L <= (int64_t(1) << 20)) return 8;
  const int64_t cs = (L + 131071) / 131072;
  return (int)std::min<int64_t>(16, cs);
}

cudaError_t launch_block_cluster(const float* x, float* y, int64_t L,
                                 int64_t nrows, uint64_t base, uint64_t key,
                                 int wl, int mode, uint32_t* status,
                                 cudaStream_t s) {
  const int cs = cluster_size_for(L);
  if (cs == 0 || nrows <= 0) return cudaErrorInvalidValue;
  switch (mode) {
    case kStochastic: return launch_cluster_m<kStochastic>(x, y, L, nrows, cs, base, key, wl, status, s);
    case kNearestAway: return launch_cluster_m<kNearestAway>(x, y, L, nrows, cs, base, key, wl, status, s);
    case kNearestZero: return launch_cluster_m<kNearestZero>(x, y, L, nrows, cs, base, key, wl, status, s);
    default: return launch_cluster_m<kNearestEven>(x, y, L, nrows, cs, base, key, wl, status, s);
  }
}

}  // namespace lpq
