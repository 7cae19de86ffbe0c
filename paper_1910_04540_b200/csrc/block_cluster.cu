// block_cluster.cu -- single-pass block floating point for long contiguous
// blocks (32K < block <= ~900K floats, e.g. the per-sample activation blocks
// of ResNet-50 at batch 256, up to 802,816 floats = 3.2 MB).
//
// A row (one block) is spread over a thread-block CLUSTER of CS CTAs (up to
// 16, one per SM).  Each CTA streams its slice HBM -> shared memory with TMA
// bulk copies (cp.async.bulk ... mbarrier::complete_tx, in chunks so the
// max-reduction starts while later chunks are in flight), reduces the slice's
// max|x|, publishes it in its shared memory, and after a cluster barrier
// reads the other CTAs' maxima through distributed shared memory
// (mapa + ld.shared::cluster).  It then quantizes its slice from shared
// memory and streams it out.  HBM sees every element exactly once each way:
// 8 algorithmic bytes per element instead of the two-pass plan's 12.
// Semantics: fused_block (proj/src/quant_ops.cpp:68-115) with block_dim such
// that blocks are contiguous rows.
#include <cuda_runtime.h>

#include <algorithm>

#include "block_common.cuh"
#include "kernels.cuh"

namespace lpq {

namespace {

using namespace blk;

constexpr int kCT = 512;            // threads per CTA
constexpr int kChunkBytes = 32768;  // TMA bulk chunk (one mbarrier each)
constexpr int kMaxChunks = 8;       // <= 256 KB per CTA

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

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n LPQ_CL_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LPQ_CL_WAIT;\n}\n" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1], %2, [%3];"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// One cluster per row; CTA `rank` owns float4s [rank*S4, min(L4,(rank+1)*S4)).
template <int M, bool IDX4>
__global__ void __launch_bounds__(kCT, 1)
    k_block_rows_cluster(const float* __restrict__ x, float* __restrict__ y,
                         int64_t L, int64_t S4, uint64_t base, uint64_t key,
                         int wl, RngMul rm, uint32_t* __restrict__ status) {
  extern __shared__ __align__(128) float4 slice[];
  __shared__ __align__(8) uint64_t bars[kMaxChunks];
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
  const int64_t bytes = len4 * 16;
  const int nchunks = (int)((bytes + kChunkBytes - 1) / kChunkBytes);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  if (threadIdx.x == 0) {
    for (int c = 0; c < nchunks; ++c) mbar_init(&bars[c], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int c = 0; c < nchunks; ++c) {
      const int64_t off = (int64_t)c * kChunkBytes;
      const uint32_t nb = (uint32_t)(bytes - off < kChunkBytes ? bytes - off : kChunkBytes);
      mbar_expect_tx(&bars[c], nb);
      bulk_load(reinterpret_cast<char*>(slice) + off,
                reinterpret_cast<const char*>(xr) + off, nb, &bars[c]);
    }
  }
  __syncthreads();

  // pass over shared memory: max|x| (NaN ignored) and the non-finite probe
  float mf = 0.0f, nf = 0.0f;
  constexpr int kChunk4 = kChunkBytes / 16;
  for (int c = 0; c < nchunks; ++c) {
    mbar_wait(&bars[c], 0);
    const int64_t ce = (int64_t)(c + 1) * kChunk4;
    const int64_t e = len4 < ce ? len4 : ce;
    for (int64_t j = (int64_t)c * kChunk4 + threadIdx.x; j < e; j += kCT)
      absmax_nf(slice[j], mf, nf);
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

  const BlockScale sc = make_block_scale(row_max, wl);
  const float kmin = -(float)(1 << (wl - 1));
  const float kmax = (float)((1 << (wl - 1)) - 1);
  const uint64_t ebase = base + (uint64_t)(row * L + s0 * 4);
  if (!two_factor(sc)) {
    for (int64_t j = threadIdx.x; j < len4; j += kCT)
      __stcs(yr + j, qb4<M, false, IDX4>(slice[j], sc, kmin, kmax, key, ebase + 4 * j, rm));
  } else {
    for (int64_t j = threadIdx.x; j < len4; j += kCT)
      __stcs(yr + j, qb4<M, true, IDX4>(slice[j], sc, kmin, kmax, key, ebase + 4 * j, rm));
  }
  uint32_t bad = (sc.bad ? 2u : 0u) | (nf != nf ? 1u : 0u);
  bad = __reduce_or_sync(kFull, bad);
  if (lane == 0 && bad) atomicOr(status, bad);
  cluster_wait();
}

template <int M, bool IDX4>
cudaError_t launch_cluster_t(const float* x, float* y, int64_t L, int64_t nrows,
                             int cs, uint64_t base, uint64_t key, int wl,
                             uint32_t* st, cudaStream_t s) {
  const int64_t L4 = L >> 2;
  const int64_t S4 = (L4 + cs - 1) / cs;
  const size_t smem = (size_t)S4 * 16;
  auto kern = k_block_rows_cluster<M, IDX4>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nrows * cs), 1, 1);
  cfg.blockDim = dim3(kCT, 1, 1);
  cfg.dynamicSmemBytes = smem;
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

template <int M>
cudaError_t launch_cluster_m(const float* x, float* y, int64_t L, int64_t nrows,
                             int cs, uint64_t base, uint64_t key, int wl,
                             uint32_t* st, cudaStream_t s) {
  if ((base & 3u) == 0)
    return launch_cluster_t<M, true>(x, y, L, nrows, cs, base, key, wl, st, s);
  return launch_cluster_t<M, false>(x, y, L, nrows, cs, base, key, wl, st, s);
}

}  // namespace

// Cluster size for a contiguous block of L floats, or 0 if the cluster plan
// does not apply (slices of at most kMaxChunks * kChunkBytes per CTA, at most
// 16 CTAs).
int cluster_size_for(int64_t L) {
  const int64_t max_slice = (int64_t)kMaxChunks * kChunkBytes / 4;  // floats
  const int64_t cap = std::min<int64_t>(max_slice,
                                        (int64_t)(device_info().max_smem_optin - 4096) / 16 * 4);
  for (int cs = 1; cs <= 16; ++cs)
    if ((L + cs - 1) / cs <= cap) return cs;
  return 0;
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
