// ew_variants.cu -- exploration benchmark (not part of the product): variants
// of the C2 streaming kernel (fixed(8,4), saturating, stochastic) on 2^30
// elements, each timed with CUDA events and checked bit-for-bit against V0.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -std=c++17 \
//        -I paper_1910_04540_b200/csrc scripts/ew_variants.cu -o build/ew_variants
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "quant_math.cuh"

using namespace lpq;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  std::printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); std::exit(1);} } while (0)

struct Op {
  FixedParams p;
  __device__ __forceinline__ float operator()(float x, uint64_t z, uint32_t m32,
                                              float& nf) const {
    const uint32_t v = variate24_zb(z, m32);
    nf = __fmaf_rn(x, 0.0f, nf);
    return quant_fixed_sat_fast<kStochastic>(x, p, v);
  }
};

__device__ __forceinline__ float4 q4(const Op& op, float4 v, uint64_t z0, uint32_t m32,
                                     float& nf) {
  float4 o;
  o.x = op(v.x, z0, m32, nf);
  o.y = op(v.y, z0 ^ 1u, m32, nf);
  o.z = op(v.z, z0 ^ 2u, m32, nf);
  o.w = op(v.w, z0 ^ 3u, m32, nf);
  return o;
}

// V0: production shape (U float4 per thread per trip, loads then compute)
template <int U>
__global__ void __launch_bounds__(256) v0(const float4* __restrict__ x, float4* __restrict__ y,
                                          int64_t n4, uint64_t key, Op op, uint32_t m32,
                                          uint32_t* st) {
  float nf = 0.f;
  const int64_t step = (int64_t)gridDim.x * 256 * U;
  for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n4; i0 += step) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i0 + (int64_t)u * 256; if (j < n4) v[u] = __ldcs(x + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t j = i0 + (int64_t)u * 256;
      if (j < n4) __stcs(y + j, q4(op, v[u], key ^ (uint64_t)(4 * j), m32, nf));
    }
  }
  if (nf != nf) atomicOr(st, 1u);
}

// V1: register double buffering -- next trip's loads issued before compute
template <int U>
__global__ void __launch_bounds__(256) v1(const float4* __restrict__ x, float4* __restrict__ y,
                                          int64_t n4, uint64_t key, Op op, uint32_t m32,
                                          uint32_t* st) {
  float nf = 0.f;
  const int64_t step = (int64_t)gridDim.x * 256 * U;
  int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x;
  float4 v[U], w[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { int64_t j = i0 + (int64_t)u * 256; if (j < n4) v[u] = __ldcs(x + j); }
  for (; i0 < n4; i0 += step) {
    const int64_t i1 = i0 + step;
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i1 + (int64_t)u * 256; if (j < n4) w[u] = __ldcs(x + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int64_t j = i0 + (int64_t)u * 256;
      if (j < n4) __stcs(y + j, q4(op, v[u], key ^ (uint64_t)(4 * j), m32, nf));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = w[u];
  }
  if (nf != nf) atomicOr(st, 1u);
}

// V3: TMA bulk loads (cp.async.bulk global->shared, mbarrier complete_tx),
// S stages of TILE floats per CTA, persistent CTAs, STG stores.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
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
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}\n" :: "r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int S, int TILE>
__global__ void __launch_bounds__(256) v3(const float* __restrict__ x, float* __restrict__ y,
                                          int64_t n, uint64_t key, Op op, uint32_t m32,
                                          uint32_t* st) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t full[S];
  const int64_t ntiles = n / TILE;  // n multiple of TILE here
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t t = blockIdx.x;
  // prologue: fill S stages
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      const int64_t tt = t + (int64_t)s * gridDim.x;
      if (tt < ntiles) {
        mbar_expect_tx(&full[s], TILE * 4);
        bulk_load(sm + s * TILE, x + tt * TILE, TILE * 4, &full[s]);
      }
    }
  }
  float nf = 0.f;
  uint32_t phase = 0;
  int s = 0;
  for (; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], phase);
    const float4* src = reinterpret_cast<const float4*>(sm + s * TILE);
    float4* dst = reinterpret_cast<float4*>(y + t * TILE);
#pragma unroll 4
    for (int j = threadIdx.x; j < TILE / 4; j += 256)
      __stcs(dst + j, q4(op, src[j], key ^ (uint64_t)(t * TILE + 4 * j), m32, nf));
    __syncthreads();  // stage s fully consumed
    if (threadIdx.x == 0) {
      const int64_t tt = t + (int64_t)S * gridDim.x;
      if (tt < ntiles) {
        mbar_expect_tx(&full[s], TILE * 4);
        bulk_load(sm + s * TILE, x + tt * TILE, TILE * 4, &full[s]);
      }
    }
    if (++s == S) { s = 0; phase ^= 1u; }
  }
  if (nf != nf) atomicOr(st, 1u);
}


__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" :: "n"(N) : "memory");
}

// V4: TMA bulk load -> compute in place in smem -> TMA bulk store.
template <int S, int TILE, int T>
__global__ void __launch_bounds__(T) v4(const float* __restrict__ x, float* __restrict__ y,
                                        int64_t n, uint64_t key, Op op, uint32_t m32,
                                        uint32_t* st) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t full[S];
  const int64_t ntiles = n / TILE;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t t0 = blockIdx.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S - 1; ++s) {  // S-1 loads in flight, one stage drains its store
      const int64_t tt = t0 + (int64_t)s * gridDim.x;
      if (tt < ntiles) {
        mbar_expect_tx(&full[s], TILE * 4);
        bulk_load(sm + s * TILE, x + tt * TILE, TILE * 4, &full[s]);
      }
    }
  }
  float nf = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t t = t0, it = 0; t < ntiles; t += gridDim.x, ++it) {
    mbar_wait(&full[s], ph);
    float4* buf = reinterpret_cast<float4*>(sm + s * TILE);
#pragma unroll 4
    for (int j = threadIdx.x; j < TILE / 4; j += T)
      buf[j] = q4(op, buf[j], key ^ (uint64_t)(t * TILE + 4 * j), m32, nf);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_store(y + t * TILE, sm + s * TILE, TILE * 4);
      bulk_commit();
      // refill the stage whose store was issued S-1 tiles ago
      const int sr = (s + S - 1) % S;
      const int64_t tt = t + (int64_t)(S - 1) * gridDim.x;
      bulk_wait_read<S - 2>();
      if (tt < ntiles) {
        mbar_expect_tx(&full[sr], TILE * 4);
        bulk_load(sm + sr * TILE, x + tt * TILE, TILE * 4, &full[sr]);
      }
    }
    if (++s == S) { s = 0; ph ^= 1u; }
  }
  if (threadIdx.x == 0) bulk_wait<0>();
  if (nf != nf) atomicOr(st, 1u);
}

// TMA bulk copy (roofline probe)
template <int S, int TILE>
__global__ void __launch_bounds__(32) tcopy(const float* __restrict__ x, float* __restrict__ y, int64_t n) {
  extern __shared__ __align__(128) float sm[];
  __shared__ __align__(8) uint64_t full[S];
  const int64_t ntiles = n / TILE;
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int s = 0; s < S - 1; ++s) {
    const int64_t tt = blockIdx.x + (int64_t)s * gridDim.x;
    if (tt < ntiles) { mbar_expect_tx(&full[s], TILE * 4); bulk_load(sm + s * TILE, x + tt * TILE, TILE * 4, &full[s]); }
  }
  int s = 0; uint32_t ph = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[s], ph);
    bulk_store(y + t * TILE, sm + s * TILE, TILE * 4);
    bulk_commit();
    const int sr = (s + S - 1) % S;
    const int64_t tt = t + (int64_t)(S - 1) * gridDim.x;
    bulk_wait_read<S - 2>();
    if (tt < ntiles) { mbar_expect_tx(&full[sr], TILE * 4); bulk_load(sm + sr * TILE, x + tt * TILE, TILE * 4, &full[sr]); }
    if (++s == S) { s = 0; ph ^= 1u; }
  }
  bulk_wait<0>();
}

template <int U, int T>
__global__ void __launch_bounds__(T) copyU(const float4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  const int64_t step = (int64_t)gridDim.x * T * U;
  for (int64_t i0 = (int64_t)blockIdx.x * T * U + threadIdx.x; i0 < n4; i0 += step) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i0 + (int64_t)u * T; if (j < n4) v[u] = __ldcs(x + j); }
#pragma unroll
    for (int u = 0; u < U; ++u) { int64_t j = i0 + (int64_t)u * T; if (j < n4) __stcs(y + j, v[u]); }
  }
}

// V5: non-persistent, one trip per thread (grid covers the tensor)
template <int U, int T>
__global__ void __launch_bounds__(T) v5(const float4* __restrict__ x, float4* __restrict__ y,
                                        int64_t n4, uint64_t key, Op op, uint32_t m32,
                                        uint32_t* st) {
  float nf = 0.f;
  const int64_t i0 = (int64_t)blockIdx.x * T * U + threadIdx.x;
  float4 v[U];
#pragma unroll
  for (int u = 0; u < U; ++u) { int64_t j = i0 + (int64_t)u * T; if (j < n4) v[u] = __ldcs(x + j); }
#pragma unroll
  for (int u = 0; u < U; ++u) {
    int64_t j = i0 + (int64_t)u * T;
    if (j < n4) __stcs(y + j, q4(op, v[u], key ^ (uint64_t)(4 * j), m32, nf));
  }
  if (__any_sync(0xffffffffu, nf != nf) && (threadIdx.x & 31) == 0) atomicOr(st, 1u);
}

__global__ void copy4(const float4* __restrict__ x, float4* __restrict__ y, int64_t n4) {
  const int64_t step = (int64_t)gridDim.x * blockDim.x * 4;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x * 4 + threadIdx.x; i0 < n4; i0 += step) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { int64_t j = i0 + (int64_t)u * blockDim.x; if (j < n4) v[u] = __ldcs(x + j); }
#pragma unroll
    for (int u = 0; u < 4; ++u) { int64_t j = i0 + (int64_t)u * blockDim.x; if (j < n4) __stcs(y + j, v[u]); }
  }
}

__global__ void gen(float* x, int64_t n, uint64_t key) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = (float)(-10.0 + 20.0 * ((double)variate24(key, (uint64_t)i) * 0x1p-24));
}

template <class F>
float time_it(F&& f, int reps = 10) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f();
  std::vector<float> ts;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); ts.push_back(ms);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

int main() {
  const int64_t n = int64_t(1) << 30, n4 = n / 4;
  float *x, *y0, *y1; uint32_t* st;
  CK(cudaMalloc(&x, n * 4)); CK(cudaMalloc(&y0, n * 4)); CK(cudaMalloc(&y1, n * 4));
  CK(cudaMalloc(&st, 4)); CK(cudaMemset(st, 0, 4));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  gen<<<sms * 8, 256>>>(x, n, stream_key(2, 0));
  Op op{make_fixed(8, 4, false, true)};
  const uint64_t key = stream_key(0x15EED, 0);
  const double gb = 8.0 * n / 1e9;
  auto report = [&](const char* name, float ms, float* y) {
    bool same = true;
    if (y != y0) {
      std::vector<uint32_t> a(1 << 20), b(1 << 20);
      for (int64_t off : {int64_t(0), n / 2, n - (1 << 20)}) {
        cudaMemcpy(a.data(), y0 + off, 4 << 20, cudaMemcpyDeviceToHost);
        cudaMemcpy(b.data(), y + off, 4 << 20, cudaMemcpyDeviceToHost);
        same &= std::memcmp(a.data(), b.data(), 4 << 20) == 0;
      }
    }
    std::printf("%-34s %8.3f ms %8.1f GB/s %s\n", name, ms, gb / (ms / 1e3), same ? "same" : "DIFF");
  };
  auto occ = [&](auto kern, int smem) { int b = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, 256, smem); return b; };
  report("copy4 (float4 x4, 256 thr)", time_it([&] { copy4<<<sms * 8, 256>>>((float4*)x, (float4*)y1, n4); }), y0);
  {
    int g = sms * occ(v0<4>, 0);
    report("V0 U=4 (production)", time_it([&] { v0<4><<<g, 256>>>((float4*)x, (float4*)y0, n4, key, op, 32u, st); }), y0);
  }
  { int g = sms * occ(v0<2>, 0); report("V0 U=2", time_it([&] { v0<2><<<g, 256>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
  { int g = sms * occ(v0<8>, 0); report("V0 U=8", time_it([&] { v0<8><<<g, 256>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
  { int g = sms * occ(v1<2>, 0); report("V1 U=2 prefetch", time_it([&] { v1<2><<<g, 256>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
  { int g = sms * occ(v1<4>, 0); report("V1 U=4 prefetch", time_it([&] { v1<4><<<g, 256>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
#define RUN_V3(S_, TILE_) { constexpr int S = S_, TILE = TILE_; const int smem = S * TILE * 4; \
    cudaFuncSetAttribute(v3<S, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    int b = occ(v3<S, TILE>, smem); char nm[64]; std::snprintf(nm, 64, "V3 TMA-ld S=%d x %dKB b=%d", S, TILE / 256, b); \
    report(nm, time_it([&] { v3<S, TILE><<<sms * b, 256, smem>>>(x, y1, n, key, op, 32u, st); }), y1); }
#define RUN_V4(S_, TILE_, T_) { constexpr int S = S_, TILE = TILE_, T = T_; const int smem = S * TILE * 4; \
    cudaFuncSetAttribute(v4<S, TILE, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    int b = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, v4<S, TILE, T>, T, smem); char nm[64]; \
    std::snprintf(nm, 64, "V4 TMA-ld+st S=%d x %dKB T=%d b=%d", S, TILE / 256, T, b); \
    report(nm, time_it([&] { v4<S, TILE, T><<<sms * b, T, smem>>>(x, y1, n, key, op, 32u, st); }), y1); }
#define RUN_TC(S_, TILE_) { constexpr int S = S_, TILE = TILE_; const int smem = S * TILE * 4; \
    cudaFuncSetAttribute(tcopy<S, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    int b = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, tcopy<S, TILE>, 32, smem); char nm[64]; \
    std::snprintf(nm, 64, "TMA copy S=%d x %dKB b=%d", S, TILE / 256, b); \
    report(nm, time_it([&] { tcopy<S, TILE><<<sms * b, 32, smem>>>(x, y1, n); }), y0); }
#define RUN_CU(U_, T_, W_) { char nm[64]; std::snprintf(nm, 64, "copy U=%d T=%d waves=%d", U_, T_, W_); \
    int b = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, copyU<U_, T_>, T_, 0); \
    report(nm, time_it([&] { copyU<U_, T_><<<sms * b * W_, T_>>>((float4*)x, (float4*)y1, n4); }), y0); }
#define RUN_V0W(U_, W_) { char nm[64]; int b = occ(v0<U_>, 0); std::snprintf(nm, 64, "V0 U=%d waves=%d (b=%d)", U_, W_, b); \
    report(nm, time_it([&] { v0<U_><<<sms * b * W_, 256>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
#define RUN_V1W(U_, W_) { char nm[64]; int b = occ(v1<U_>, 0); std::snprintf(nm, 64, "V1 U=%d pf waves=%d (b=%d)", U_, W_, b); \
    report(nm, time_it([&] { v1<U_><<<sms * b * W_, 256>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
#define RUN_V5(U_, T_) { char nm[64]; std::snprintf(nm, 64, "V5 U=%d T=%d one-trip", U_, T_); \
    const int64_t g = (n4 + (int64_t)U_ * T_ - 1) / ((int64_t)U_ * T_); \
    report(nm, time_it([&] { v5<U_, T_><<<(unsigned)g, T_>>>((float4*)x, (float4*)y1, n4, key, op, 32u, st); }), y1); }
  RUN_CU(1, 256, 64) RUN_CU(1, 512, 64) RUN_CU(2, 256, 32)
  RUN_V5(1, 256) RUN_V5(2, 256) RUN_V5(4, 256) RUN_V5(8, 256) RUN_V5(1, 512) RUN_V5(2, 512) RUN_V5(4, 128) RUN_V5(2, 128) RUN_V5(4, 512)
  RUN_V0W(4, 32) RUN_V0W(8, 16)
  CK(cudaDeviceSynchronize());
  uint32_t h; cudaMemcpy(&h, st, 4, cudaMemcpyDeviceToHost);
  std::printf("status %u\n", h);
  return 0;
}
