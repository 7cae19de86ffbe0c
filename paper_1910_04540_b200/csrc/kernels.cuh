// kernels.cuh -- launch interfaces of the sm_100a quantizer kernels.
// Internal to liblpq.so; the public boundary is include/lpq.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "quant_math.cuh"

namespace lpq {

// Error bits the kernels OR into the caller's device status word.
enum : uint32_t { kStatusNonFinite = 1u, kStatusBlockRange = 2u,
                  kStatusInvalidValue = 4u };

struct DeviceInfo {
  int sm_count;
  int max_smem_optin;
};
const DeviceInfo& device_info();  // of the current device (cached)

void note_launch(int n = 1);      // library-wide launch counter

// ---- elementwise float / fixed (one HBM pass) ----------------------------
// x, y: device fp32 (4-byte aligned); n elements; base: flat index of x[0].
cudaError_t launch_fixed(const float* x, float* y, int64_t n, uint64_t base,
                         uint64_t key, const FixedParams& p, int mode,
                         uint32_t* status, cudaStream_t s);
cudaError_t launch_float(const float* x, float* y, int64_t n, uint64_t base,
                         uint64_t key, const FloatParams& p, int mode,
                         uint32_t* status, cudaStream_t s);

// ---- block floating point -------------------------------------------------
// The tensor is viewed as [outer, extent, stride]; block b = index along
// `extent` (whole tensor: outer = extent = 1, stride = n).
struct BlockGeom {
  int64_t outer;
  int64_t extent;
  int64_t stride;
};

// Which plan a block quantization uses (and how many HBM passes it makes).
enum class BlockPlan { kRowsInRegisters, kRowsCluster, kRowsChunked,
                       kTwoPassSegments, kTwoPassColumns };
BlockPlan block_plan(const BlockGeom& g, const float* x, const float* y);
// the cluster (single-pass) plan can run this geometry
bool block_cluster_ok(const BlockGeom& g, const float* x, const float* y);
inline int block_plan_passes(BlockPlan p) {
  return (p == BlockPlan::kRowsInRegisters || p == BlockPlan::kRowsCluster ||
          p == BlockPlan::kRowsChunked) ? 1 : 2;
}
inline bool block_plan_single_pass(BlockPlan p) { return block_plan_passes(p) == 1; }
// the plan leaves max|x| bits per block in ws[0 .. extent) (u32)
inline bool block_plan_maxima_in_ws(BlockPlan p) {
  return p == BlockPlan::kRowsChunked || !block_plan_single_pass(p);
}
// cluster plan (block_cluster.cu): CTAs per row for a contiguous block of L
// floats, 0 if too long
int cluster_size_for(int64_t L);
cudaError_t launch_block_cluster(const float* x, float* y, int64_t L,
                                 int64_t nrows, uint64_t base, uint64_t key,
                                 int wl, int mode, uint32_t* status,
                                 cudaStream_t s);
// chunk-rendezvous plan (block_chunks.cu): nrows contiguous rows of L floats
// (L % 4 == 0, 16-byte aligned x / y), single HBM pass, workspace
// block_chunks_workspace(nrows) bytes (rowmax[nrows] first)
bool block_chunks_ok(int64_t L, int64_t nrows);
size_t block_chunks_workspace(int64_t nrows);
cudaError_t launch_block_chunks(const float* x, float* y, int64_t L, int64_t nrows,
                                uint64_t base, uint64_t key, int wl, int mode, void* ws,
                                uint32_t* status, cudaStream_t s);
// Workspace bytes for a plan: extent uint32 maxima (two-pass plans), the
// chunk plan's row state; 0 for the other single-pass plans.
size_t block_workspace(const BlockGeom& g, BlockPlan p);

cudaError_t launch_block(const float* x, float* y, const BlockGeom& g,
                         BlockPlan plan, uint64_t base, uint64_t key, int wl,
                         int mode, void* ws, uint32_t* status, cudaStream_t s);

cudaError_t launch_block_reduce(const float* x, const BlockGeom& g,
                                uint32_t* maxima, cudaStream_t s);
// the quantize pass alone, with maxima[extent] given (max|x| bits per block)
cudaError_t launch_block_apply(const float* x, float* y, const BlockGeom& g,
                               const uint32_t* maxima, uint64_t base, uint64_t key,
                               int wl, int mode, uint32_t* status, cudaStream_t s);

// ---- generators -------------------------------------------------------------
// One-byte codes of quantized values for the host path's device->host copy
// (runtime.cu): see ByteCode.  q: quantized fp32 values (device), c: codes.
struct ByteCode {
  int32_t kind;     // 0: none, 1: fixed (k = q * 2^fl), 2: float (sign|E|man)
  float scale;      // fixed: 2^fl
  int32_t man;      // float: mantissa bits kept
  int32_t min_exp;  // float: exponent of code E = 1
};
cudaError_t launch_encode8(const float* q, uint8_t* c, int64_t n, const ByteCode& bc,
                           cudaStream_t s);
// Block formats with wl <= 8 (NearestEven / Stochastic: zeros are +0):
// code = k = q / delta_b, delta_b = 2^(E_b - (wl - 2)) from the block maxima
// (max|x| bits, maxima[extent], the two-pass plans' workspace); the host
// decodes float(double(k) * delta_b).  An element whose q is not exactly
// k * delta_b (a result in the fp32 subnormal range that rounded) sets
// *not_exact, and the caller copies the fp32 values instead.
cudaError_t launch_encode_block8(const float* q, uint8_t* c, const BlockGeom& g,
                                 const uint32_t* maxima, int wl, uint32_t* not_exact,
                                 cudaStream_t s);

// ---- programmatic dependent launch (LPQ_PDL=0 disables it) -----------------
// A kernel launched by launch_pdl may be scheduled while the previous kernel
// of the stream drains; it calls pdl_trigger() first (so its own successor
// can only be scheduled once every CTA of this grid has started) and
// pdl_wait() before its first global memory access (which returns once the
// predecessor has completed and its writes are visible).  Without the launch
// attribute both are no-ops.  Used by k_elementwise; the block-row and
// grouped kernels under it measured no different (C5 6284-6285 either way).
bool pdl_enabled();
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, cudaStream_t s,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, args...);
}

cudaError_t launch_uniform(float* y, int64_t n, uint64_t base, uint64_t key,
                           float lo, float hi, cudaStream_t s);
cudaError_t launch_variates(float* y, int64_t n, uint64_t base, uint64_t key,
                            cudaStream_t s);

// ---- GEMMs ------------------------------------------------------------------
struct GemmScan {        // pre-scan of A and B (device-written)
  uint32_t a_min_nz_exp_field;  // min exponent field over nonzero |a| (255 if none)
  uint32_t a_max_exp_field;
  uint32_t b_min_nz_exp_field;
  uint32_t b_max_exp_field;
  uint32_t a_low_bits;          // OR of (bits & 0xFFFF) over A: 0 iff bf16-exact
  uint32_t b_low_bits;
  uint32_t nonfinite;           // any non-finite in A or B
  uint32_t pad;
};

cudaError_t launch_quant_gemm(const float* A, const float* B, float* C,
                              int64_t M, int64_t N, int64_t K,
                              int64_t row_base, const FloatParams& qm,
                              const FloatParams& qa, bool bf16_formats,
                              int mode, uint64_t seed, uint64_t call,
                              GemmScan* scan, uint32_t* status,
                              cudaStream_t s);

cudaError_t launch_matmul_q(const float* A, const float* B, float* C,
                            int64_t M, int64_t N, int64_t K, int64_t row_base,
                            int kind, const FloatParams& fp,
                            const FixedParams& xp, int mode, uint64_t key,
                            uint32_t* status, cudaStream_t s);

}  // namespace lpq
