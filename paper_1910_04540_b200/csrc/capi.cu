// capi.cu -- the extern "C" boundary of liblpq.so (include/lpq.h): argument
// and format validation, dispatch to the sm_100a kernels, status mapping.
//
// Mirrors the reference entry points:
//   lpq_quantize         <- quantize_fused_at   proj/src/quant_ops.cpp:154-164
//   lpq_validate_format  <- validate            proj/include/lpsim/formats.hpp:82-112
//   lpq_uniform          <- random_uniform      proj/src/tensor.cpp:430-440
//   lpq_variates         <- variate_tensor      proj/src/tensor.cpp:281-290
//   lpq_pass_count       <- pass_count          proj/src/tensor.cpp:306-307
// No C++ exception crosses this file's functions; CUDA errors become
// LPQ_ERR_CUDA with the message kept in lpq_last_cuda_error().
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lpq.h"
#include "kernels.cuh"
#include "runtime.h"

namespace lpq {

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<uint64_t> g_passes{0};
thread_local std::string t_cuda_error;
std::mutex g_dev_mu;
std::vector<DeviceInfo> g_dev_info;
std::vector<bool> g_dev_known;
}  // namespace

void note_launch(int n) { g_launches.fetch_add((uint64_t)n, std::memory_order_relaxed); }
namespace {
thread_local int t_pass_scope = 0;  // > 0: inside a host call that counts itself
}
void note_passes(int n) {
  if (t_pass_scope == 0) g_passes.fetch_add((uint64_t)n, std::memory_order_relaxed);
}
PassScope::PassScope() { ++t_pass_scope; }
PassScope::~PassScope() { --t_pass_scope; }

lpq_status cuda_fail(cudaError_t e) {
  t_cuda_error = cudaGetErrorString(e);
  return e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver
             ? LPQ_ERR_NO_DEVICE
             : LPQ_ERR_CUDA;
}

const DeviceInfo& device_info() {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if ((int)g_dev_info.size() <= dev) {
    g_dev_info.resize(dev + 1);
    g_dev_known.resize(dev + 1, false);
  }
  if (!g_dev_known[dev]) {
    DeviceInfo di{148, 227 * 1024};
    cudaDeviceGetAttribute(&di.sm_count, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&di.max_smem_optin,
                           cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    g_dev_info[dev] = di;
    g_dev_known[dev] = true;
  }
  return g_dev_info[dev];
}

lpq_status check_format(const lpq_format* f) {
  if (!f) return LPQ_ERR_ARGUMENT;
  switch (f->kind) {
    case LPQ_FLOAT:
      if (f->exp_bits < 1 || f->exp_bits > 8) return LPQ_ERR_FORMAT;
      if (f->man_bits < 0 || f->man_bits > 23) return LPQ_ERR_FORMAT;
      return LPQ_OK;
    case LPQ_FIXED:
      if (f->wl < 2 || f->wl > 24) return LPQ_ERR_FORMAT;
      if (f->fl < f->wl - 128 || f->fl > 126) return LPQ_ERR_FORMAT;
      return LPQ_OK;
    case LPQ_BLOCK:
      if (f->wl < 2 || f->wl > 24) return LPQ_ERR_FORMAT;
      if (f->block_dim < -1) return LPQ_ERR_FORMAT;
      return LPQ_OK;
    default:
      return LPQ_ERR_FORMAT;
  }
}

lpq_status check_shape(const int64_t* shape, int rank, int64_t* numel) {
  if (rank < 0 || (rank > 0 && !shape)) return LPQ_ERR_ARGUMENT;
  int64_t n = 1;
  bool zero = false;
  for (int d = 0; d < rank; ++d) {
    if (shape[d] < 0) return LPQ_ERR_SHAPE;  // tensor.cpp:237-244
    if (shape[d] == 0) zero = true;
  }
  for (int d = 0; d < rank && !zero; ++d) {
    if (shape[d] > INT64_MAX / 4 / n) return LPQ_ERR_SHAPE;  // bytes overflow int64
    n *= shape[d];
  }
  if (zero) n = 0;
  *numel = n;
  return LPQ_OK;
}

lpq_status block_geometry(const lpq_format* f, const int64_t* shape, int rank,
                          BlockGeom* g) {
  int64_t n = 1;
  for (int d = 0; d < rank; ++d) n *= shape[d];
  if (f->block_dim < 0) {
    *g = BlockGeom{1, 1, n};
    return LPQ_OK;
  }
  if (f->block_dim >= rank) return LPQ_ERR_SHAPE;  // quant_ops.cpp:70-71
  int64_t outer = 1, inner = 1;
  for (int d = 0; d < f->block_dim; ++d) outer *= shape[d];
  for (int d = f->block_dim + 1; d < rank; ++d) inner *= shape[d];
  *g = BlockGeom{outer, shape[f->block_dim], inner};
  return LPQ_OK;
}

lpq_status map_status_bits(uint32_t bits) {
  // the earliest op of the reference's chain throws first: the composed
  // chain's validation, then fused_block's pass 1, then the quantize pass
  if (bits & kStatusInvalidValue) return LPQ_ERR_INVALID_VALUE;
  if (bits & kStatusBlockRange) return LPQ_ERR_BLOCK_RANGE;
  if (bits & kStatusNonFinite) return LPQ_ERR_INVALID_INPUT;
  return LPQ_OK;
}

lpq_status quantize_device(const float* x, float* y, const int64_t* shape,
                           int rank, uint64_t index_base, const lpq_format* f,
                           int mode, uint64_t seed, uint64_t call, void* ws,
                           size_t ws_bytes, uint32_t* d_status,
                           cudaStream_t s) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
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
  if (!x || !y || !d_status) return LPQ_ERR_ARGUMENT;
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 3u)
    return LPQ_ERR_ARGUMENT;
  const uint64_t key = stream_key(seed, call);
  cudaError_t e = cudaSuccess;
  if (f->kind == LPQ_FIXED) {
    const FixedParams p = make_fixed(f->wl, f->fl, f->symmetric != 0, f->saturate != 0);
    e = launch_fixed(x, y, n, index_base, key, p, mode, d_status, s);
    note_passes(1);
  } else if (f->kind == LPQ_FLOAT) {
    const FloatParams p = make_float(f->exp_bits, f->man_bits);
    e = launch_float(x, y, n, index_base, key, p, mode, d_status, s);
    note_passes(1);
  } else {
    BlockPlan plan = block_plan(g, x, y);
    const size_t need = block_workspace(g, plan);
    if (need > 0 && (!ws || ws_bytes < need)) {
      if (!block_cluster_ok(g, x, y)) return LPQ_ERR_WORKSPACE;
      plan = BlockPlan::kRowsCluster;  // single pass, no workspace
    }
    e = launch_block(x, y, g, plan, index_base, key, f->wl, mode, ws, d_status, s);
    note_passes(block_plan_passes(plan));
  }
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

}  // namespace lpq

using namespace lpq;

extern "C" {

int lpq_abi_version(void) { return LPQ_ABI_VERSION; }

const char* lpq_status_string(lpq_status s) {
  switch (s) {
    case LPQ_OK: return "ok";
    case LPQ_ERR_FORMAT: return "format_error: number format parameters out of range";
    case LPQ_ERR_SHAPE: return "shape_error: block dimension out of range or bad shape";
    case LPQ_ERR_INVALID_INPUT: return "invalid_input_error: quantize: non-finite input";
    case LPQ_ERR_UNSUPPORTED: return "unsupported_format_error: operation does not support the format";
    case LPQ_ERR_BLOCK_RANGE: return "invalid_input_error: block maximum too large to represent";
    case LPQ_ERR_ARGUMENT: return "invalid argument (null or misaligned pointer, bad mode or rank)";
    case LPQ_ERR_WORKSPACE: return "workspace too small";
    case LPQ_ERR_CUDA: return "CUDA runtime error";
    case LPQ_ERR_NO_DEVICE: return "no CUDA device available";
    case LPQ_ERR_INVALID_VALUE: return "invalid_value_error: non-finite result";
  }
  return "unknown status";
}

lpq_status lpq_validate_format(const lpq_format* f) { return check_format(f); }

size_t lpq_workspace_size(const lpq_format* f, const int64_t* shape, int rank) {
  if (!f || f->kind != LPQ_BLOCK || check_format(f) != LPQ_OK) return 0;
  int64_t n = 0;
  if (check_shape(shape, rank, &n) != LPQ_OK) return 0;
  BlockGeom g;
  if (block_geometry(f, shape, rank, &g) != LPQ_OK) return 0;
  // upper bound over plans (the plan also depends on pointer alignment)
  return std::max(block_workspace(g, BlockPlan::kTwoPassColumns),
                  block_workspace(g, BlockPlan::kRowsChunked));
}

uint64_t lpq_launch_count(void) { return g_launches.load(); }
uint64_t lpq_pass_count(void) { return g_passes.load(); }
void lpq_reset_pass_count(void) { g_passes.store(0); }
const char* lpq_last_cuda_error(void) { return t_cuda_error.c_str(); }

lpq_status lpq_quantize(const float* x, float* y, const int64_t* shape,
                        int rank, uint64_t index_base, const lpq_format* f,
                        int mode, uint64_t seed, uint64_t call, void* ws,
                        size_t ws_bytes, uint32_t* d_status, void* stream) {
  return quantize_device(x, y, shape, rank, index_base, f, mode, seed, call,
                         ws, ws_bytes, d_status, static_cast<cudaStream_t>(stream));
}

static lpq_status block_split_args(const float* x, const int64_t* shape, int rank,
                                   const lpq_format* f, BlockGeom* g, int64_t* n) {
  lpq_status st = check_format(f);
  if (st != LPQ_OK) return st;
  if (f->kind != LPQ_BLOCK) return LPQ_ERR_UNSUPPORTED;
  st = check_shape(shape, rank, n);
  if (st != LPQ_OK) return st;
  st = block_geometry(f, shape, rank, g);
  if (st != LPQ_OK) return st;
  if (*n > 0 && (!x || (reinterpret_cast<uintptr_t>(x) & 3u))) return LPQ_ERR_ARGUMENT;
  return LPQ_OK;
}

lpq_status lpq_block_absmax(const float* x, const int64_t* shape, int rank,
                            const lpq_format* f, uint32_t* maxima, void* stream) {
  BlockGeom g;
  int64_t n = 0;
  lpq_status st = block_split_args(x, shape, rank, f, &g, &n);
  if (st != LPQ_OK) return st;
  if (g.extent == 0) return LPQ_OK;
  if (!maxima) return LPQ_ERR_ARGUMENT;
  // launch_block_reduce zeroes maxima first (an empty part contributes 0)
  cudaError_t e = launch_block_reduce(x, g, maxima, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

lpq_status lpq_quantize_block_apply(const float* x, float* y, const int64_t* shape,
                                    int rank, uint64_t index_base,
                                    const lpq_format* f, int mode, uint64_t seed,
                                    uint64_t call, const uint32_t* maxima,
                                    uint32_t* d_status, void* stream) {
  BlockGeom g;
  int64_t n = 0;
  lpq_status st = block_split_args(x, shape, rank, f, &g, &n);
  if (st != LPQ_OK) return st;
  if (mode < 0 || mode > 3) return LPQ_ERR_ARGUMENT;
  if (n == 0) return LPQ_OK;
  if (!y || !maxima || !d_status || (reinterpret_cast<uintptr_t>(y) & 3u))
    return LPQ_ERR_ARGUMENT;
  cudaError_t e = launch_block_apply(x, y, g, maxima, index_base, stream_key(seed, call),
                                     f->wl, mode, d_status, static_cast<cudaStream_t>(stream));
  note_passes(1);
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

lpq_status lpq_status_fetch(uint32_t* d_status, void* stream) {
  if (!d_status) return LPQ_ERR_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  uint32_t bits = 0;
  cudaError_t e = cudaMemcpyAsync(&bits, d_status, sizeof(bits),
                                  cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e == cudaSuccess && bits) e = cudaMemsetAsync(d_status, 0, sizeof(uint32_t), s);
  if (e != cudaSuccess) return cuda_fail(e);
  return map_status_bits(bits);
}

lpq_status lpq_uniform(float* y, int64_t n, uint64_t index_base, uint64_t seed,
                       uint64_t call, float lo, float hi, void* stream) {
  if (n < 0 || (n > 0 && !y)) return LPQ_ERR_ARGUMENT;
  cudaError_t e = launch_uniform(y, n, index_base, stream_key(seed, call), lo,
                                 hi, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

lpq_status lpq_variates(float* y, int64_t n, uint64_t index_base,
                        uint64_t seed, uint64_t call, void* stream) {
  if (n < 0 || (n > 0 && !y)) return LPQ_ERR_ARGUMENT;
  cudaError_t e = launch_variates(y, n, index_base, stream_key(seed, call),
                                  static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? LPQ_OK : cuda_fail(e);
}

}  // extern "C"
