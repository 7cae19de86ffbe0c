// runtime.h -- internal helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lpq.h"
#include "kernels.cuh"

namespace lpq {

void note_passes(int n);
// While alive, the calling thread's device calls do not count data passes: a
// host entry point that streams one tensor through several device calls
// (chunks) counts the passes of the whole tensor once itself.
struct PassScope {
  PassScope();
  ~PassScope();
};
lpq_status cuda_fail(cudaError_t e);
lpq_status check_format(const lpq_format* f);
lpq_status check_shape(const int64_t* shape, int rank, int64_t* numel);
lpq_status block_geometry(const lpq_format* f, const int64_t* shape, int rank,
                          BlockGeom* g);
lpq_status map_status_bits(uint32_t bits);
lpq_status quantize_device(const float* x, float* y, const int64_t* shape,
                           int rank, uint64_t index_base, const lpq_format* f,
                           int mode, uint64_t seed, uint64_t call, void* ws,
                           size_t ws_bytes, uint32_t* d_status,
                           cudaStream_t s);

lpq_status quantize_composed_device(const float* x, float* y,
                                    const int64_t* shape, int rank,
                                    uint64_t index_base, const lpq_format* f,
                                    int mode, uint64_t seed, uint64_t call,
                                    void* ws, size_t ws_bytes,
                                    uint32_t* status, cudaStream_t s);

// Scoped cudaSetDevice (restores the caller's device).
class DeviceGuard {
 public:
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev_);
    if (dev >= 0 && dev != prev_) {
      cudaSetDevice(dev);
      switched_ = true;
    }
  }
  ~DeviceGuard() {
    if (switched_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0;
  bool switched_ = false;
};

}  // namespace lpq
