// Issue-rate probe (diagnostic): HFMA2.BF16 (hmul2) alone, cvt.rn.bf16x2.f32
// alone, and the two interleaved -- whether the conversion shares the
// FMA-heavy pipe with the packed bf16 math.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/pipe_probe scripts/pipe_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hmul2(uint32_t a, uint32_t b) {
  uint32_t d; asm volatile("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b)); return d; }
__device__ __forceinline__ uint32_t cvt2(float a, float b) {
  uint32_t d; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(a), "f"(b)); return d; }

template <int MODE>
__global__ void k(uint32_t* out, int iters) {
  uint32_t r[8]; float f[8];
  for (int i = 0; i < 8; ++i) { r[i] = 0x3f803f80u + threadIdx.x + i; f[i] = 1.0f + i * threadIdx.x; }
  const uint32_t m = 0x3f813f81u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0 || MODE == 2) r[i] = hmul2(r[i], m);
      if (MODE == 1 || MODE == 2) { const uint32_t c = cvt2(f[i], f[(i + 1) & 7]); f[i] = __uint_as_float(c) + 1.0f; }
    }
  }
  uint32_t s = 0; for (int i = 0; i < 8; ++i) s ^= r[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* o; cudaMalloc(&o, 4 * sms * 8 * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 8192;
  const char* names[3] = {"hmul2 only", "cvt.bf16x2 (+FADD) only", "interleaved"};
  for (int rep = 0; rep < 2; ++rep)
  for (int mode = 0; mode < 3; ++mode) {
    float ms;
    cudaEventRecord(e0);
    if (mode == 0) k<0><<<sms * 8, 256>>>(o, iters);
    if (mode == 1) k<1><<<sms * 8, 256>>>(o, iters);
    if (mode == 2) k<2><<<sms * 8, 256>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = (double)sms * 8 * 8 * iters * 8;  // per instruction kind
    printf("%-26s %.3f ms  -> %.2f G warp-instr/s per kind\n", names[mode], ms, warp_instr / ms / 1e6);
  }
  return 0;
}
