// cvt_pipe_probe.cu -- which issue pipe does cvt.rn.bf16x2.f32 (F2FP) share?
// Times dependent-free streams of HADD2.BF16, F2FP, FMUL and their mixes on
// one B200; if a mix takes the sum of its parts' times, they share a pipe.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/cvt_pipe_probe.cu -o build/cvt_pipe_probe
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

__device__ __forceinline__ uint32_t badd2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t cvt2(float hi, float lo) {
  uint32_t d;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}

// MODE bit 0: HADD2 stream, bit 1: F2FP stream, bit 2: FMUL stream
template <int MODE>
__global__ void k(uint32_t* out, float s, int iters) {
  uint32_t a[8];
  float f[8];
  for (int i = 0; i < 8; ++i) {
    a[i] = threadIdx.x * 7u + i;
    f[i] = (float)(threadIdx.x + i) * 1e-3f;
  }
  uint32_t c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE & 1) a[i] = badd2(a[i], 0x3f803f80u);
      if (MODE & 2) c[i] ^= cvt2(f[i], f[(i + 1) & 7]);
      if (MODE & 4) f[i] = f[i] * s;
    }
  }
  uint32_t r = 0;
  for (int i = 0; i < 8; ++i) r ^= a[i] ^ c[i] ^ __float_as_uint(f[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
float run(uint32_t* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<148 * 4, 256>>>(out, 1.0000001f, iters);
  cudaEventRecord(e0);
  k<MODE><<<148 * 4, 256>>>(out, 1.0000001f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, sizeof(uint32_t) * 148 * 4 * 256);
  const int it = 4096;
  printf("HADD2       %.3f ms\n", run<1>(out, it));
  printf("F2FP        %.3f ms\n", run<2>(out, it));
  printf("FMUL        %.3f ms\n", run<4>(out, it));
  printf("HADD2+F2FP  %.3f ms\n", run<3>(out, it));
  printf("HADD2+FMUL  %.3f ms\n", run<5>(out, it));
  printf("F2FP+FMUL   %.3f ms\n", run<6>(out, it));
  printf("all three   %.3f ms\n", run<7>(out, it));
  return 0;
}
