// FP64 throughput probe: DMMA m8n8k4 vs DFMA, register-resident (diagnostic).
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma_rate scripts/dmma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[16];
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = __fma_rn(a, b, c[i]);
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int w = 0; w < 2; ++w) {
    float ms;
    cudaEventRecord(e0);
    k_dmma<<<sms * 4, 256>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    // per warp per mma: 8*8*4 MACs = 256 MAC = 512 FLOP
    const double fl = 512.0 * 8 * iters * (sms * 4 * 256 / 32);
    printf("DMMA: %.1f TFLOP/s\n", fl / ms / 1e9);
    cudaEventRecord(e0);
    k_dfma<<<sms * 4, 256>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    const double fl2 = 2.0 * 16 * iters * (double)(sms * 4 * 256);
    printf("DFMA: %.1f TFLOP/s\n", fl2 / ms / 1e9);
  }
  return 0;
}
