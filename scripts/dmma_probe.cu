// Does the FP64 tensor-core MMA (mma.sync m8n8k4 f64) round like a chain of
// DFMAs in ascending k?  Compares D = A*B + C from one DMMA with
// fma(a3,b3, fma(a2,b2, fma(a1,b1, fma(a0,b0,c)))) on adversarial inputs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/dmma scripts/dmma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// fp32 values (as the quantized_matmul operands are) with wide exponents
__device__ double val(uint64_t r, int mode) {
  float f;
  const uint32_t bits = (uint32_t)r;
  int e = (int)((r >> 32) % (mode ? 60u : 20u)) - (mode ? 30 : 10);
  f = ldexpf(1.0f + (float)(bits & 0xFFFFFF) / 16777216.0f, e);
  if ((r >> 40) & 1) f = -f;
  if (mode == 2 && ((r >> 41) & 3) == 0) f = ldexpf(1.0f, e);  // powers of two: ties
  return (double)f;
}

__global__ void probe(uint64_t seed, int mode, unsigned long long* mism_chain,
                      unsigned long long* mism_fused, unsigned long long* total) {
  const int lane = threadIdx.x & 31;
  const uint64_t base = mix(seed ^ (blockIdx.x * 1315423911ull + (threadIdx.x >> 5)));
  // fragments: A 8x4 row, B 4x8 col: lane holds A[lane/4][lane%4], B[lane%4][lane/4]
  const int ar = lane >> 2, ak = lane & 3;
  double a = val(mix(base ^ (uint64_t)(ar * 4 + ak) * 7919), mode);
  double b = val(mix(base ^ (uint64_t)(100 + ak * 8 + ar) * 104729), mode);
  // C 8x8: lane holds C[lane/4][2*(lane%4) + {0,1}]
  double c0 = val(mix(base ^ (uint64_t)(200 + lane * 2)), mode);
  double c1 = val(mix(base ^ (uint64_t)(201 + lane * 2)), mode);
  if (mode == 2) { c0 = ldexp(c0, 20); c1 = -c1; }
  double d0, d1;
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
  // reference: gather A row and B columns via shuffles
  const int row = lane >> 2;
  double res[2] = {d0, d1}, cc[2] = {c0, c1};
  for (int h = 0; h < 2; ++h) {
    const int col = 2 * (lane & 3) + h;
    double chain = cc[h];
    double ap[4], bp[4];
    for (int k = 0; k < 4; ++k) {
      ap[k] = __shfl_sync(0xFFFFFFFFu, a, row * 4 + k);
      bp[k] = __shfl_sync(0xFFFFFFFFu, b, col * 4 + k);
    }
    for (int k = 0; k < 4; ++k) chain = __fma_rn(ap[k], bp[k], chain);
    // "fused": exact products (fp32*fp32 exact in double) summed with one
    // rounding -- approximated by a double-double sum
    double s = cc[h], err = 0.0;
    for (int k = 0; k < 4; ++k) {
      const double p = ap[k] * bp[k];
      const double t = s + p;
      const double bb = t - s;
      err += (s - (t - bb)) + (p - bb);
      s = t;
    }
    const double fused = s + err;
    if (__double_as_longlong(res[h]) != __double_as_longlong(chain)) atomicAdd(mism_chain, 1ull);
    if (__double_as_longlong(res[h]) != __double_as_longlong(fused)) atomicAdd(mism_fused, 1ull);
    atomicAdd(total, 1ull);
  }
}

int main() {
  unsigned long long *d, h[3];
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(d, 0, 3 * sizeof(unsigned long long));
    for (int it = 0; it < 20; ++it) probe<<<4096, 256>>>(it * 77 + mode, mode, d, d + 1, d + 2);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d: %llu outputs, %llu differ from the DFMA chain, %llu differ from one-rounding sum\n",
           mode, h[2], h[0], h[1]);
  }
  return 0;
}
