// Max active clusters per cluster size on this GPU (diagnostic):
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/cluster_probe scripts/cluster_probe.cu
// A dummy 512-thread kernel whose dynamic shared memory caps residency at
// 1 or 2 CTAs per SM, like the block-cluster kernel (2 by registers).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) k_dummy(float* p) {
  extern __shared__ float s[];
  if (p) p[threadIdx.x] = s[threadIdx.x];
}

int main() {
  int sms = 0, optin = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int per_sm = 1; per_sm <= 2; ++per_sm) {
    const int smem = optin / per_sm - 2048;
    cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 64, 1, 1);
      cfg.blockDim = dim3(512, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute a[1];
      a[0].id = cudaLaunchAttributeClusterDimension;
      a[0].val.clusterDim.x = cs;
      a[0].val.clusterDim.y = 1;
      a[0].val.clusterDim.z = 1;
      cfg.attrs = a;
      cfg.numAttrs = 1;
      int n = 0;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
      printf("ctas/sm %d cs %2d: max active clusters %3d -> %4d CTAs = %.3f of %d slots %s\n",
             per_sm, cs, n, n * cs, (double)(n * cs) / (sms * per_sm), sms * per_sm,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
