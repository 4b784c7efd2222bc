// How many 8-CTA clusters can be co-resident, vs shared memory per CTA (diagnostics).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1, 1, 1) dummy() {}
__global__ void k8(float* o) {
  extern __shared__ float s[];
  if (threadIdx.x == 0) s[0] = 1.f;
  if (o && s[0] == 2.f) o[0] = s[0];
}
int main() {
  for (int cs : {2, 4, 8, 16}) {
    for (int smem : {16 << 10, 64 << 10, 120 << 10, 201 << 10, 227 << 10}) {
      cudaFuncSetAttribute(k8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (cs > 8) cudaFuncSetAttribute(k8, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr;
      attr.id = cudaLaunchAttributeClusterDimension;
      attr.val.clusterDim.x = cs;
      attr.val.clusterDim.y = 1;
      attr.val.clusterDim.z = 1;
      cfg.blockDim = dim3(256);
      cfg.gridDim = dim3(cs * 64);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = &attr;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k8, &cfg);
      printf("cluster %2d smem %3d KB: %d clusters (%d CTAs) %s\n", cs, smem >> 10, n, n * cs, cudaGetErrorString(e));
    }
  }
}
