// Probe: how many clusters of size C (128 threads, S bytes smem) can be co-resident on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kern(double* p) { extern __shared__ double s[]; s[threadIdx.x] = 1; if (p) p[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("sms %d\n", sms);
  for (int threads : {128, 160, 256}) for (int smem : {90000, 101000, 110000, 200000}) for (int C : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(C * 64); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    int b = -1; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, threads, smem);
    printf("threads %d smem %d C %2d: clusters %d (CTAs %d) blocks/SM %d %s\n", threads, smem, C, n, n * C, b, e ? cudaGetErrorString(e) : "");
  }
  return 0;
}
