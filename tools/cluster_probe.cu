// Max co-resident thread-block clusters per size (1 CTA per SM at the decode core's
// shared-memory footprint), including non-portable sizes 9..16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/cluster_probe.cu -o tools/cluster_probe
#include <cuda_runtime.h>
#include <cstdio>

__global__ void probe_kernel(int* out) {
  extern __shared__ int s[];
  if (threadIdx.x == 0 && out) out[blockIdx.x] = s[0];
}

int main() {
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c = 1; c <= 16; ++c) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(c * 32);
    cfg.blockDim = dim3(576);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    const cudaError_t e = cudaOccupancyMaxActiveClusters(&n, probe_kernel, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d SMs (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}
