// Development probe (K1-TC bottleneck analysis). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_<name> tools/<name>.cu
// Feasibility probe (development tool): can a cooperative launch use 2-CTA
// clusters with ~210 KB of shared memory per CTA, and how many clusters fit?
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) probe(int* out) {
  extern __shared__ char sm[];
  sm[threadIdx.x] = 1;
  if (threadIdx.x == 0) atomicAdd(out, 1);
}

int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaMemset(d, 0, 4);
  const int smem = 210 * 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int clusters = -1;
  cfg.gridDim = dim3(148);
  cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, probe, &cfg);
  printf("max active 2-clusters: %d (%s)\n", clusters, cudaGetErrorString(e));
  cudaLaunchAttribute at2[2];
  at2[0] = at[0];
  at2[1].id = cudaLaunchAttributeCooperative;
  at2[1].val.cooperative = 1;
  cfg.attrs = at2;
  cfg.numAttrs = 2;
  for (int g : {148, 2 * clusters}) {
    cfg.gridDim = dim3(g);
    e = cudaLaunchKernelEx(&cfg, probe, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    int h = 0;
    cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
    printf("cooperative+cluster grid %d: launch %s, sync %s, blocks ran %d\n", g, cudaGetErrorString(e),
           cudaGetErrorString(e2), h);
    cudaMemset(d, 0, 4);
  }
  return 0;
}
