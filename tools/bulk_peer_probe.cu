// Development probe: can a CTA bulk-copy global -> the PEER CTA's shared memory
// (cluster of 2) with complete_tx on its OWN mbarrier?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_bulk_peer_probe tools/bulk_peer_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __cluster_dims__(2, 1, 1) probe(const uint8_t* src, int* out) {
  __shared__ __align__(128) uint8_t buf[4096];
  __shared__ __align__(8) uint64_t bar;
  unsigned rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = 0;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0 && threadIdx.x == 0) {
    uint32_t dst_local = (uint32_t)__cvta_generic_to_shared(buf), dst_peer;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 1;" : "=r"(dst_peer) : "r"(dst_local));
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 4096, [%2];" ::"r"(dst_peer),
                 "l"(src), "r"(b)
                 : "memory");
    uint32_t ok = 0;
    for (int i = 0; i < (1 << 24) && !ok; ++i)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(b) : "memory");
    out[2] = ok;
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 1 && threadIdx.x == 0) {
    int good = 1;
    for (int i = 0; i < 4096; ++i) good &= buf[i] == (uint8_t)(i * 7);
    out[rank] = good;
  }
}

int main() {
  uint8_t h[4096];
  for (int i = 0; i < 4096; ++i) h[i] = (uint8_t)(i * 7);
  uint8_t* src;
  int* out;
  cudaMalloc(&src, 4096);
  cudaMalloc(&out, 16);
  cudaMemcpy(src, h, 4096, cudaMemcpyHostToDevice);
  cudaMemset(out, 0, 16);
  probe<<<2, 128>>>(src, out);
  cudaError_t e = cudaDeviceSynchronize();
  int r[4] = {0};
  cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
  printf("launch %s; leader barrier completed %d; peer data correct %d\n", cudaGetErrorString(e), r[2], r[1]);
  return 0;
}
