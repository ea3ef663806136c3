// Development probe (K1-TC bottleneck analysis). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_<name> tools/<name>.cu
// Development probe: aggregate L2 -> shared-memory bulk-copy bandwidth with
// k copies in flight per SM (the conv loader's pattern), all 148 SMs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}

__global__ void __launch_bounds__(32, 1) probe(int rounds, int bytes, int inflight, const uint8_t* src, size_t span, int shared_w) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 200 * 1024);
  if (threadIdx.x == 0) {
    for (int i = 0; i < inflight; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + i)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    uint32_t par = 0;
    const int slot_bytes = (200 * 1024 / inflight) & ~1023;
    for (int r = 0; r < rounds; ++r) {
      const int s = r % inflight;
      if (r >= inflight) {
        while (!try_wait(smem_u32(bar + s), (par >> s) & 1)) {
        }
        par ^= 1u << s;
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + s)), "r"(bytes) : "memory");
      if (shared_w) {
        // conv pattern: 36 KB of weights shared by all CTAs of the same ob (4 groups) + a private 14 KB window
        const size_t woff = ((size_t)(blockIdx.x % 4) * 16 + (r % 16)) * 36864;
        const size_t xoff = (32ull << 20) + ((size_t)(blockIdx.x * 7919 + r * 104729) * 4096) % (16ull << 20);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + s * slot_bytes)), "l"(src + woff), "r"(36864), "r"(smem_u32(bar + s)) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + s * slot_bytes + 36864)), "l"(src + xoff), "r"(bytes - 36864), "r"(smem_u32(bar + s)) : "memory");
      } else {
        const size_t off = ((size_t)(blockIdx.x * 7919 + r * 104729) * 4096) % (span - bytes);
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(sm + s * slot_bytes)), "l"(src + (off & ~(size_t)255)), "r"(bytes), "r"(smem_u32(bar + s)) : "memory");
      }
    }
    for (int s = 0; s < inflight; ++s) {
      while (!try_wait(smem_u32(bar + s), (par >> s) & 1)) {
      }
    }
  }
}

int main() {
  const size_t span = 64ull << 20;  // 64 MB: L2-resident after the first pass
  uint8_t* src;
  cudaMalloc(&src, span);
  cudaMemset(src, 1, span);
  const int smem = 200 * 1024 + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int shared_w = 0; shared_w < 2; ++shared_w)
  for (int bytes : {12288, 36864, 51200}) {
    if (shared_w && bytes != 51200) continue;
    for (int inflight : {2, 3, 4}) {
      if (bytes * inflight > 200 * 1024) continue;
      const int rounds = 400;
      probe<<<148, 32, smem>>>(20, bytes, inflight, src, span, shared_w);
      cudaEventRecord(e0);
      probe<<<148, 32, smem>>>(rounds, bytes, inflight, src, span, shared_w);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double b = 148.0 * rounds * bytes;
      printf("%s copy %6d B x %d in flight: %.0f GB/s = %.0f B/clk/SM @1.9GHz  %s\n", shared_w ? "conv-pattern" : "distinct", bytes, inflight, b / ms / 1e6,
             b / (ms * 1e-3 * 1.9e9) / 148, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
