// Development probe (K1-TC bottleneck analysis). Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_<name> tools/<name>.cu
// Development probe: tcgen05 int8 MMA throughput (M128 N256 K32, cta_group::1)
// with and without concurrent bulk copies into shared memory, and with the
// conv kernel's operand pattern (weights 9 x 4 KB, window + tap offsets).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b, uint32_t acc) {
  const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(t), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(bar), "r"(par) : "memory");
  return ok;
}

// mode 0: resident operands, same descriptors; 1: conv pattern (A walks 9 taps, B shifts);
// 2: conv pattern, ONE accumulator for every MMA (the conv tile); 3: conv pattern,
// accumulator alternating every MMA; 4: as 2 with random operand bytes;
// copy_bytes > 0: warp 1 streams that many bytes per round into a separate region
__global__ void __launch_bounds__(128, 1) probe(int iters, int mode, int copy_bytes, const uint8_t* src, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  // layout: [0, 64K) operands, [64K, 64K + 96K) copy target, bars at 160K
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 216 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 216 * 1024 + 64);
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = mode == 4 ? (uint32_t)(i * 2654435761u) ^ 0x9e3779b9u : 0x01010101u * (i & 3);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    for (int k = 1; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + k)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  volatile int* stop = reinterpret_cast<volatile int*>(sm + 216 * 1024 + 128);
  if (threadIdx.x == 0) *stop = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    const long long c0 = clock64();
    const uint32_t base = smem_u32(sm);
    for (int it = 0; it < iters; ++it) {
      for (int tp = 0; tp < 9; ++tp) {
        uint64_t a, b;
        if (mode == 0) {
          a = desc(base);
          b = desc(base + 4096);
        } else {
          a = desc(base + 16384 + tp * 4096);                         // weights of tap tp
          b = desc(base + ((tp / 3) * 10 + (tp % 3)) * 256);          // window shifted by the tap
        }
        const uint32_t accb = mode == 1 ? (it & 1) : mode == 3 ? (tp & 1) : mode == 0 ? (it & 1) : 0;
        mma(tmem + accb * 256, a, b, 1);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
    while (!try_wait(smem_u32(bar), 0)) {
    }
    if (blockIdx.x == 0) reinterpret_cast<long long*>(sink)[1] = clock64() - c0;
    *stop = 1;
  } else if (threadIdx.x == 32 && copy_bytes > 0) {
    // three copies of copy_bytes in flight (ring of 3 slots), like the conv loader
    uint32_t par = 0;
    for (int r = 0; !*stop && r < (1 << 30); ++r) {
      const int k = r % 3;
      if (r >= 3) {
        while (!try_wait(smem_u32(bar + 1 + k), (par >> k) & 1)) {
        }
        par ^= 1u << k;
      }
      const uint32_t dst = smem_u32(sm + 64 * 1024 + k * 50 * 1024);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + 1 + k)), "r"(copy_bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src + (size_t)((r * 7 + blockIdx.x * 13) % 64) * 65536), "r"(copy_bytes), "r"(smem_u32(bar + 1 + k)) : "memory");
    }
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v == 0x5eed) sink[0] = v;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  uint8_t* src;
  int* sink;
  cudaMalloc(&src, 64 * 65536 + 200000);
  cudaMemset(src, 1, 64 * 65536 + 200000);
  cudaMalloc(&sink, 16);
  const int smem = 216 * 1024 + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  for (int mode = 0; mode < 5; ++mode)
    for (int cb : {0, 51200}) {
      probe<<<148, 128, smem>>>(50, mode, cb, src, sink);
      cudaEventRecord(e0);
      probe<<<148, 128, smem>>>(iters, mode, cb, src, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = 148.0 * iters * 9 * 2.0 * 128 * 256 * 32;
      long long cyc[2];
      cudaMemcpy(cyc, sink, 16, cudaMemcpyDeviceToHost);
      printf("mode %d copies of %6d B (3 in flight): %.1f TOPS, %.1f SM cycles per MMA (clock64), %.0f MHz %s\n", mode, cb,
             ops / ms / 1e9, cyc[1] / (iters * 9.0), cyc[1] / (ms * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
