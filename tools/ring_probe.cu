// Development probe: cost of the K1-TC stage protocol around
// the MMAs — issuer waits full[s], fences, issues 9 conv-pattern MMAs into one
// accumulator, commits to empty[s]; the loader thread waits empty[s] and
// re-arms full[s] (no copies). Reports SM cycles per MMA (clock64).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_ring_probe tools/ring_probe.cu
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
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

// flags: 1 = fence::after_thread_sync after each full wait, 2 = loader sleeps 32 ns per poll,
//        4 = each stage's operands at their own 51200-byte ring slot (the conv ring layout)
template <int NST>
__global__ void __launch_bounds__(64, 1) ring(int stages, int flags, long long* out, int gap) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 210 * 1024);  // full[NST], empty[NST], done
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 210 * 1024 + 8 * (2 * NST + 1));
  for (int i = threadIdx.x; i < 210 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i * 2654435761u;
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int k = 0; k < 2 * NST + 1; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + k)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  const uint32_t base = smem_u32(sm);
  if (threadIdx.x == 0) {
    const long long c0 = clock64();
    uint32_t par = 0;
    for (int it = 0; it < stages; ++it) {
      const int s = it % NST;
      if (gap) {  // issuer busy `gap` cycles between stages (descriptor / loop overhead)
        const long long g0 = clock64();
        while (clock64() - g0 < gap) {
        }
      }
      while (!try_wait(smem_u32(bar + s), (par >> s) & 1)) {
      }
      par ^= 1u << s;
      if (flags & 1) asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sb = (flags & 4) ? base + s * 51200 : base;  // window at sb, weights at sb + 14336
#pragma unroll
      for (int tp = 0; tp < 9; ++tp)
        mma(tmem, desc(sb + 14336 + tp * 4096), desc(sb + ((tp / 3) * 10 + (tp % 3)) * 256), (it | tp) != 0);
      commit(smem_u32(bar + NST + s));
    }
    commit(smem_u32(bar + 2 * NST));
    while (!try_wait(smem_u32(bar + 2 * NST), 0)) {
    }
    if (blockIdx.x == 0) out[0] = clock64() - c0;
  } else if (threadIdx.x == 32) {
    uint32_t par = 0;
    for (int it = 0; it < stages; ++it) {
      const int s = it % NST;
      if (it >= NST) {
        while (!try_wait(smem_u32(bar + NST + s), (par >> s) & 1))
          if (flags & 2) __nanosleep(32);
        par ^= 1u << s;
      }
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar + s)) : "memory");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* out;
  cudaMalloc(&out, 64);
  const int smem = 210 * 1024 + 256;
  cudaFuncSetAttribute(ring<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(ring<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int stages = 4000;
  for (int gap : {0, 50, 100, 150, 200, 300, 400})
    for (int flags : {7}) {
      long long cyc = 0;
      ring<4><<<148, 64, smem>>>(stages, flags, out, gap);
      cudaMemcpy(&cyc, out, 8, cudaMemcpyDeviceToHost);
      printf("gap %3d cycles between stages: %.1f cycles per MMA %s\n", gap, cyc / (stages * 9.0),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
