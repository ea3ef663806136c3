// Development probe: tcgen05.ld (TMEM -> registers) throughput per SM for the
// 32x32b shapes x16 / x32 / x64 with 4 / 8 / 16 loading warps, alone and with
// one warp issuing back-to-back int8 MMAs (M128 N256 K32) into the other half
// of TMEM — does the epilogue's TMEM read rate survive concurrent MMAs?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_tmem_probe tools/tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma(uint32_t t, uint64_t a, uint64_t b) {
  const uint32_t idesc = (2u << 4) | (1u << 7) | (0u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\ttcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(t), "l"(a), "l"(b), "r"(idesc));
}

template <int X>
__device__ __forceinline__ uint32_t ld(uint32_t taddr);

template <>
__device__ __forceinline__ uint32_t ld<16>(uint32_t t) {
  uint32_t v[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s ^= v[i];
  return s;
}
__device__ __forceinline__ uint32_t ld32(uint32_t t) {
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s ^= v[i];
  return s;
}

// warp 0: MMAs (if mma_on) into columns [0, 256); warps 1..nld: loads from columns [256, 512)
__global__ void __launch_bounds__(544, 1) probe(int iters, int mma_on, int shape, int nld, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536);
  volatile int* stop = reinterpret_cast<volatile int*>(sm + 65536 + 64);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    *stop = 0;
    *reinterpret_cast<int*>(sm + 65536 + 128) = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (mma_on && threadIdx.x == 0) {
      const uint32_t base = smem_u32(sm);
      while (!*stop) {
        for (int k = 0; k < 16; ++k) mma(tmem, desc(base), desc(base + 4096));
      }
    }
  } else if (warp <= nld) {
    const int quad = warp & 3;
    const uint32_t t = tmem + 256 + ((uint32_t)(quad * 32) << 16);
    uint32_t acc = 0;
    const long long c0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int c = 0; c < 256; c += shape) {
        if (shape == 16) acc ^= ld<16>(t + c);
        else acc ^= ld32(t + c);
      }
    }
    const long long c1 = clock64();
    if (acc == 0x5eed) sink[2] = acc;
    if (blockIdx.x == 0 && warp == 1) reinterpret_cast<long long*>(sink)[1] = c1 - c0;
    __syncwarp();
    // the last loading warp to finish releases the MMA warp (it spins on *stop)
    if ((threadIdx.x & 31) == 0 && atomicAdd(reinterpret_cast<int*>(sm + 65536 + 128), 1) == nld - 1) *stop = 1;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  int* sink;
  cudaMalloc(&sink, 32);
  const int smem = 65536 + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 200;
  for (int mma_on = 0; mma_on < 2; ++mma_on)
    for (int shape : {16, 32})
      for (int nld : {4, 8, 16}) {
        probe<<<148, 32 * (1 + nld), smem>>>(10, mma_on, shape, nld, sink);
        cudaDeviceSynchronize();
        probe<<<148, 32 * (1 + nld), smem>>>(iters, mma_on, shape, nld, sink);
        cudaDeviceSynchronize();
        long long cyc[2];
        cudaMemcpy(cyc, sink, 16, cudaMemcpyDeviceToHost);
        // bytes per warp per iteration: 32 lanes x 256 columns x 4 B
        const double bytes = (double)nld * iters * 32 * 256 * 4;
        printf("mma %d  x%-2d  %2d load warps: %6.1f B/cycle/SM  (%s)\n", mma_on, shape, nld, bytes / cyc[1],
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
