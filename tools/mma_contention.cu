// Development probe: does concurrent epilogue-like work slow the int8 MMAs?
// Warp 0 times NM back-to-back tcgen05.mma.kind::i8 (M128 N256 K32) into TMEM
// columns [0, 256) (commit -> mbarrier -> clock64); warps 1..nw meanwhile run
//   mode 0: nothing        mode 1: tcgen05.ld x32 from columns [256, 512)
//   mode 2: IMAD-heavy arithmetic only (no TMEM)
//   mode 3: tcgen05.ld x32 + the arithmetic (an epilogue without stores)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/_mma_contention tools/mma_contention.cu
#include <cstdint>
#include <cstdio>
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

__device__ __forceinline__ void ld32(uint32_t t, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
}

__device__ __forceinline__ long long mad_wide(int32_t a, int32_t b, long long c) {
  long long d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

__global__ void __launch_bounds__(544, 1) probe(int nm, int mode, int nw, int k8, int skip0, int lean, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint32_t* slot = reinterpret_cast<uint32_t*>(sm + 65536);
  volatile int* stop = reinterpret_cast<volatile int*>(sm + 65536 + 64);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536 + 128);
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x01010101u * (i & 3);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    *stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) {
      const uint32_t base = smem_u32(sm);
      // let the other warps get going
      const long long w0 = clock64();
      while (clock64() - w0 < 20000) {
      }
      const long long c0 = clock64();
      if (lean == 2) {  // descriptors precomputed in VECTOR registers: one vector->uniform move per operand
        uint32_t va[7], vb[7];
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          asm volatile("mov.u32 %0, %1;" : "=r"(va[j]) : "r"((uint32_t)desc(base + j * 4096)));
          asm volatile("mov.u32 %0, %1;" : "=r"(vb[j]) : "r"((uint32_t)desc(base + 32768 + j * 256)));
        }
        const uint32_t hi = (uint32_t)(desc(base) >> 32);
        for (int k = 0; k + 7 <= nm; k += 7) {
#pragma unroll
          for (int j = 0; j < 7; ++j) {
            uint64_t a, b;
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(va[j]), "r"(hi));
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(b) : "r"(vb[j]), "r"(hi));
            mma(tmem, a, b, 1u);
          }
        }
      } else if (lean == 3) {  // + one vector add per MMA (the B operand's tap offset)
        uint32_t va[7], vb[7];
#pragma unroll
        for (int j = 0; j < 7; ++j) {
          asm volatile("mov.u32 %0, %1;" : "=r"(va[j]) : "r"((uint32_t)desc(base + j * 4096)));
          asm volatile("mov.u32 %0, %1;" : "=r"(vb[j]) : "r"((uint32_t)(j * 16)));
        }
        uint32_t b0;
        asm volatile("mov.u32 %0, %1;" : "=r"(b0) : "r"((uint32_t)desc(base + 32768)));
        const uint32_t hi = (uint32_t)(desc(base) >> 32);
        for (int k = 0; k + 7 <= nm; k += 7) {
#pragma unroll
          for (int j = 0; j < 7; ++j) {
            uint64_t a, b;
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(a) : "r"(va[j]), "r"(hi));
            asm volatile("mov.b64 %0, {%1, %2};" : "=l"(b) : "r"(b0 + vb[j]), "r"(hi));
            mma(tmem, a, b, 1u);
          }
          asm volatile("add.u32 %0, %0, 0;" : "+r"(b0));
        }
      } else if (lean) {  // descriptors precomputed: the issue loop has no multiply / modulo
        uint64_t da[7], db[7];
#pragma unroll
        for (int j = 0; j < 7; ++j) da[j] = desc(base + j * 4096), db[j] = desc(base + 32768 + j * 256);
        mma(tmem, da[0], db[0], 0u);
        for (int k = 1; k + 7 <= nm; k += 7) {
#pragma unroll
          for (int j = 0; j < 7; ++j) mma(tmem, da[j], db[j], 1u);
        }
      } else {
        for (int k = 0; k < nm; ++k)
          mma(tmem, desc(base + (k % 7) * 4096), desc(base + 32768 + (k % 7) * 256), k ? 1u : 0u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                   : "memory");
      uint32_t ok = 0;
      while (!ok)
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar))
            : "memory");
      const long long c1 = clock64();
      if (blockIdx.x == 0) out[0] = c1 - c0;
      *stop = 1;
    }
  } else if (warp <= nw && mode && !(skip0 && (warp & 3) == 0)) {
    const int quad = warp & 3;
    const uint32_t t = tmem + 256 + ((uint32_t)(quad * 32) << 16);
    uint32_t v[32];
    for (int i = 0; i < 32; ++i) v[i] = threadIdx.x * 7 + i;
    long long acc = 0;
    long long its = 0;
    while (!*stop) {
      for (int c = 0; c < 256; c += 32) {
        if (mode & 1) ld32(t + c, v);
        if (mode & 4) {  // ALU-only arithmetic (no IMAD)
#pragma unroll
          for (int j = 0; j < 32; ++j) acc = (acc ^ (long long)v[j]) + ((acc >> 3) | (long long)v[(j + 5) & 31]);
        } else if (mode & 2) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int32_t* P = reinterpret_cast<const int32_t*>(v + 8 * j);
            long long lo = mad_wide(P[3], k8 * k8 * k8, mad_wide(P[2], k8 * k8, mad_wide(P[1], k8, mad_wide(P[0], 1, acc))));
            long long hi = mad_wide(P[7], k8 * k8 * k8, mad_wide(P[6], k8 * k8, mad_wide(P[5], k8, mad_wide(P[4], 1, lo))));
            acc ^= hi + (long long)__umul64hi((unsigned long long)hi, 0x123456789abcdefull) * 77;
          }
        } else {
          acc += v[c & 31];
        }
      }
      ++its;
    }
    if (acc == 0x5eed) out[2] = acc;
    if (blockIdx.x == 0 && threadIdx.x == 32) out[1] = its;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  long long* out;
  cudaMalloc(&out, 64);
  const int smem = 65536 + 256;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int nm = 4096;
  const char* names[] = {"idle", "tmem ld", "compute", "ld+compute", "alu", "ld+alu"};
  for (int lean = 0; lean < 4; ++lean)
  for (int mode : {0, 2, 3})
    for (int nw : {8, 12})
      for (int skip0 = 0; skip0 < 1; ++skip0) {
        if (mode == 0 && (nw > 8 || skip0)) continue;
        probe<<<148, 32 * (1 + nw), smem>>>(64, mode, nw, 256, skip0, lean, out);
        cudaDeviceSynchronize();
        probe<<<148, 32 * (1 + nw), smem>>>(nm, mode, nw, 256, skip0, lean, out);
        cudaDeviceSynchronize();
        long long r[2];
        cudaMemcpy(r, out, 16, cudaMemcpyDeviceToHost);
        printf("%s %-11s %2d warps%s: %7.1f cycles per MMA (M128 N256 K32 int8; 129 at peak)  other-warp loops %lld  (%s)\n",
               lean == 3 ? "vec+add   " : lean == 2 ? "vec regs  " : lean ? "lean issue" : "loop issue", names[mode], mode ? nw : 0, skip0 ? " (none on the MMA warp's SMSP)" : "", (double)r[0] / nm, r[1],
               cudaGetErrorString(cudaGetLastError()));
      }
  return 0;
}
