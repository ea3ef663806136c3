// conv_tc.cu — K1-TC: the Flash convolution core on the 5th-gen tensor cores.
//
// Same contraction as conv.cu (conv._proposed_channel conv.py:326-352, closed
// form SURVEY §8a-1), re-expressed as an exact int8 GEMM:
//   out[o][p][s] = Σ_{t,j} w[o][j][t] · E_j[p][s + step_t]          (mod q)
// where E_j is channel j's negacyclic extension ([q-a | a | q-a], conv.py:251)
// aligned so every channel sits at the same slot. Each 60-bit coefficient is
// split into 8 unsigned byte planes, x = Σ_d 256^d x_d, so
//   Σ w·x = Σ_d 256^d P_d,   P_d = Σ w·x_d   (|P_d| ≤ 127·255·K < 2^31 exactly)
// and P_d is one tcgen05.mma.kind::i8 (u8 x s8 -> s32) accumulation.
//
// Layout trick: GEMM row m = (position, plane) with the 8 planes of a position
// as the 8 rows of one UMMA core matrix. A tap's DRot shift then moves the A
// operand by whole core-matrix groups, so one shared-memory window of
// positions [s0-h, s0+S+h) serves all f_w² taps (descriptor start offsets, no
// re-load, no im2col). Operands are pre-arranged in HBM in the canonical
// no-swizzle K-major core-matrix order (8 rows x 16 B), so each pipeline
// stage is two 1-D bulk copies (cp.async.bulk -> mbarrier complete_tx).
//
// CTA = 256 threads: thread 0 issues bulk copies and MMAs (single-thread
// tcgen05 issue), all 8 warps run the epilogue: tcgen05.ld of the s32 plane
// sums (warp w: TMEM lane quadrant w%4, column half w/4), a column-major
// shared-memory transpose, V = lo + 2^32 hi recombination and one canonical
// reduction mod q per coefficient (+ the fused bias of plain_add).
#include "common.cuh"

namespace fhe {
namespace tc {

constexpr int kThreads = 256;
constexpr int kMaxTaps = 64;
constexpr int kEStride = 128 + 8;  // epilogue staging column stride (int32, 16-B aligned)

struct TcArgs {
  const uint8_t* X;   // [2][F][JB][Y][256]  prepared digit planes
  const uint8_t* W;   // [OB][JB][taps][N/8][256] packed int8 weights
  const uint64_t* bias;
  const uint8_t* bmask;
  uint64_t* out;
  ModDesc m;
  uint64_t w32, w32p;  // 2^32 mod q, Shoup companion
  int n, Y, JB, F, c_o, taps, h, stage_bytes, a_bytes;
  int tap_off[kMaxTaps];  // step_t + h
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (uint32_t i = 0; !mbar_try(bar, parity); ++i)
    if (i > (1u << 28)) __trap();  // never hang the GPU on a protocol bug
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :
               : "r"(dst), "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  // K-major, no swizzle: core matrix = 8 rows x 16 B; LBO (K-halves) = 128 B,
  // SBO (8-row groups) = 256 B; version 1 (sm_100).
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}

template <int N>
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  constexpr uint32_t idesc = (2u << 4)              // D: s32
                             | (0u << 7)            // A: u8 (digit planes)
                             | (1u << 10)           // B: s8 (weights)
                             | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      :
      : "r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

#define TMEM_LD32(taddr, v)                                                                                      \
  asm volatile(                                                                                                  \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17," \
      "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                        \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),         \
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),   \
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), \
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])  \
      : "r"(taddr))

// N: output channels per CTA tile; NACC: 16-position M tiles per CTA.
template <int N, int NACC>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int S = 16 * NACC;       // positions per CTA
  constexpr int TM_COLS = N * NACC;  // TMEM columns (power of 2 required)
  static_assert(TM_COLS == 32 || TM_COLS == 64 || TM_COLS == 128 || TM_COLS == 256 || TM_COLS == 512, "tmem");
  static_assert(N % 64 == 0, "epilogue splits N into two halves of 32-column chunks");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int s0 = blockIdx.x * S;
  const int ob = blockIdx.y;
  const int p = blockIdx.z & 1, f = blockIdx.z >> 1;
  const int JB = a.JB, taps = a.taps;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * a.stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);
  const uint32_t full0 = smem_u32(&bars[0]), done0 = smem_u32(&bars[2]), acc_bar = smem_u32(&bars[4]);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 5; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  const size_t plane_stride = (size_t)a.Y * 256;
  const uint8_t* xbase = a.X + ((size_t)(p * a.F + f) * JB) * plane_stride + (size_t)s0 * 256;
  const size_t wstage = (size_t)taps * N * 32;
  const uint8_t* wbase = a.W + (size_t)ob * JB * wstage;
  const uint32_t a_load = (uint32_t)((S + 2 * a.h) * 256);

  if (tid == 0) {
    auto load = [&](int jb) {
      const int st = jb & 1;
      const uint32_t sa = smem_u32(smem + st * a.stage_bytes);
      const uint32_t bar = full0 + 8 * st;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(a_load + (uint32_t)wstage)
                   : "memory");
      bulk_load(sa, xbase + (size_t)jb * plane_stride, a_load, bar);
      bulk_load(sa + a.a_bytes, wbase + (size_t)jb * wstage, (uint32_t)wstage, bar);
    };
    load(0);
    for (int jb = 0; jb < JB; ++jb) {
      if (jb + 1 < JB) {
        if (jb >= 1) mbar_wait(done0 + 8 * ((jb + 1) & 1), ((jb - 1) >> 1) & 1);
        load(jb + 1);
      }
      mbar_wait(full0 + 8 * (jb & 1), (jb >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sa = smem_u32(smem + (jb & 1) * a.stage_bytes);
      const uint32_t sb = sa + a.a_bytes;
      for (int t = 0; t < taps; ++t) {
        const uint64_t bdesc = umma_desc(sb + t * N * 32);
        const uint32_t aoff = (uint32_t)a.tap_off[t] * 256;
#pragma unroll
        for (int mi = 0; mi < NACC; ++mi)
          mma_i8<N>(tmem + mi * N, umma_desc(sa + aoff + mi * 16 * 256), bdesc, (jb | t) != 0);
      }
      mma_commit(done0 + 8 * (jb & 1));
    }
    mma_commit(acc_bar);  // tracks every earlier tcgen05.mma of this CTA
  }
  // single-use barrier: its phase 0 completes exactly when all MMAs are done
  // (waiting on a reused stage barrier could match an older phase's parity)
  mbar_wait(acc_bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");

  // Staging is column-major (stage[col][row], row = position*8 + plane): the
  // TMEM->smem stores are 32 consecutive words per warp and each output's 8
  // planes are two aligned 16-byte loads.
  int32_t* stage = reinterpret_cast<int32_t*>(smem);  // reuse the operand buffers
  const uint64_t q = a.m.q;
  const int quad = warp & 3, half = warp >> 2;
  const int row = quad * 32 + lane;
  constexpr int HALF = N / 2;
  constexpr int PER_THREAD = 16 * N / kThreads;
  for (int mi = 0; mi < NACC; ++mi) {
#pragma unroll
    for (int c0 = half * HALF; c0 < (half + 1) * HALF; c0 += 32) {
      uint32_t v[32];
      TMEM_LD32(tmem + ((uint32_t)(quad * 32) << 16) + mi * N + c0, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int c = 0; c < 32; ++c) stage[(c0 + c) * kEStride + row] = (int32_t)v[c];
    }
    __syncthreads();
    // recombine the 8 planes of each (position, channel) and reduce mod q
#pragma unroll
    for (int k = 0; k < PER_THREAD; ++k) {
      const int idx = tid + k * kThreads;
      const int sp = idx & 15, col = idx >> 4;
      const int o = ob * N + col;
      const int s = s0 + mi * 16 + sp;
      if (o < a.c_o && s < a.n) {
        const int4* e4 = reinterpret_cast<const int4*>(stage + col * kEStride + sp * 8);
        const int4 e0 = e4[0], e1 = e4[1];
        long long lo = (long long)e0.x + ((long long)e0.y << 8) + ((long long)e0.z << 16) + ((long long)e0.w << 24);
        long long hi = (long long)e1.x + ((long long)e1.y << 8) + ((long long)e1.z << 16) + ((long long)e1.w << 24);
        const uint64_t l = reduce_i64(lo, a.m), hh = reduce_i64(hi, a.m);
        uint64_t val = csub(l + csub(shoup_lazy(hh, a.w32, a.w32p, q), q), q);
        if (p == 0 && a.bias) {
          const uint64_t bd = a.bias[o];
          if (bd && a.bmask[(size_t)f * a.n + s]) val = csub(val + bd, q);
        }
        a.out[((size_t)(o * a.F + f) * 2 + p) * a.n + s] = val;
      }
    }
    __syncthreads();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TM_COLS));
}

// ------------------------------------------------------------- relayout
// X[p][f][jb][y][kh][d][16]: digit d of channel j = jb*32 + kh*16 + jj at
// extension slot (n - h + y + shift_j) of source ciphertext src_j + f*fstride.
// chan[j] = (src_j, shift_j) (the channel packing of conv.py:113-130).
// grid: x over (y, kh) pairs, y = jb, z = p*F + f — no runtime divisions.
__global__ void __launch_bounds__(256) prep_kernel(const uint64_t* __restrict__ in, uint8_t* __restrict__ X,
                                                   const int2* __restrict__ chan, int n, int Y, int F, int c_i,
                                                   int h, int fstride, uint64_t q) {
  const int yk = blockIdx.x * blockDim.x + threadIdx.x;
  if (yk >= 2 * Y) return;
  const int y = yk >> 1, kh = yk & 1;
  const int jb = blockIdx.y, JB = gridDim.y;
  const int pf = blockIdx.z, p = pf / F, f = pf - p * F;
  const int ebase = n - h + y;
  uint2 v[16];
#pragma unroll
  for (int jj = 0; jj < 16; ++jj) {
    const int j = jb * 32 + kh * 16 + jj;
    uint64_t x = 0;
    if (j < c_i) {
      const int2 cs = __ldg(&chan[j]);
      int e = ebase + cs.y;  // in [0, 3n)
      const bool lo = e < n, hi = e >= 2 * n;
      e -= lo ? 0 : (hi ? 2 * n : n);
      x = __ldg(&in[((size_t)(cs.x + f * fstride) * 2 + p) * n + e]);
      x = ((lo || hi) && x) ? q - x : x;
    }
    v[jj] = make_uint2((uint32_t)x, (uint32_t)(x >> 32));
  }
  uint4* dst = reinterpret_cast<uint4*>(X + ((((size_t)pf * JB + jb) * Y + y) * 256 + kh * 128));
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const unsigned sel = (unsigned)(d & 3) | ((unsigned)((d & 3) + 4) << 4);
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t a0 = d < 4 ? v[4 * k].x : v[4 * k].y, a1 = d < 4 ? v[4 * k + 1].x : v[4 * k + 1].y;
      const uint32_t a2 = d < 4 ? v[4 * k + 2].x : v[4 * k + 2].y, a3 = d < 4 ? v[4 * k + 3].x : v[4 * k + 3].y;
      const uint32_t t0 = __byte_perm(a0, a1, sel), t1 = __byte_perm(a2, a3, sel);
      w[k] = __byte_perm(t0, t1, 0x5410);
    }
    dst[d] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

template <int N, int NACC>
static int launch(TcArgs& a, const int32_t* tap_steps_host, cudaStream_t st) {
  constexpr int S = 16 * NACC;
  if (a.n % S) return fail(FHE_ERR_VALUE, "n must be a multiple of %d for the tc path", S);
  for (int t = 0; t < a.taps; ++t) {
    const int off = tap_steps_host[t] + a.h;
    if (off < 0 || off > 2 * a.h) return fail(FHE_ERR_VALUE, "tap step outside the halo");
    a.tap_off[t] = off;
  }
  a.a_bytes = ((S + 2 * a.h) * 256 + 1023) / 1024 * 1024;
  a.stage_bytes = a.a_bytes + a.taps * N * 32;
  const size_t epi = (size_t)N * kEStride * 4;
  if ((size_t)2 * a.stage_bytes < epi) a.stage_bytes = (int)((epi + 1) / 2 + 1023) / 1024 * 1024;
  const size_t smem = 2 * (size_t)a.stage_bytes + 64;
  if (smem > 227 * 1024) return fail(FHE_ERR_VALUE, "halo too large for the tc path");
  static bool attr = false;
  if (!attr) {
    FHE_CUDA(cudaFuncSetAttribute(conv_tc_kernel<N, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  dim3 grid(a.n / S, (a.c_o + N - 1) / N, 2 * a.F);
  conv_tc_kernel<N, NACC><<<grid, kThreads, smem, st>>>(a);
  FHE_CHECK_LAUNCH("conv_tc_kernel");
  return FHE_OK;
}

// Largest position tile that still gives >= 1.5 waves of CTAs on 148 SMs.
template <int N, int NACC_BIG, int NACC_SMALL>
static int run_tile(TcArgs& a, const int32_t* tap_steps_host, cudaStream_t st) {
  const long ctas_big = (long)(a.n / (16 * NACC_BIG)) * ((a.c_o + N - 1) / N) * 2 * a.F;
  if (ctas_big >= 222) return launch<N, NACC_BIG>(a, tap_steps_host, st);
  return launch<N, NACC_SMALL>(a, tap_steps_host, st);
}

// Dense int8 tcgen05 roofline probe: back-to-back M=128 N=256 K=32 MMAs on
// resident shared-memory operands (no loads, no epilogue).
__global__ void __launch_bounds__(128, 1) peak_tc_kernel(int iters, uint32_t* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 12288);
  uint32_t* slot = reinterpret_cast<uint32_t*>(smem + 12296);
  for (int i = threadIdx.x; i < 12288 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x01010101u * (i & 3);
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    const uint64_t ad = umma_desc(smem_u32(smem)), bd = umma_desc(smem_u32(smem + 4096));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_i8<256>(tmem + (k & 1) * 256, ad, bd, 1);
    }
    mma_commit(smem_u32(bar));
  }
  mbar_wait(smem_u32(bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x < 32) {
    uint32_t v[32];
    TMEM_LD32(tmem + ((uint32_t)(threadIdx.x & ~31) << 16), v);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (v[0] == 0x5eed) sink[0] = v[1];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace tc
}  // namespace fhe

using namespace fhe;

extern "C" {

int fhe_peak_tc_i8(int blocks, int iters, uint32_t* sink, void* stream) {
  if (blocks < 1 || iters < 1 || !sink) return fail(FHE_ERR_VALUE, "bad peak arguments");
  tc::peak_tc_kernel<<<blocks, 128, 12288 + 64, (cudaStream_t)stream>>>(iters, sink);
  FHE_CHECK_LAUNCH("peak_tc_kernel");
  return FHE_OK;
}

int fhe_conv_tc_prep(uint64_t q, int n, const uint64_t* in, int c_i, int frags, int fstride, const int32_t* chan,
                     int h, uint8_t* X, void* stream) {
  if (n < 64 || (n & (n - 1)) || c_i < 1 || frags < 1 || h < 0 || h >= n || !in || !X || !chan)
    return fail(FHE_ERR_VALUE, "bad tc prep arguments");
  const int JB = (c_i + 31) / 32, Y = n + 2 * h;
  if (JB > 65535 || 2 * frags > 65535) return fail(FHE_ERR_VALUE, "tc prep grid too large");
  dim3 grid((unsigned)((2 * Y + 255) / 256), JB, 2 * frags);
  tc::prep_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(in, X, reinterpret_cast<const int2*>(chan), n, Y, frags,
                                                          c_i, h, fstride, q);
  FHE_CHECK_LAUNCH("tc prep_kernel");
  return FHE_OK;
}

int fhe_conv_tc(uint64_t q, int n, const uint8_t* X, int c_i, int frags, int h, const int8_t* Wpacked, int c_o,
                int taps, int n_tile, const int32_t* tap_steps_host, const uint64_t* bias_delta,
                const uint8_t* bias_mask, uint64_t* out, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (n < 64 || (n & (n - 1)) || c_i < 1 || frags < 1 || c_o < 1 || taps < 1 || taps > tc::kMaxTaps)
    return fail(FHE_ERR_VALUE, "bad tc conv arguments");
  if (!X || !Wpacked || !out || !tap_steps_host) return fail(FHE_ERR_VALUE, "null tc operand");
  if (bias_delta && !bias_mask) return fail(FHE_ERR_VALUE, "bias needs a mask");
  tc::TcArgs a;
  a.X = X;
  a.W = reinterpret_cast<const uint8_t*>(Wpacked);
  a.bias = bias_delta;
  a.bmask = bias_mask;
  a.out = out;
  a.m = ms.m[0];
  a.w32 = (uint64_t)(((u128_t)1 << 32) % q);
  a.w32p = h_shoup(a.w32, q);
  a.n = n;
  a.Y = n + 2 * h;
  a.JB = (c_i + 31) / 32;
  a.F = frags;
  a.c_o = c_o;
  a.taps = taps;
  a.h = h;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_tile == 64) return tc::run_tile<64, 8, 4>(a, tap_steps_host, st);
  if (n_tile == 128) return tc::run_tile<128, 4, 2>(a, tap_steps_host, st);
  return fail(FHE_ERR_VALUE, "n_tile must be 64 or 128");
}

}  // extern "C"
