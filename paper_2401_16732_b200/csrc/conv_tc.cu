// conv_tc.cu — K1-TC: the Flash convolution core on the 5th-gen tensor cores.
//
// Same contraction as conv.cu (conv._proposed_channel conv.py:326-352, closed
// form SURVEY §8a-1), re-expressed as an exact int8 GEMM:
//   out[o][p][s] = Σ_{t,j} w[o][j][t] · E_j[p][s + step_t]          (mod q)
// where E_j is channel j's negacyclic extension ([q-a | a | q-a], conv.py:251)
// shifted so every packed channel sits at the same slot (conv.py:342's
// alignment DRot folded into the indexing). Each 60-bit coefficient is split
// into 8 unsigned byte planes, x = Σ_d 256^d x_d, so
//   Σ w·x = Σ_d 256^d P_d,   P_d = Σ w·x_d   (|P_d| ≤ 127·255·K < 2^31 exactly)
// and P_d is one tcgen05.mma.kind::i8 (s8 x u8 -> s32) accumulation.
//
// GEMM shape: M = 128 output channels (A = packed weights of one tap),
// N = 8·NPOS rows (position, plane) (B = digit-plane window), K = 32 input
// channels per stage. The 8 planes of a position are the 8 rows of one UMMA
// core matrix (K-major, no swizzle: 8 rows x 16 B, LBO = 128 B between the two
// 16-channel K halves, SBO = 256 B between positions), so a tap's DRot shift
// moves the B operand by whole positions: one shared-memory window of
// positions [s0-h, s0+NPOS+h) serves all f_w² taps via descriptor start
// offsets — no im2col. The accumulator puts one output channel per TMEM lane
// and the 8 planes of a position in 8 adjacent columns, so the epilogue
// recombines V = Σ_d 256^d P_d inside each thread (no cross-lane traffic).
//
// Two launches per layer:
//  * prep_kernel: ciphertexts -> digit-plane operand X in that core-matrix
//    order (coalesced loads, a shared-memory byte transpose, 1 KB-contiguous
//    warp stores; X stays L2-resident for the GEMM).
//  * conv_tc_kernel: persistent (one CTA per SM), warp-specialised:
//      warp 0     MMA issue (one thread: tcgen05.mma, tcgen05.commit)
//      warp 1     stage loads (one thread: two cp.async.bulk per stage,
//                 window + packed weights, mbarrier complete_tx)
//      warps 2-9  epilogue: tcgen05.ld of the s32 plane sums, in-thread
//                 recombination and one canonical reduction mod q per
//                 coefficient (+ fused bias), 32-byte row stores.
//    NST-deep stage ring (full/empty mbarriers) and two TMEM accumulator
//    buffers (tmem_full/tmem_empty): the epilogue of tile i overlaps the
//    MMAs of tile i+1.
#include "common.cuh"

namespace fhe {
namespace tc {

constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant
constexpr int kWarps = 2 + kEpiWarps;
constexpr int kThreads = 32 * kWarps;
constexpr int kMaxTaps = 64;
constexpr int kMaxStages = 6;
constexpr int kEpilogue = 32 * kEpiWarps;
constexpr int kOcTile = 128;                  // output channels per tile (MMA M)
constexpr int kWTap = kOcTile * 32;           // packed weight bytes per (tap, 32 channels)

struct TcArgs {
  const uint8_t* X;  // [2][F][JB][Y][256] prepared digit planes
  const uint8_t* W;  // [OB][JB][taps][16][256] packed int8 weights
  const uint64_t* bias;
  const uint8_t* bmask;
  uint64_t* out;
  uint64_t q, w32p;  // modulus; Shoup companion of 2^32 (q > 2^56)
  int n, Y, JB, F, c_o, OB, taps, h, nst, stage_bytes, win_bytes, tiles;
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

// Bounded waits: a protocol bug traps instead of hanging the GPU. Roles that
// are not on the critical path back off so they do not steal issue slots.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  for (uint32_t i = 0; !mbar_try(bar, parity); ++i)
    if (i > (1u << 28)) __trap();
}

__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity, unsigned ns) {
  for (uint32_t i = 0; !mbar_try(bar, parity); ++i) {
    if (i > (1u << 24)) __trap();
    __nanosleep(ns);
  }
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :
               : "r"(dst), "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// K-major, no-swizzle shared-memory matrix descriptor (LBO 128 B, SBO 256 B)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}

// D[128 x N] (+)= A[128 x 32] (s8 weights) · B[N x 32]^T (u8 digit planes)
template <int N>
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  constexpr uint32_t idesc = (2u << 4)              // D: s32
                             | (1u << 7)            // A: s8
                             | (0u << 10)           // B: u8
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

struct Tile {
  int ob, p, f, s0;
};

// Optional timeline instrumentation (fhe_debug_trace): CTA 0 records
// clock64() at pipeline events, [kind][index] with 4096 slots per kind.
__device__ unsigned long long* g_trace = nullptr;
#define TC_TRACE(kind, idx)                                                                     \
  do {                                                                                          \
    if (g_trace && blockIdx.x == 0 && (idx) < 4096) g_trace[(kind) * 4096 + (idx)] = clock64(); \
  } while (0)

// tile t -> (output-channel block fastest, so CTAs running together share the
// same window in L2; then position block, fragment, poly)
template <int NPOS>
__device__ __forceinline__ Tile tile_of(int t, const TcArgs& a) {
  Tile r;
  r.ob = t % a.OB;
  t /= a.OB;
  const int nsb = a.n / NPOS;
  r.s0 = (t % nsb) * NPOS;
  t /= nsb;
  r.f = t % a.F;
  r.p = t / a.F;
  return r;
}

// a value the compiler cannot constant-fold or strength-reduce
__device__ __forceinline__ int opaque(int x) {
  int y;
  asm("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

// a * b + c with a 32x32 -> 64-bit signed product (one IMAD.WIDE)
__device__ __forceinline__ long long mad_wide(int32_t a, int32_t b, long long c) {
  long long d;
  asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
  return d;
}

// NPOS: positions per tile (MMA N = 8·NPOS TMEM columns per accumulator).
template <int NPOS>
__global__ void __launch_bounds__(kThreads, 1) conv_tc_kernel(const TcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int MN = 8 * NPOS;         // MMA N = TMEM columns per accumulator
  constexpr int TM_COLS = 2 * MN;      // double buffered
  static_assert(TM_COLS == 256 || TM_COLS == 512, "tmem");

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NST = a.nst, JB = a.JB, taps = a.taps, n = a.n;

  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * a.stage_bytes);
  // [0,NST) full, [NST,2NST) empty, 2NST+{0,1} tmem_full, 2NST+{2,3} tmem_empty
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages + 4);
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto empty_bar = [&](int s) { return bar0 + 8 * (NST + s); };
  auto tfull_bar = [&](int b) { return bar0 + 8 * (2 * NST + b); };
  auto tempty_bar = [&](int b) { return bar0 + 8 * (2 * NST + 2 + b); };

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < NST; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_bar(s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty_bar(s)));
    }
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tfull_bar(b)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tempty_bar(b)), "r"(kEpilogue));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t wstage = (uint32_t)taps * kWTap;
  const size_t plane_stride = (size_t)a.Y * 256;
  const uint32_t win_load = (uint32_t)((NPOS + 2 * a.h) * 256);

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issue
    if (lane == 0) {
      int it = 0, tl = 0;
      for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++tl) {
        const int buf = tl & 1;
        mbar_wait(tempty_bar(buf), ((tl >> 1) & 1) ^ 1);  // epilogue released this buffer
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + buf * MN;
        for (int jb = 0; jb < JB; ++jb, ++it) {
          const int s = it % NST;
          mbar_wait(full_bar(s), (it / NST) & 1);
          TC_TRACE(0, it);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sx = smem_u32(smem + s * a.stage_bytes);
          const uint32_t sw = sx + a.win_bytes;
          for (int tp = 0; tp < taps; ++tp)
            mma_i8<MN>(acc, umma_desc(sw + tp * kWTap), umma_desc(sx + (uint32_t)a.tap_off[tp] * 256),
                       (jb | tp) != 0);
          mma_commit(empty_bar(s));  // stage free once these MMAs retire
          TC_TRACE(1, it);
        }
        mma_commit(tfull_bar(buf));  // accumulator complete
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ stage loads
    if (lane == 0) {
      int it = 0;
      for (int t = blockIdx.x; t < a.tiles; t += gridDim.x) {
        const Tile T = tile_of<NPOS>(t, a);
        const uint8_t* xbase = a.X + ((size_t)(T.p * a.F + T.f) * JB) * plane_stride + (size_t)T.s0 * 256;
        const uint8_t* wbase = a.W + (size_t)T.ob * JB * wstage;
        for (int jb = 0; jb < JB; ++jb, ++it) {
          const int s = it % NST;
          mbar_wait_sleep(empty_bar(s), ((it / NST) & 1) ^ 1, 32);
          const uint32_t sx = smem_u32(smem + s * a.stage_bytes);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full_bar(s)),
                       "r"(win_load + wstage)
                       : "memory");
          TC_TRACE(4, it);
          bulk_load(sx, xbase + (size_t)jb * plane_stride, win_load, full_bar(s));
          bulk_load(sx + a.win_bytes, wbase + (size_t)jb * wstage, wstage, full_bar(s));
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    // lane = output channel within the quadrant; a 32-column TMEM chunk holds
    // 4 positions x 8 planes. lo = q + Σ_{d<4} 2^(8d) P_d and hi = q + Σ_{d>=4}
    // 2^(8(d-4)) P_d lie in (0, 2q) (|P_d| < 2^31, q > 2^56); V = lo + 2^32 hi.
    const int quad = warp & 3;        // TMEM lane quadrant (hardware: warp id % 4)
    const int sub = (warp - 2) >> 2;  // which warp of the quadrant
    const uint64_t q = a.q;
    const int k8 = opaque(1 << 8), k16 = opaque(1 << 16), k24 = opaque(1 << 24);
    int tl = 0;
    for (int t = blockIdx.x; t < a.tiles; t += gridDim.x, ++tl) {
      const Tile T = tile_of<NPOS>(t, a);
      const int buf = tl & 1;
      const int o = T.ob * kOcTile + quad * 32 + lane;
      const bool active = T.ob * kOcTile + quad * 32 < a.c_o;  // warp-uniform
      mbar_wait_sleep(tfull_bar(buf), (tl >> 1) & 1, 64);
      if (lane == 0 && warp == 2) TC_TRACE(5, tl);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (active) {
        const uint64_t bd = (T.p == 0 && a.bias && o < a.c_o) ? a.bias[o] : 0;
        const uint32_t acc = tmem + buf * MN + ((uint32_t)(quad * 32) << 16);
        uint64_t* orow = a.out + ((size_t)(o * a.F + T.f) * 2 + T.p) * n + T.s0;
#pragma unroll 1
        for (int k = sub; k < NPOS / 4; k += kEpiWarps / 4) {
          uint32_t v[32];
          TMEM_LD32(acc + k * 32, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          uint64_t r[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int32_t* P = reinterpret_cast<const int32_t*>(v + 8 * j);
            const long long lo =
                mad_wide(P[3], k24, mad_wide(P[2], k16, mad_wide(P[1], k8, (long long)q + P[0])));
            const long long hi =
                mad_wide(P[7], k24, mad_wide(P[6], k16, mad_wide(P[5], k8, (long long)q + P[4])));
            // 2^32 hi mod q by Shoup (w = 2^32 < q): result in [0, 2q)
            const uint64_t uh = ((uint64_t)hi << 32) - __umul64hi(a.w32p, (uint64_t)hi) * q;
            uint64_t val = (uint64_t)lo + uh;  // < 4q
            val = val >= 2 * q ? val - 2 * q : val;
            r[j] = val >= q ? val - q : val;
          }
          if (bd) {
            const uint32_t mk = *reinterpret_cast<const uint32_t*>(a.bmask + (size_t)T.f * n + T.s0 + 4 * k);
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if ((mk >> (8 * j)) & 0xff) r[j] = csub(r[j] + bd, q);
          }
          if (o < a.c_o) {
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(orow + 4 * k);
            dst[0] = make_ulonglong2(r[0], r[1]);
            dst[1] = make_ulonglong2(r[2], r[3]);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      mbar_arrive(tempty_bar(buf));
      if (lane == 0 && warp == 2) TC_TRACE(6, tl);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TM_COLS));
}

// ------------------------------------------------------------- relayout
// X[p][f][jb][y][kh][d][16]: digit d of channel j = jb*32 + kh*16 + jj at
// extension slot (n - h + y + shift_j) of source ciphertext src_j + f*fstride.
// A CTA (128 threads) converts kPrepY window positions x 32 channels in three
// phases (many small CTAs per SM hide the load latency):
//  1. coalesced 8-byte loads (lane = position, warp = 8 channels) into a
//     shared [position][channel] tile, negacyclic sign applied on the fly;
//  2. thread (position, K half, low/high word) byte-transposes 16 coefficients
//     into 4 plane words x 4 (4x4 PRMT transposes) and stages 64 B in shared
//     memory (16-byte chunks XOR-swizzled by position: conflict-free);
//  3. the CTA streams the staged 8 KB to X with fully coalesced 16 B stores.
constexpr int kPrepY = 32;
constexpr int kPrepThreads = 128;

__device__ __forceinline__ void transpose4x4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t& p0,
                                             uint32_t& p1, uint32_t& p2, uint32_t& p3) {
  const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a0, a1, 0x7362);
  const uint32_t t2 = __byte_perm(a2, a3, 0x5140), t3 = __byte_perm(a2, a3, 0x7362);
  p0 = __byte_perm(t0, t2, 0x5410);
  p1 = __byte_perm(t0, t2, 0x7632);
  p2 = __byte_perm(t1, t3, 0x5410);
  p3 = __byte_perm(t1, t3, 0x7632);
}

__global__ void __launch_bounds__(kPrepThreads) prep_kernel(const uint64_t* __restrict__ in,
                                                            uint8_t* __restrict__ X, const int2* __restrict__ chan,
                                                            int n, int Y, int F, int c_i, int h, int fstride,
                                                            uint64_t q) {
  __shared__ __align__(16) uint64_t raw[kPrepY][33];  // [position][channel] (+1 pad); reused for staging
  const int y0 = blockIdx.x * kPrepY, jb = blockIdx.y, JB = gridDim.y;
  const int pf = blockIdx.z, p = pf / F, f = pf - p * F;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // 1. load: warp w handles channels 8w..8w+7
  const int y = y0 + lane;
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
    const int jl = warp * 8 + cc, j = jb * 32 + jl;
    uint64_t x = 0;
    if (j < c_i && y < Y) {
      const int2 cs = __ldg(&chan[j]);
      int e = n - h + y + cs.y;  // in [0, 3n)
      const bool lo = e < n, hi = e >= 2 * n;
      e -= lo ? 0 : (hi ? 2 * n : n);
      x = __ldg(&in[((size_t)(cs.x + f * fstride) * 2 + p) * n + e]);
      x = ((lo || hi) && x) ? q - x : x;
    }
    raw[lane][jl] = x;
  }
  __syncthreads();
  // 2. pack: thread -> (position yl, K half kh, word half wh): planes 4wh..4wh+3
  const int yl = threadIdx.x >> 2, kh = (threadIdx.x >> 1) & 1, wh = threadIdx.x & 1;
  uint32_t w[4][4];
#pragma unroll
  for (int g4 = 0; g4 < 4; ++g4) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(&raw[yl][kh * 16 + g4 * 4]) + wh;
    transpose4x4(r[0], r[2], r[4], r[6], w[0][g4], w[1][g4], w[2][g4], w[3][g4]);
  }
  __syncthreads();
  uint4* stage = reinterpret_cast<uint4*>(&raw[0][0]);  // [position][16 chunks of 16 B], chunk ^= yl & 7
#pragma unroll
  for (int dd = 0; dd < 4; ++dd)
    stage[yl * 16 + kh * 8 + ((4 * wh + dd) ^ (yl & 7))] = make_uint4(w[dd][0], w[dd][1], w[dd][2], w[dd][3]);
  __syncthreads();
  // 3. coalesced copy-out of the CTA's contiguous [kPrepY][256 B] slab
  const int rows = min(kPrepY, Y - y0);
  uint4* dst = reinterpret_cast<uint4*>(X + (((size_t)pf * JB + jb) * Y + y0) * 256);
#pragma unroll
  for (int i = 0; i < kPrepY * 16 / kPrepThreads; ++i) {
    const int idx = threadIdx.x + kPrepThreads * i, pos = idx >> 4, ch = idx & 15;
    if (pos < rows) dst[idx] = stage[pos * 16 + (ch & 8) + ((ch & 7) ^ (pos & 7))];
  }
}

template <int NPOS>
static int launch(TcArgs& a, const int32_t* tap_steps_host, cudaStream_t st) {
  if (a.n % NPOS) return fail(FHE_ERR_VALUE, "n must be a multiple of %d for the tc path", NPOS);
  for (int t = 0; t < a.taps; ++t) {
    const int off = tap_steps_host[t] + a.h;
    if (off < 0 || off > 2 * a.h) return fail(FHE_ERR_VALUE, "tap step outside the halo");
    a.tap_off[t] = off;
  }
  a.win_bytes = ((NPOS + 2 * a.h) * 256 + 1023) / 1024 * 1024;
  a.stage_bytes = a.win_bytes + a.taps * kWTap;
  a.nst = (214 * 1024) / a.stage_bytes;
  if (a.nst > kMaxStages) a.nst = kMaxStages;
  if (a.nst < 2) return fail(FHE_ERR_VALUE, "halo too large for the tc path");
  const size_t smem = (size_t)a.nst * a.stage_bytes + 8 * (2 * kMaxStages + 4) + 16;
  a.tiles = (a.n / NPOS) * a.OB * 2 * a.F;
  static bool attr = false;
  if (!attr) {
    FHE_CUDA(cudaFuncSetAttribute(conv_tc_kernel<NPOS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    FHE_CUDA(cudaGetDevice(&dev));
    FHE_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const int grid = a.tiles < sms ? a.tiles : sms;
  conv_tc_kernel<NPOS><<<grid, kThreads, smem, st>>>(a);
  FHE_CHECK_LAUNCH("conv_tc_kernel");
  return FHE_OK;
}

// Dense int8 tcgen05 roofline probe: back-to-back M=128 N K=32 MMAs on
// resident shared-memory operands (no loads, no epilogue).
template <int N>
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
      for (int k = 0; k < 8; ++k) mma_i8<N>(tmem + (k & 1) * 256, ad, bd, 1);
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

int fhe_debug_trace(void* dev_buf) {
  unsigned long long* p = (unsigned long long*)dev_buf;
  FHE_CUDA(cudaMemcpyToSymbol(tc::g_trace, &p, sizeof(p)));
  return FHE_OK;
}

int fhe_peak_tc_i8(int blocks, int n_tile, int iters, uint32_t* sink, void* stream) {
  if (blocks < 1 || iters < 1 || !sink) return fail(FHE_ERR_VALUE, "bad peak arguments");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_tile == 64)
    tc::peak_tc_kernel<64><<<blocks, 128, 12288 + 64, st>>>(iters, sink);
  else if (n_tile == 128)
    tc::peak_tc_kernel<128><<<blocks, 128, 12288 + 64, st>>>(iters, sink);
  else if (n_tile == 256)
    tc::peak_tc_kernel<256><<<blocks, 128, 12288 + 64, st>>>(iters, sink);
  else
    return fail(FHE_ERR_VALUE, "n_tile must be 64, 128 or 256");
  FHE_CHECK_LAUNCH("peak_tc_kernel");
  return FHE_OK;
}

int fhe_conv_tc_prep(uint64_t q, int n, const uint64_t* in, int c_i, int frags, int fstride, const int32_t* chan,
                     int h, uint8_t* X, void* stream) {
  if (n < 64 || (n & (n - 1)) || c_i < 1 || frags < 1 || h < 0 || h >= n || !in || !X || !chan)
    return fail(FHE_ERR_VALUE, "bad tc prep arguments");
  const int JB = (c_i + 31) / 32, Y = n + 2 * h;
  if (JB > 65535 || 2 * frags > 65535) return fail(FHE_ERR_VALUE, "tc prep grid too large");
  dim3 grid((unsigned)((Y + tc::kPrepY - 1) / tc::kPrepY), JB, 2 * frags);
  tc::prep_kernel<<<grid, tc::kPrepThreads, 0, (cudaStream_t)stream>>>(in, X, reinterpret_cast<const int2*>(chan), n, Y, frags,
                                                          c_i, h, fstride, q);
  FHE_CHECK_LAUNCH("tc prep_kernel");
  return FHE_OK;
}

int fhe_conv_tc(uint64_t q, int n, const uint8_t* X, int c_i, int frags, int h, const int8_t* Wpacked, int c_o,
                int taps, int pos_tile, const int32_t* tap_steps_host, const uint64_t* bias_delta,
                const uint8_t* bias_mask, uint64_t* out, void* stream) {
  if (q < (1ull << 56) || q >= (1ull << 62)) return fail(FHE_ERR_VALUE, "tc path needs 2^56 <= q < 2^62");
  if (n < 64 || (n & (n - 1)) || c_i < 1 || frags < 1 || c_o < 1 || taps < 1 || taps > tc::kMaxTaps || h < 0 ||
      h >= n)
    return fail(FHE_ERR_VALUE, "bad tc conv arguments");
  if (!X || !Wpacked || !out || !tap_steps_host) return fail(FHE_ERR_VALUE, "null tc operand");
  if (bias_delta && !bias_mask) return fail(FHE_ERR_VALUE, "bias needs a mask");
  if (127ll * 255 * ((c_i + 31) / 32 * 32) * taps >= (1ll << 31))
    return fail(FHE_ERR_VALUE, "tc path: plane sums would exceed s32");
  tc::TcArgs a;
  a.X = X;
  a.W = reinterpret_cast<const uint8_t*>(Wpacked);
  a.bias = bias_delta;
  a.bmask = bias_mask;
  a.out = out;
  a.q = q;
  a.w32p = h_shoup(1ull << 32, q);
  a.n = n;
  a.Y = n + 2 * h;
  a.JB = (c_i + 31) / 32;
  a.F = frags;
  a.c_o = c_o;
  a.OB = (c_o + tc::kOcTile - 1) / tc::kOcTile;
  a.taps = taps;
  a.h = h;
  cudaStream_t st = (cudaStream_t)stream;
  if (pos_tile == 16) return tc::launch<16>(a, tap_steps_host, st);
  if (pos_tile == 32) return tc::launch<32>(a, tap_steps_host, st);
  return fail(FHE_ERR_VALUE, "pos_tile must be 16 or 32");
}

}  // extern "C"
