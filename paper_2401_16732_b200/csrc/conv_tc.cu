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
// N = 8·npos rows (position, plane) (B = digit-plane window), K = 32 input
// channels per stage. The 8 planes of a position are the 8 rows of one UMMA
// core matrix (K-major, no swizzle: 8 rows x 16 B, LBO = 128 B between the two
// 16-channel K halves, SBO = 256 B between positions), so a tap's DRot shift
// moves the B operand by whole positions: one shared-memory window of
// positions [s0-h, s0+npos+h) serves all f_w² taps via descriptor start
// offsets — no im2col. The accumulator puts one output channel per TMEM lane
// and the 8 planes of a position in 8 adjacent columns, so the epilogue
// recombines V = Σ_d 256^d P_d inside each thread (no cross-lane traffic).
// Layers with c_o <= 64 fill the 128 rows with two position groups: stacked
// (LayerDesc.rep: block-diagonal weights, the same MMA count, every TMEM
// quadrant busy in the epilogue) or, when taps can merge, INTERLEAVED
// (LayerDesc.ilv: row 2o + r = channel o at positions 2u + r; taps of the two
// groups with the same window offset share one full-height MMA).
//
// Code size matters here: the five roles' hot loops share the SM's 32 KB L1.5
// instruction cache, and code added to one of them has cost 1-4 % of the whole
// step even when it never ran (profiles/r02e_icache_ab.txt). Keep the role
// loops lean; instrumentation inside them is opt-in (FHE_TC_TRACE).
//
// One cooperative persistent launch (one CTA per SM) runs a whole STACK of
// independent conv layers (one layer for conv_proposed; a network's layers or
// many requests for the serving path):
//  relayout  warps 10-13 (and, for layer 0, the epilogue warps) stream through
//            the layers in order, each taking (32 positions x 16 channels)
//            units round-robin and writing that layer's own digit-plane
//            region of X; the CTA's last warp publishes one per-layer count
//            (release fences: generic -> async proxy, then gpu scope);
//  GEMM      per layer, once its X count reaches the grid size:
//             warp 1     the loader: grabs the CTA's tiles from a per-layer
//                        counter (dynamic scheduling; the launch's last grab
//                        resets it), publishes the tile sequence in a
//                        shared-memory ring, and fills the stage ring with
//                        cp.async.bulk (window + weights, or the window only
//                        when the layer's weights are resident);
//             warp 0     MMA issue (elect.sync: tcgen05.mma kind::i8, commits);
//             warps 2-9  epilogue: tcgen05.ld, in-thread recombination of the
//                        eight byte planes, one canonical reduction mod q
//                        (pseudo-Mersenne or Shoup; + fused bias), row stores;
//            two TMEM accumulator buffers (a 64-position tile uses both).
// Roles move on to the next layer as soon as their part of this one is done:
// relayout runs ahead of the GEMM and no per-layer launch gap remains.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace fhe {
namespace tc {

#ifndef FHE_EPI_WARPS
#define FHE_EPI_WARPS 8
#endif
constexpr int kEpiWarps = FHE_EPI_WARPS;  // two (or four) per TMEM lane quadrant
#ifndef FHE_REL_SKIP0
#define FHE_REL_SKIP0 0  // 1 measured ~1 % slower on config 5 (one relayout warp fewer per other sub-partition)
#endif
#ifndef FHE_REL_WARPS
#define FHE_REL_WARPS (4 + FHE_REL_SKIP0)
#endif
constexpr int kRelWarps = FHE_REL_WARPS;  // dedicated relayout warps (run ahead of the GEMM)
constexpr int kWarps = 2 + kEpiWarps + kRelWarps;
// The MMA issuer (warp 0) shares sub-partition 0 with warps 4k. Integer-heavy
// warps there delay its per-MMA descriptor moves enough to starve the tensor
// pipe (tools/mma_contention.cu; config-5 stem MMAs ran at ~2.3x their issue
// time with every quadrant's epilogue busy). With FHE_REL_SKIP0 the relayout
// warps on sub-partition 0 help with layer 0 only; the others stream the rest.
__host__ __device__ constexpr bool rel_late(int w) { return !(FHE_REL_SKIP0 && (w & 3) == 0); }
__host__ __device__ constexpr int rel_late_rank(int w) {  // rank of relayout warp w among the late ones
  int r = 0;
  for (int v = 2 + kEpiWarps; v < w; ++v) r += rel_late(v) ? 1 : 0;
  return r;
}
constexpr int kRelLate = rel_late_rank(kWarps);  // relayout warps of layers 1..
constexpr int kThreads = 32 * kWarps;
constexpr int kMaxTaps = 64;
constexpr int kMaxStages = 6;
constexpr int kMaxLayers = 24;
constexpr int kEpilogue = 32 * kEpiWarps;
constexpr int kOcTile = 128;         // output channels per tile (MMA M)
constexpr int kWTap = kOcTile * 32;  // packed weight bytes per (tap, 32 channels)
constexpr int kStg = 2048;           // relayout staging bytes per warp (16 positions x 128 B)
// stage ring: what 227 KB leaves after the relayout staging (kRelWarps x 2 KB) and the
// barriers — 4 stages of the 16x16-map layers (54 KB each) fit, 3 did at 212 KB
constexpr int kRingBudget = 227 * 1024 - kRelWarps * kStg - 1024;
constexpr int kSlotWords = 4 + kMaxLayers;  // tmem, epoch, (pad), per-layer relayout-done counts of this CTA
constexpr int kAccCols = 256;        // TMEM columns per accumulator buffer (npos <= 32)
#ifndef FHE_RELAYOUT_STATIC
#define FHE_RELAYOUT_STATIC 1
#endif
#ifndef FHE_GEM_ALWAYS
#define FHE_GEM_ALWAYS 0  // 1: the per-layer GEMM-done barrier + count in every mode (A/B probe)
#endif
#ifndef FHE_REL_TWO
#define FHE_REL_TWO 0  // static relayout: 1 = two units in flight per warp. 0 (one unit: half the relayout
                       // code in the roles' shared 32 KB instruction cache) measured 2.6 % faster on config 5
#endif
#ifndef FHE_UNITS_PER_GRAB
#define FHE_UNITS_PER_GRAB 1
#endif
constexpr int kUnitsPerGrab = FHE_UNITS_PER_GRAB;  // relayout units taken per work-counter grab
#ifndef FHE_PF_AHEAD
#define FHE_PF_AHEAD 2
#endif
constexpr int kPfAhead = FHE_PF_AHEAD;
#ifndef FHE_XFENCE
#define FHE_XFENCE 1  // relayout writers order their X stores into the async proxy (0: A/B probe only)
#endif  // relayout inputs are prefetched into L2 this many layers ahead
#ifndef FHE_EPI_PIPE
#define FHE_EPI_PIPE 0  // 1: software-pipelined TMEM loads in the pair epilogue (measured 2.5 % slower on config 5)
#endif
#ifndef FHE_ILV_EPI
#define FHE_ILV_EPI 1  // 0: A/B probe of the interleaved-group epilogue code's cost (interleaved layers then wrong)
#endif
#ifndef FHE_ILV_FAST
#define FHE_ILV_FAST 1  // unrolled MMA issue paths for 8 and 12 merged taps
#endif
#ifndef FHE_EPI_SLEEP
#define FHE_EPI_SLEEP 0
#endif
#ifndef FHE_EPI_PAIR
#define FHE_EPI_PAIR 0  // 1: two TMEM chunk loads per tcgen05.wait::ld (measured 3 % slower on configs 4 and 5)
#endif

struct LayerDesc {
  const uint64_t* in;  // input ciphertext rows [n_in][2][n]
  const int2* chan;    // [c_i] (source ciphertext, slot shift) of each channel
  uint8_t* X;          // [2][F][JB][Y][256] digit planes (written by phase 1)
  const uint8_t* W;    // [OB][JB][taps][16][256] packed int8 weights
  const uint64_t* bias;
  const uint8_t* bmask;
  uint64_t* out;
  size_t in_bytes, w_bytes;  // extents of the input and weights (L2 prefetch, FHE_CHECKS)
  size_t x_bytes, out_bytes;  // extents of this layer's X region and output (FHE_CHECKS)
  int Y, JB, F, c_i, fstride, c_o, OB, taps, h, npos, nst, stage_bytes, win_bytes, tiles, units;
  int toff;  // tiles of the previous layers mod gridDim.x: tiles are dealt round-robin over the whole stack
  int nacc;  // accumulators per tile: 1, or 2 (a 64-position tile: weights reused by both, TMEM single-buffered)
  int tpos;  // positions per tile = npos * nacc, or npos * rep
  int slot_bytes, nslots;  // ring partition this layer runs in: nslots slots of slot_bytes >= stage_bytes
  int res_bytes;           // > 0: the layer's weights (one output block) stay resident at the ring base and
                           // a stage is just the window (slots follow the weights); loaded once per CTA
  int rep;   // 32-position groups stacked in the 128 accumulator rows (c_o <= 128 / rep): 1, 2 or 4
  int pair;  // 1: plane sums are below 2^31 / 257 (short contraction): the epilogue pairs planes in 32 bits
  int ilv;   // 1 (rep == 2): the two position groups interleave — accumulator row 2 o + r computes channel o at
             // positions s0 + 2 u + r, so the taps of both groups that read the same window offset share ONE
             // full-height MMA (7 column taps -> 8 MMAs per 64 positions instead of 14 half-empty ones; 3x3 ->
             // 12 instead of 18). X is stored de-interleaved per plane ([even positions | odd positions], Y/2
             // each) and a window is two bulk copies, so column u of a tap is a plain contiguous read:
             // tap_off = (e & 1)(32 + h) + (e >> 1) for window offset e — the MMA issue loop sees an
             // ordinary layer
  int16_t tap_off[kMaxTaps];  // step_t + h
};

constexpr int kRdy = 3 + kMaxLayers;      // sync index of layer 0's relayout-done counter
constexpr int kGem = 3 + 2 * kMaxLayers;  // sync index of layer 0's GEMM-done counter
constexpr int kTile = 3 + 3 * kMaxLayers; // sync index of layer 0's tile counter (dynamic tile scheduling)
constexpr int kSyncWords = 3 + 4 * kMaxLayers;  // counter words of a sync buffer (conv.SYNC_WORDS)
static_assert(kTile + kMaxLayers == kSyncWords, "sync layout");
constexpr int kTq = 32;                   // tile-sequence ring entries (loader -> MMA issuer, epilogue)

// ML = layers the parameter block holds: kMaxLayers for stacks, 1 for the
// one-layer launches of the drop-in path (an 8 KB parameter block copied at
// every launch would cost that path microseconds of launch overhead)
template <int ML>
struct StackArgsT {
  LayerDesc L[ML];
  unsigned long long* sync;  // 3 + 3 * kMaxLayers counters (see the protocol note below)
  uint64_t q, w32p;          // modulus; Shoup companion of 2^32 (q > 2^56)
  int n, nl;
  int k1, k8, k16, k24;      // 1, 2^8, 2^16, 2^24 as launch values: ptxas cannot strength-reduce the epilogue's
                             // plane recombination into shift / sign / carry sequences (one IMAD.WIDE each)
  int xrot;                  // 1: three X buffers rotate (layer l reuses l-3's); 0: every layer has its own
  int dyn;                   // 1: CTAs grab tiles from per-layer counters (dynamic); 0: static round-robin
  // pseudo-Mersenne epilogue (pm = 1 when q = 2^60 - delta with delta < 2^35, the reference's
  // default modulus): 2^60 = delta (mod q) folds the 2^32-shifted half in two multiply-adds
  // instead of a 64x64 Shoup product (see finish_pm)
  int pm;
  uint32_t pm_dlo, pm_dhi;   // delta = pm_dhi * 2^32 + pm_dlo
  uint64_t pm_ca;            // = -2^88 (mod q), >= 2^56: the low half's offset (the high half's is 2^56)
};
using StackArgs = StackArgsT<kMaxLayers>;

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

// instruction descriptor: D s32, A s8 (weights), B u8 (digit planes), M = 128
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// D[128 x N] (+)= A[128 x 32] (s8 weights) · B[N x 32]^T (u8 digit planes)
__device__ __forceinline__ void mma_i8(uint32_t tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}"
      :
      : "r"(tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// D[128 x N] (+)= A · B^T with the descriptors given as (low, high) words:
// the high word (SBO, layout bits) is the same for every operand here.
__device__ __forceinline__ void mma_i8w(uint32_t tmem, uint32_t alo, uint32_t blo, uint32_t dhi, uint32_t idesc,
                                        uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "mov.b64 da, {%1, %3};\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %4, p;\n\t}"
      :
      : "r"(tmem), "r"(alo), "r"(blo), "r"(dhi), "r"(idesc), "r"(accum));
}

// Warp-wide forms: every lane of the MMA warp runs the issue loop (uniform
// control flow, so loop state can live in uniform registers) and elect.sync
// picks the one lane that issues.
__device__ __forceinline__ void mma_i8w_elect(uint32_t tmem, uint32_t alo, uint32_t blo, uint32_t dhi,
                                              uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 da, db;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "mov.b64 da, {%1, %3};\n\t"
      "mov.b64 db, {%2, %3};\n\t"
      "setp.ne.b32 p, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], da, db, %4, p;\n\t}"
      :
      : "r"(tmem), "r"(alo), "r"(blo), "r"(dhi), "r"(idesc), "r"(accum));
}

__device__ __forceinline__ void mma_commit_elect(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(bar)
      : "memory");
}

// The 9 (or 1) MMAs of one accumulator for one stage. Descriptors advance by
// adding 16-byte units to the start-address field of the low word (addresses
// stay below 256 KB, so the 14-bit field never carries): weights by 256 units
// per tap, the window by the tap's DRot offset. `before_last` runs between the
// last two MMAs (while the tensor pipe still holds queued work): the issuer
// uses it to wait for the NEXT stage there, so the gap between stages stays
// under the ~100 cycles the pipe tolerates (tools/ring_probe.cu).
template <int TAPS, class F>
__device__ __forceinline__ void issue_taps(uint32_t acc, uint32_t alo, uint32_t blo, uint32_t dhi,
                                           const uint32_t* off16, uint32_t idesc, bool first, F&& before_last) {
#pragma unroll
  for (int tp = 0; tp < TAPS; ++tp) {
    if (tp == TAPS - 1) before_last();
    mma_i8w_elect(acc, alo + (uint32_t)(tp * (4096 >> 4)), blo + off16[tp], dhi, idesc, (first && tp == 0) ? 0u : 1u);
  }
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

// tcgen05.wait::ld that also "rewrites" the 32 destination registers of the
// outstanding load: arithmetic on them cannot be scheduled above the wait
// (the software-pipelined epilogue computes on one chunk while the next loads)
#define TMEM_WAIT32(v)                                                                                            \
  asm volatile("tcgen05.wait::ld.sync.aligned;"                                                                   \
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7]),  \
                 "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]), "+r"(v[12]), "+r"(v[13]), "+r"(v[14]),         \
                 "+r"(v[15]), "+r"(v[16]), "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),       \
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]), "+r"(v[27]), "+r"(v[28]),       \
                 "+r"(v[29]), "+r"(v[30]), "+r"(v[31])                                                            \
               :                                                                                                  \
               : "memory")

// Optional timeline instrumentation (fhe_debug_trace): CTA 0 records
// clock64() at pipeline events, [kind][index] with 4096 slots per kind.
__device__ unsigned long long* g_trace = nullptr;
// (kernels copy g_trace into a local `trc` once: no global load per event)
// The per-event points inside the role loops are compiled in only with -DFHE_TC_TRACE=1
// (tools/build_probe.py trace -DFHE_TC_TRACE=1): the roles' hot code shares a 32 KB
// instruction cache and every event point in a loop costs measurable time. The per-CTA
// start / end stamps (bench.py's kernel clock) are always there.
#ifndef FHE_TC_TRACE
#define FHE_TC_TRACE 0
#endif
#if FHE_TC_TRACE
#define TC_TRACE(kind, idx)                                                             \
  do {                                                                                  \
    if (trc && blockIdx.x == 0 && (idx) < 4096) trc[(kind) * 4096 + (idx)] = clock64(); \
  } while (0)
#else
#define TC_TRACE(kind, idx) \
  do {                      \
  } while (0)
#endif

struct Tile {
  int ob, p, f, s0;
};

// tile t -> (output-channel block fastest, so CTAs running together share the
// same window in L2; then position block, fragment, poly)
__device__ __forceinline__ Tile tile_of(int t, const LayerDesc& d, int n) {
  Tile r;
  r.ob = t % d.OB;
  t /= d.OB;
  const int nsb = n / d.tpos;
  r.s0 = (t % nsb) * d.tpos;
  t /= nsb;
  r.f = t % d.F;
  r.p = t / d.F;
  return r;
}

// first tile of layer d for this CTA (continuing the stack-wide round-robin)
__device__ __forceinline__ int first_tile(const LayerDesc& d) {
  const int G = gridDim.x;
  return ((int)blockIdx.x - d.toff + G) % G;
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

// V = Σ_d 2^(8d) P_d mod q for q = 2^60 - delta, delta < 2^35 (|P_d| < 2^31):
//   A = ca + Σ_{d<4} 2^(8d) P_d   in (2^54, 2^60.2)     (ca in [2^56, 2^56 + q), ca = -2^88 mod q)
//   B = 2^56 + Σ_{d>=4} 2^(8(d-4)) P_d in (2^55, 2^56.6)
//   A + 2^32 B = V + ca + 2^88 = V (mod q);  B = bh 2^28 + bl, 2^60 = delta:
//   W = A + bl 2^32 + delta bh      < 2^60.2 + 2^60 + 2^63.6 < 2^64
//   W = wh 2^60 + wl:  U = wl + delta wh < 2^60 + 2^39 < 2q;  r = U mod q (one subtraction)
// 30 integer instructions per coefficient instead of ~50 (Shoup on the high half).
// (A, B) -> A + 2^32 B mod q, the pseudo-Mersenne folds
__device__ __forceinline__ uint64_t reduce_pm(long long a, long long b, uint32_t dlo, uint32_t dhi, uint64_t q) {
  const uint32_t blo = (uint32_t)b, bhi = (uint32_t)((unsigned long long)b >> 32);
  const uint32_t bh = __funnelshift_r(blo, bhi, 28), bl = blo & 0x0FFFFFFFu;
  uint64_t w = (uint64_t)bh * dlo + (uint64_t)a;  // IMAD.WIDE.U32 with a 64-bit addend
  uint32_t wlo = (uint32_t)w, whi = (uint32_t)(w >> 32) + (bh * dhi + bl);
  const uint32_t wh = whi >> 28;
  whi &= 0x0FFFFFFFu;
  uint64_t u = (uint64_t)wh * dlo + (((uint64_t)whi << 32) | wlo);
  u += (uint64_t)(wh * dhi) << 32;
  return u >= q ? u - q : u;
}

__device__ __forceinline__ uint64_t finish_pm(const int32_t* P, int k1, int k8, int k16, int k24, uint64_t ca,
                                              uint32_t dlo, uint32_t dhi, uint64_t q) {
  const long long a = mad_wide(P[3], k24, mad_wide(P[2], k16, mad_wide(P[1], k8, mad_wide(P[0], k1, (long long)ca))));
  const long long b =
      mad_wide(P[7], k24, mad_wide(P[6], k16, mad_wide(P[5], k8, mad_wide(P[4], k1, 1ll << 56))));
  return reduce_pm(a, b, dlo, dhi, q);
}

// Short contractions (LayerDesc.pair: 127·255·257·K < 2^31 for the K = c_i·taps
// products summed into one accumulator row — the stems and the 1x1 projections):
// byte-plane pairs P_2i + 2^8 P_2i+1 are exact in 32 bits, so each half is two
// 32-bit multiply-adds and two wide ones instead of four wide ones and their adds.
__device__ __forceinline__ uint64_t finish_pm_pair(const int32_t* P, int k1, int k8, int k16, uint64_t ca,
                                                   uint32_t dlo, uint32_t dhi, uint64_t q) {
  const int32_t q0 = P[1] * k8 + P[0], q1 = P[3] * k8 + P[2], q2 = P[5] * k8 + P[4], q3 = P[7] * k8 + P[6];
  const long long a = mad_wide(q1, k16, mad_wide(q0, k1, (long long)ca));
  const long long b = mad_wide(q3, k16, mad_wide(q2, k1, 1ll << 56));
  return reduce_pm(a, b, dlo, dhi, q);
}

__device__ __forceinline__ void transpose4x4(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t& p0,
                                             uint32_t& p1, uint32_t& p2, uint32_t& p3) {
  const uint32_t t0 = __byte_perm(a0, a1, 0x5140), t1 = __byte_perm(a0, a1, 0x7362);
  const uint32_t t2 = __byte_perm(a2, a3, 0x5140), t3 = __byte_perm(a2, a3, 0x7362);
  p0 = __byte_perm(t0, t2, 0x5410);
  p1 = __byte_perm(t0, t2, 0x7632);
  p2 = __byte_perm(t1, t3, 0x5410);
  p3 = __byte_perm(t1, t3, 0x7632);
}

// Phase 1 — relayout. X[p][f][jb][y][kh][d][16]: digit d of channel
// j = jb*32 + kh*16 + jj at extension slot (n - h + y + shift_j) of source
// ciphertext src_j + f*fstride (the negacyclic extension [q-a | a | q-a] of
// conv.py:251; the alignment DRot of conv.py:342 is the slot shift).
// One warp converts one unit = 32 positions x 16 channels: lane = position,
// 16 unconditional (clamped, in-bounds) coalesced 8-byte loads issued back to
// back, validity and the negacyclic sign applied afterwards from per-lane
// masks, 8 in-register 4x4 byte transposes into the lane's 128-byte half
// record, staged through the warp's shared memory (XOR-swizzled 16-byte
// chunks) so X is written with full 128-byte lines.
// FHE_CHECKS builds (tools/build_probe.py checked -DFHE_CHECKS=1; the sanitizer
// substitute on a pool where compute-sanitizer is closed): every global
// access of the kernel is bounds-checked against its operand's extent and the
// shared-memory ring placement against the ring; a violation traps.
#ifdef FHE_CHECKS
#define FHE_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define FHE_CHECK(cond) \
  do {                  \
  } while (0)
#endif

struct UnitLoad {
  uint64_t x[16];
  uint32_t neg, keep;
  int y0, jb, pf, kh;
};

// load half: all 16 loads issued back to back
__device__ __forceinline__ void relayout_load(const LayerDesc& d, int n, int unit, int lane, UnitLoad& U) {
  const int nyb = (d.Y + 31) / 32;
  const int kh = unit & 1, item = unit >> 1;  // a unit is one 16-channel K half of an item
  const int y0 = (item % nyb) * 32, jb = (item / nyb) % d.JB;
  const int pf = item / (nyb * d.JB), p = pf / d.F, f = pf - p * d.F;
  U.y0 = y0, U.jb = jb, U.pf = pf, U.kh = kh;
  // lane c (< 16) resolves channel jb*32 + kh*16 + c once: its row pointer and
  // the extension slot of position y0; the loop broadcasts them
  const int jm = jb * 32 + kh * 16 + (lane & 15);
  const int2 cm = jm < d.c_i ? __ldg(&d.chan[jm]) : make_int2(0, 0);
  const uint64_t* rowm = d.in + ((size_t)(cm.x + f * d.fstride) * 2 + p) * n;
  const int e0m = n - d.h + y0 + cm.y;  // in [0, 3n)
  const int live = max(0, min(16, d.c_i - jb * 32 - kh * 16));
  const int yoff = min(lane, d.Y - 1 - y0);  // clamped: every load is in bounds
  uint32_t neg = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    const uint64_t* row = reinterpret_cast<const uint64_t*>(
        __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rowm), c));
    int e = __shfl_sync(0xffffffffu, e0m, c) + yoff;
    const bool lo = e < n, hi = e >= 2 * n;
    e -= lo ? 0 : (hi ? 2 * n : n);
    FHE_CHECK(e >= 0 && e < n &&
              (const uint8_t*)(row + e) + 8 <= (const uint8_t*)d.in + d.in_bytes && (const uint64_t*)row >= d.in);
    U.x[c] = __ldg(&row[e]);
    neg |= (uint32_t)(lo || hi) << c;
  }
  U.keep = y0 + lane < d.Y ? (1u << live) - 1u : 0u;
  U.neg = neg & U.keep;
}

// store half: validity / sign masks, 8 in-register 4x4 byte transposes into
// the lane's 128-byte half record, staged (XOR-swizzled 16-byte chunks) so X
// is written with full 128-byte lines
__device__ __forceinline__ void relayout_store(const LayerDesc& d, uint64_t q, int lane, UnitLoad& U,
                                               uint8_t* stg) {
  if (!__all_sync(0xffffffffu, U.keep == 0xffffu)) {
#pragma unroll
    for (int c = 0; c < 16; ++c) U.x[c] = ((U.keep >> c) & 1) ? U.x[c] : 0;
  }
  if (__any_sync(0xffffffffu, U.neg != 0)) {
#pragma unroll
    for (int c = 0; c < 16; ++c)
      if (((U.neg >> c) & 1) && U.x[c]) U.x[c] = q - U.x[c];
  }
  uint32_t w[8][4];
#pragma unroll
  for (int g4 = 0; g4 < 4; ++g4) {
    const int c = g4 * 4;
    transpose4x4((uint32_t)U.x[c], (uint32_t)U.x[c + 1], (uint32_t)U.x[c + 2], (uint32_t)U.x[c + 3], w[0][g4],
                 w[1][g4], w[2][g4], w[3][g4]);
    transpose4x4((uint32_t)(U.x[c] >> 32), (uint32_t)(U.x[c + 1] >> 32), (uint32_t)(U.x[c + 2] >> 32),
                 (uint32_t)(U.x[c + 3] >> 32), w[4][g4], w[5][g4], w[6][g4], w[7][g4]);
  }
  // two rounds of 16 lanes through a 2 KB staging area: 16 positions x 128 B
  const int rows = min(32, d.Y - U.y0);
  // interleaved layers: position y of a plane lives at (y & 1) * Y/2 + (y >> 1) (y0 is even)
  const int ilv = d.ilv, yh = d.Y >> 1;
  uint4* dst = reinterpret_cast<uint4*>(d.X + (((size_t)U.pf * d.JB + U.jb) * d.Y + (ilv ? U.y0 >> 1 : U.y0)) * 256 +
                                        U.kh * 128);
  const uint4* st4 = reinterpret_cast<const uint4*>(stg);
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    if ((lane >> 4) == half) {
      uint4* mine = reinterpret_cast<uint4*>(stg + (lane & 15) * 128);
#pragma unroll
      for (int dd = 0; dd < 8; ++dd) mine[dd ^ (lane & 7)] = make_uint4(w[dd][0], w[dd][1], w[dd][2], w[dd][3]);
    }
    __syncwarp();
    // copy-out: 8 lanes per position half-record (128 contiguous bytes of X)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = i * 32 + lane, pl = idx >> 3, ch = idx & 7, pos = half * 16 + pl;
      if (pos < rows) {
        const int pd = ilv ? (pos & 1) * yh + (pos >> 1) : pos;
        FHE_CHECK((const uint8_t*)(dst + pd * 16 + ch + 1) <= d.X + d.x_bytes);
        dst[pd * 16 + ch] = st4[pl * 8 + (ch ^ (pl & 7))];
      }
    }
    __syncwarp();
  }
}

// Cross-CTA protocol — monotonic launch-scoped counters in `sync` (never
// reset, so CUDA-graph replays are safe); the grid is cooperative (every CTA
// resident) and all spins are bounded (a protocol bug traps, never hangs).
// P(l) = warps per CTA that relayout layer l: epilogue + relayout warps for
// layer 0 (nothing else to do yet), the kRelWarps relayout warps afterwards.
//   sync[0]             launch arrivals: epoch e = arrivals / gridDim.x + 1
//   sync[3 + l]         layer l's relayout work counter (dynamic relayout
//                       mode only), taken g = kUnitsPerGrab units at a time:
//                       launch e starts at (e-1)·(g·ceil(units/g) + g·G·P(l))
//                       (each participating warp overshoots it exactly once)
//   sync[kRdy + l]      layer l's relayout completions, one per CTA (its last
//                       participating warp publishes, see `publish`): its X
//                       is complete at e·G
//   sync[kGem + l]      layer l's GEMM completions (one per CTA): its X has
//                       been fully consumed at e·G
// Every layer has its OWN completion counters: warps and CTAs run ahead by
// up to three layers, so a shared running count can reach "layer l done"
// while a slow CTA is still on layer l (the config-5 stack, whose 80-fragment
// stem is relaid out next to two small layers, showed exactly that).
// X buffers: with x_stride > 0 three buffers rotate and the relayout warps run
// up to three layers ahead of the GEMM (layer l's buffer is overwritten only
// after every CTA finished the GEMM of layer l-3); with x_stride == 0 every
// layer owns its region of X and the relayout warps stream through the whole
// stack without waiting for the GEMM (the default: the small early layers'
// relayouts no longer throttle on the GEMMs three layers back). The loader
// waits for "X ready" before layer l's first stage.
// This CTA's 1/gridDim.x share of [p, p + bytes) into L2 (bulk prefetch).
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes) {
  const size_t share = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~(size_t)15;
  const size_t off = share * blockIdx.x;
  if (off >= bytes) return;
  const size_t len = min(share, bytes - off) & ~(size_t)15;
  if (len)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const uint8_t*>(p) + off),
                 "r"((uint32_t)len)
                 : "memory");
}

// Polls are relaxed (an acquire load would invalidate L1 on every poll); one
// acquire fence follows a successful poll.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void wait_count(const unsigned long long* p, unsigned long long target) {
  for (uint32_t i = 0; ld_relaxed(p) < target; ++i) {
    if (i > (1u << 26)) __trap();
    __nanosleep(64);
  }
  fence_acquire();
}

__device__ __forceinline__ bool mbar_test(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

// Tile-sequence ring: the loader decides which tile this CTA runs next (a
// static round-robin share or a dynamic grab) and publishes entry sq =
// {tag = sq + 1, layer << 24 | tile} with one release store; the MMA issuer
// and the epilogue warps read the same sequence (acquire loads). A sentinel
// entry with layer = nl ends it. The ring cannot overflow: the loader writes
// entry sq only after a stage slot freed by the MMAs of tile >= sq - 6 - 1, and
// the MMA issuer starts tile i only after the epilogue released tile i - 2.
__device__ __forceinline__ void tq_put(uint64_t* tq, int sq, int l, int t) {
  const uint64_t v = ((uint64_t)(((uint32_t)l << 24) | (uint32_t)t) << 32) | (uint32_t)(sq + 1);
  asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(tq + (sq % kTq))), "l"(v) : "memory");
}
__device__ __forceinline__ bool tq_peek(const uint64_t* tq, int sq, uint32_t& lt) {
  uint64_t v;
  asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(smem_u32(tq + (sq % kTq))) : "memory");
  lt = (uint32_t)(v >> 32);
  return (uint32_t)v == (uint32_t)(sq + 1);
}
__device__ __forceinline__ uint32_t tq_get(const uint64_t* tq, int sq) {
  uint32_t lt;
  for (uint32_t i = 0; !tq_peek(tq, sq, lt); ++i)
    if (i > (1u << 28)) __trap();
  return lt;
}

#if defined(FHE_STACK_MAXNREG)  // probe builds: a register cap instead of launch bounds
#define FHE_STACK_BOUNDS __maxnreg__(FHE_STACK_MAXNREG)
#else
#define FHE_STACK_BOUNDS __launch_bounds__(kThreads, 1)
#endif
template <int ML>
__global__ void FHE_STACK_BOUNDS conv_tc_stack_kernel(const __grid_constant__ StackArgsT<ML> A) {
  extern __shared__ __align__(1024) uint8_t smem[];
  unsigned long long* const trc = g_trace;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = A.n, nl = A.nl, G = gridDim.x;
  const uint64_t q = A.q;
  int ring_bytes = kEpiWarps * kStg;  // (same rule as the host's smem sizing)
  for (int l = 0; l < nl; ++l) ring_bytes = max(ring_bytes, A.L[l].res_bytes + A.L[l].nslots * A.L[l].slot_bytes);
  // relayout staging: the relayout warps own areas after the ring; the epilogue
  // warps (layer 0 only, before any stage is loaded) borrow the ring
  uint8_t* stg = warp >= 2 + kEpiWarps ? smem + ring_bytes + (warp - 2 - kEpiWarps) * kStg
                                       : smem + (warp - 2) * kStg;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ring_bytes + kRelWarps * kStg);
  // [0,6) full, [6,12) empty, 12+{0,1} tmem_full, 12+{2,3} tmem_empty
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2 * kMaxStages + 4);
  uint64_t* const tq = reinterpret_cast<uint64_t*>(slot + kSlotWords);  // [kTq] tile sequence
  const uint32_t bar0 = smem_u32(bars);
  auto full_bar = [&](int s) { return bar0 + 8 * s; };
  auto empty_bar = [&](int s) { return bar0 + 8 * (kMaxStages + s); };
  auto tfull_bar = [&](int b) { return bar0 + 8 * (2 * kMaxStages + b); };
  auto tempty_bar = [&](int b) { return bar0 + 8 * (2 * kMaxStages + 2 + b); };

  if (tid == 0) slot[1] = (unsigned)(atomicAdd(A.sync, 1ull) / (unsigned long long)G);  // epoch - 1
  unsigned* const cta_done = reinterpret_cast<unsigned*>(slot + 4);  // [kMaxLayers] warps of this CTA done
  if (tid < kMaxLayers) cta_done[tid] = 0;
  if (tid < kTq) tq[tid] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)),
                 "n"(2 * kAccCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int s = 0; s < kMaxStages; ++s) {
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
  // one CTA per SM allocates all 512 columns: the allocation starts at lane 0,
  // column 0. Using the constant (checked) keeps the MMA issuer's accumulator
  // addresses in uniform registers (no vector-to-uniform moves per MMA).
  if (slot[0] != 0) __trap();
  constexpr uint32_t tmem = 0;
  auto gtime = [] {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
  };
  if (trc && tid == 0) {  // per-CTA start (globaltimer ns, SM clock)
    trc[8 * 4096 + 2 * blockIdx.x] = gtime();
    trc[8 * 4096 + 512 + 2 * blockIdx.x] = clock64();
  }
  const unsigned long long e1 = slot[1];  // epoch - 1
  constexpr int P0 = kEpiWarps + kRelWarps;  // warps per CTA relaying out layer 0
  const unsigned long long Gu = (unsigned long long)G;
  auto ready_target = [&](int) { return (e1 + 1) * Gu; };  // one count per CTA per layer
  auto gemm_target = [&](int) { return (e1 + 1) * Gu; };
  // relayout units of layer l until none is left, then publish this warp's completion
  // relayout units of layer l until none is left, then publish this warp's
  // completion. The next grab's atomic is issued before the current unit is
  // processed, so its round trip overlaps useful work.
  // A warp finished its share of layer l's relayout (lane 0, after the warp
  // barrier): the CTA's last participating warp publishes ONE count for the
  // CTA (148 global atomics per layer instead of 148 x participants, all on
  // one address). Each warp's gpu-scope fence precedes its shared-memory
  // increment; the last warp, having read every increment, fences again
  // before the global count (cumulative release of all the CTA's X stores).
  auto publish = [&](int l, int participants) {
    __threadfence();
    if (atomicAdd(&cta_done[l], 1u) == (unsigned)participants - 1) {
      __threadfence();
      atomicAdd(A.sync + kRdy + l, 1ull);
#if FHE_TC_TRACE
      if (trc && l < 2) trc[8 * 4096 + 1024 + 2 * blockIdx.x + l] = gtime();  // this CTA's layer-0/1 relayout done (trace)
#endif
    }
  };
  auto relayout_layer = [&](int l, int participants) {
    const LayerDesc& d = A.L[l];
#if FHE_RELAYOUT_STATIC
    // static round-robin: relayout warp r of R takes units r, r + R, ... two at
    // a time. No shared work counter: ~1.7k atomics per layer on one address
    // serialised the early (small, latency-bound) layers; 2 % faster stack.
    {
      const int wi = participants == P0 ? warp - 2 : rel_late_rank(warp);
      const int R = G * participants;
#if FHE_REL_TWO
      for (int u = wi * G + (int)blockIdx.x; u < d.units; u += 2 * R) {
        UnitLoad U0, U1;
        const bool two = u + R < d.units;
        relayout_load(d, n, u, lane, U0);
        if (two) relayout_load(d, n, u + R, lane, U1);
        relayout_store(d, q, lane, U0, stg);
        if (two) relayout_store(d, q, lane, U1, stg);
      }
#else
#pragma unroll 1
      for (int u = wi * G + (int)blockIdx.x; u < d.units; u += R) {
        UnitLoad U0;
        relayout_load(d, n, u, lane, U0);
        relayout_store(d, q, lane, U0, stg);
      }
#endif
      // this warp's generic-proxy X stores -> the async proxy (the loaders'
      // cp.async.bulk reads, in any CTA) and its ring staging (layer 0, epilogue
      // warps) -> later bulk copies into the ring; then the release
#if FHE_XFENCE
      asm volatile("fence.proxy.async.global;");
#endif
      asm volatile("fence.proxy.async.shared::cta;");
      __threadfence();

      // every lane's X stores happen-before lane 0 (warp barrier), and lane 0's
      // own gpu-scope fence AFTER the barrier makes them (cumulatively) visible
      // before its completion count: a fence only before the barrier orders a
      // lane's stores with that lane's later operations, not lane 0's atomic
      __syncwarp();
      if (lane == 0) publish(l, participants);
      return;
    }
#endif
    constexpr unsigned long long kG = kUnitsPerGrab;
    const unsigned long long base = e1 * (kG * ((d.units + kG - 1) / kG) + kG * Gu * participants);
    unsigned long long nxt = 0;
    if (lane == 0) nxt = atomicAdd(A.sync + 3 + l, kG);
    for (;;) {
      const unsigned long long u = __shfl_sync(0xffffffffu, nxt, 0) - base;
      if (u >= (unsigned long long)d.units) break;
      if (lane == 0) nxt = atomicAdd(A.sync + 3 + l, kG);
      if (kUnitsPerGrab == 1) {
        UnitLoad U0;
        relayout_load(d, n, (int)u, lane, U0);
        relayout_store(d, q, lane, U0, stg);
      } else {
        UnitLoad U0, U1;
        const bool two = u + 1 < (unsigned long long)d.units;
        relayout_load(d, n, (int)u, lane, U0);
        if (two) relayout_load(d, n, (int)u + 1, lane, U1);
        relayout_store(d, q, lane, U0, stg);
        if (two) relayout_store(d, q, lane, U1, stg);
      }
    }
    asm volatile("fence.proxy.async.global;");      // X stores -> the async proxy (cp.async.bulk readers)
    asm volatile("fence.proxy.async.shared::cta;");  // (epilogue warps) ring staging before later bulk copies
    __threadfence();  // this warp's X stores before its completion count
    __syncwarp();
    if (lane == 0) publish(l, participants);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ MMA issue
    // TMEM: two 256-column accumulator buffers. A 32-position tile takes the
    // next buffer in turn (the epilogue of one overlaps the MMAs of the next);
    // a 64-position tile takes both (acc a <- positions 32a..32a+31, same
    // weights: half the weight traffic per position). Per-buffer use counts
    // give the tmem_full / tmem_empty parities on both sides.
    {  // the whole warp runs the issue loop; elect.sync issues (see mma_i8w_elect)
      int s_mma = 0, prev_sb = -1, prev_ns = -1, prev_res = 0, tl = 0, nb = 0;
      uint32_t par = 0, use = 0;  // per-stage full parity; per-buffer use parity (bit b)
      const uint64_t desc0 = umma_desc(smem_u32(smem));  // ring base; stage s adds s * stage_bytes / 16
      const uint32_t dlo0 = (uint32_t)desc0, dhi = (uint32_t)(desc0 >> 32);
      bool pre = false;  // the current stage's full barrier was already waited for
      uint32_t lt = tq_get(tq, 0);  // the loader's tile sequence (layers in increasing order)
      for (int l = 0; l < nl; ++l) {
        if ((int)(lt >> 24) != l) continue;  // no tiles of this layer here
        const LayerDesc& d = A.L[l];
        // Per-layer values in registers, scoped to the layer: the barrier asm below
        // clobbers memory, so fields read through `d` inside the loops would be
        // re-fetched from the parameter bank (dependent LDCs) at every stage, and
        // loop-carried copies leave the issue path vector-to-uniform moves per MMA.
        const int slot_bytes = d.slot_bytes, JB = d.JB, nacc = d.nacc, taps = d.taps, nst = d.nslots;
        const int res = d.res_bytes;
        // the loader drained and re-partitioned the ring (resident weights: always)
        if (slot_bytes != prev_sb || nst != prev_ns || res || prev_res) s_mma = 0;
        prev_sb = slot_bytes;
        prev_ns = nst;
        prev_res = res;
        const uint32_t rlo = dlo0 + (uint32_t)(res >> 4);  // first slot (after any resident weights)
        const uint32_t wtap = (uint32_t)(taps * (kWTap >> 4));  // resident weights: one 32-channel block
        const uint32_t idesc = idesc_i8(8 * d.npos);
        const uint32_t sstep = (uint32_t)(slot_bytes >> 4), wdesc = (uint32_t)(d.win_bytes >> 4);
        const uint32_t adelta = (uint32_t)(d.npos * 256 >> 4);  // second accumulator's positions
        uint32_t off16[16];  // this layer's DRot offsets in 16-byte descriptor units (fast paths)
#pragma unroll
        for (int tp = 0; tp < 16; ++tp) off16[tp] = tp < taps ? (uint32_t)d.tap_off[tp] * 16 : 0u;
        const int nstage = JB;
        for (;; ++tl) {  // this CTA's tiles of layer l, in the loader's order
          int b0 = 0, b1 = 1;
          if (nacc == 1) {
            b0 = nb;
            nb ^= 1;
          }
          if (lane == 0) TC_TRACE(0, tl);
          for (int jb = 0; jb < nstage; ++jb) {  // stage = one 32-channel block
            const int s = s_mma;
            const int s_next = s + 1 == nst ? 0 : s + 1;
            if (!pre) {
              mbar_wait(full_bar(s), (par >> s) & 1);
              par ^= 1u << s;
            }
            pre = false;
            asm volatile("tcgen05.fence::after_thread_sync;");
            const uint32_t blo0 = rlo + (uint32_t)s * sstep;  // window at the stage base
            // weights after the window, or resident at the ring base
            const uint32_t alo = res ? dlo0 + (uint32_t)jb * wtap : blo0 + wdesc;
            // a next stage of this layer: within the tile, or the sequence's next tile
            // when it is already published and of this layer
            bool has_next = jb + 1 < nstage;
            if (!has_next) {
              uint32_t nlt;
              has_next = tq_peek(tq, tl + 1, nlt) && (int)(nlt >> 24) == l;
            }
            for (int a = 0; a < nacc; ++a) {
              const int b = a == 0 ? b0 : b1;
              if (jb == 0) {  // first use of this buffer in the tile: the epilogue must have drained it
                mbar_wait(tempty_bar(b), ((use >> b) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                if (a == 0 && lane == 0) TC_TRACE(4, tl);
              }
              const uint32_t acc = tmem + b * kAccCols;
              const uint32_t blo = blo0 + (uint32_t)a * adelta;
              auto wait_next = [&] {
                if (a == nacc - 1 && has_next) {
                  mbar_wait(full_bar(s_next), (par >> s_next) & 1);
                  par ^= 1u << s_next;
                  pre = true;
                }
              };
              if (taps == 9) {
                issue_taps<9>(acc, alo, blo, dhi, off16, idesc, jb == 0, wait_next);
              } else if (taps == 1) {
                issue_taps<1>(acc, alo, blo, dhi, off16, idesc, jb == 0, wait_next);
              } else if (taps == 14) {  // 7 column taps x 2 stacked position groups (the 7x7 stem)
                issue_taps<14>(acc, alo, blo, dhi, off16, idesc, jb == 0, wait_next);
              } else if (taps == 7) {
                issue_taps<7>(acc, alo, blo, dhi, off16, idesc, jb == 0, wait_next);
#if FHE_ILV_FAST
              } else if (taps == 8) {  // 7 column taps, two interleaved position groups (the 7x7 stem)
                issue_taps<8>(acc, alo, blo, dhi, off16, idesc, jb == 0, wait_next);
              } else if (taps == 12) {  // 3x3, two interleaved position groups
                issue_taps<12>(acc, alo, blo, dhi, off16, idesc, jb == 0, wait_next);
#endif
              } else {
                for (int tp = 0; tp < taps; ++tp) {
                  if (tp == taps - 1) wait_next();
                  mma_i8w_elect(acc, alo + (uint32_t)(tp * (4096 >> 4)), blo + (uint32_t)d.tap_off[tp] * 16, dhi,
                                idesc, (jb | tp) != 0);
                }
              }
            }
            mma_commit_elect(empty_bar(s));  // stage free once these MMAs retire
            s_mma = s_next;
          }
          for (int a = 0; a < nacc; ++a) {
            const int b = a == 0 ? b0 : b1;
            mma_commit_elect(tfull_bar(b));  // accumulator complete
            use ^= 1u << b;
          }
          if (lane == 0) TC_TRACE(1, tl);
          lt = tq_get(tq, tl + 1);
          if ((int)(lt >> 24) != l) {
            ++tl;
            break;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ stage loads
    if (lane == 0) {
      int s_ld = 0, prev_sb = -1, prev_ns = -1, prev_res = 0, sq = 0;
      uint32_t par = 0, used = 0;  // per-stage fill parity; stages filled at least once
      for (int l = 0; l < nl; ++l) {
        const LayerDesc& d = A.L[l];
        const int tiles = d.tiles;
        // this CTA's tiles of layer l: a static round-robin share, or grabbed from the
        // layer's counter (one grab stays in flight ahead of the loads). Every CTA
        // overshoots the counter exactly once, so the grab that returns tiles + G - 1
        // is the launch's last one: that CTA resets the counter for the next launch
        // (no epoch arithmetic: a counter buffer shared by different stacks stays valid).
        unsigned long long* const ctr = A.sync + kTile + l;
        int t_static = first_tile(d);
        if (!A.dyn && tiles <= t_static) continue;  // no tiles of this layer here
        wait_count(A.sync + kRdy + l, ready_target(l));  // layer l's X is complete
        TC_TRACE(7, l);
        asm volatile("fence.proxy.async.global;");  // generic-proxy X stores -> cp.async.bulk reads
        unsigned long long nxt = A.dyn ? atomicAdd(ctr, 1ull) : 0ull;
        bool first = true, res_pending = false;
        const uint32_t wstage = (uint32_t)d.taps * kWTap;
        const size_t plane_stride = (size_t)d.Y * 256;
        const uint32_t win_load = (uint32_t)((d.tpos + 2 * d.h) * 256);
        for (;;) {
          int t;
          if (A.dyn) {
            if (nxt >= (unsigned long long)tiles) {
              if (nxt == (unsigned long long)tiles + Gu - 1) atomicExch(ctr, 0ull);
              break;
            }
            t = (int)nxt;
            nxt = atomicAdd(ctr, 1ull);
          } else {
            if (t_static >= tiles) break;
            t = t_static;
            t_static += G;
          }
          if (first) {
            first = false;
            if (d.slot_bytes != prev_sb || d.nslots != prev_ns || d.res_bytes || prev_res) {
              // new ring partition (or new resident weights): every stage of the old one must be
              // consumed first (MMAs complete in order: the last stage's release also frees the
              // previous layer's resident weights)
              for (int s = 0; s < kMaxStages; ++s)
                if ((used >> s) & 1) mbar_wait_sleep(empty_bar(s), ((par >> s) & 1) ^ 1, 32);
              s_ld = 0;
              prev_sb = d.slot_bytes;
              prev_ns = d.nslots;
              prev_res = d.res_bytes;
            }
            res_pending = d.res_bytes > 0;  // the resident weights ride on the layer's first stage
          }
#if FHE_TC_TRACE
          if (trc && blockIdx.x == 0 && sq < 1024) trc[7 * 4096 + 1024 + sq] = l;  // the sequence's layers (trace)
#endif
          tq_put(tq, sq++, l, t);
          const Tile T = tile_of(t, d, n);
          const uint8_t* xbase = d.X + ((size_t)(T.p * d.F + T.f) * d.JB) * plane_stride + (size_t)T.s0 * 256;
          const uint8_t* xilv = xbase - (size_t)(T.s0 >> 1) * 256;  // (interleaved: the even half starts at s0 / 2)
          const uint8_t* wbase = d.W + (size_t)T.ob * d.JB * wstage;
          for (int jb = 0; jb < d.JB; ++jb) {  // stage = one 32-channel block
            const int s = s_ld;
            if ((used >> s) & 1) mbar_wait_sleep(empty_bar(s), ((par >> s) & 1) ^ 1, 32);
            used |= 1u << s;
            par ^= 1u << s;
            const uint32_t pos = (uint32_t)(d.res_bytes + s * d.slot_bytes);
            const uint32_t sx = smem_u32(smem + pos);
#ifdef TC_PROBE_NOFILL  // timing probe only: MMAs on stale stage data, no fill traffic
            (void)sx;
            (void)xbase;
            (void)wbase;
            mbar_arrive(full_bar(s));
#else
            if (d.res_bytes) {  // window only; the first stage also brings the resident weights
              const uint32_t extra = res_pending ? (uint32_t)d.res_bytes : 0u;
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full_bar(s)),
                           "r"(win_load + extra)
                           : "memory");
              FHE_CHECK(pos + (uint32_t)d.slot_bytes <= (uint32_t)(d.res_bytes + d.nslots * d.slot_bytes) &&
                        win_load <= (uint32_t)d.slot_bytes && d.OB == 1 &&
                        xbase + (size_t)jb * plane_stride + win_load <= d.X + d.x_bytes &&
                        (size_t)d.res_bytes <= d.w_bytes);
              if (d.ilv) {  // even positions, then odd positions (each 32 + h) of the plane
                bulk_load(sx, xilv + (size_t)jb * plane_stride, win_load >> 1, full_bar(s));
                bulk_load(sx + (win_load >> 1), xilv + (size_t)jb * plane_stride + (plane_stride >> 1), win_load >> 1,
                          full_bar(s));
              } else {
                bulk_load(sx, xbase + (size_t)jb * plane_stride, win_load, full_bar(s));
              }
              if (res_pending) bulk_load(smem_u32(smem), d.W, (uint32_t)d.res_bytes, full_bar(s));
              res_pending = false;
            } else {
              asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(full_bar(s)),
                           "r"(win_load + wstage)
                           : "memory");
              FHE_CHECK(pos + (uint32_t)d.stage_bytes <= (uint32_t)(d.nslots * d.slot_bytes) &&
                        d.stage_bytes <= d.slot_bytes &&
                        win_load <= (uint32_t)d.win_bytes && xbase + (size_t)jb * plane_stride + win_load <= d.X + d.x_bytes &&
                        wbase + (size_t)(jb + 1) * wstage <= d.W + d.w_bytes);
              if (d.ilv) {
                bulk_load(sx, xilv + (size_t)jb * plane_stride, win_load >> 1, full_bar(s));
                bulk_load(sx + (win_load >> 1), xilv + (size_t)jb * plane_stride + (plane_stride >> 1), win_load >> 1,
                          full_bar(s));
              } else {
                bulk_load(sx, xbase + (size_t)jb * plane_stride, win_load, full_bar(s));
              }
              bulk_load(sx + d.win_bytes, wbase + (size_t)jb * wstage, wstage, full_bar(s));
            }
#endif
            s_ld = s + 1 == d.nslots ? 0 : s + 1;
          }
        }
      }
      tq_put(tq, sq, nl, 0);  // end of this CTA's sequence
    }
  } else if (warp >= 2 + kEpiWarps) {
    // ------------------------------------------------------- relayout warps
    if (tid == 32 * (2 + kEpiWarps)) TC_TRACE(2, 0);
    const bool pf = tid == 32 * (2 + kEpiWarps);  // one thread per CTA issues the L2 prefetches
    if (pf) {  // the first layers' inputs (read by relayout) and layer 0's weights (read by the GEMM)
      for (int k = 1; k <= kPfAhead && k < nl; ++k) prefetch_l2(A.L[k].in, A.L[k].in_bytes);
      prefetch_l2(A.L[0].W, A.L[0].w_bytes);
    }
    relayout_layer(0, P0);
    for (int l = 1; l < nl && rel_late(warp); ++l) {
      if (pf) {  // the input kPfAhead layers on, and this layer's weights
        if (l + kPfAhead < nl) prefetch_l2(A.L[l + kPfAhead].in, A.L[l + kPfAhead].in_bytes);
        prefetch_l2(A.L[l].W, A.L[l].w_bytes);
      }
      if (A.xrot && l >= 3) wait_count(A.sync + kGem + l - 3, gemm_target(l - 3));  // X[l % 3] no longer read anywhere
      if (lane == 0 && warp == 2 + kEpiWarps) TC_TRACE(2, 64 + l);  // this warp starts layer l's relayout
      relayout_layer(l, kRelLate);
      if (lane == 0 && warp == 2 + kEpiWarps) TC_TRACE(3, l);
    }
  } else {
    // -------------------------------------------------------------- epilogue
    const int quad = warp & 3, sub = (warp - 2) >> 2;
    const int k1 = A.k1, k8 = A.k8, k16 = A.k16, k24 = A.k24;
    const int pm = A.pm;
    const uint64_t pm_ca = A.pm_ca;
    const uint32_t pm_dlo = A.pm_dlo, pm_dhi = A.pm_dhi;
    relayout_layer(0, P0);  // nothing to do yet but help with layer 0
    int nb = 0, tl = 0;
    uint32_t use = 0;  // per-buffer use parity (mirrors the MMA thread)
    uint32_t lt = tq_get(tq, 0);  // the loader's tile sequence (layers in increasing order)
    for (int l = 0; l < nl; ++l) {
      if ((int)(lt >> 24) == l) {
        const LayerDesc& d = A.L[l];
        // per-layer values in registers (the store asm below clobbers memory:
        // fields read through `d` in the chunk loop were re-fetched from the
        // parameter bank every chunk)
        const int c_o = d.c_o, F = d.F, npos = d.npos, nacc = d.nacc, pair = d.pair;
        // rows of the accumulator: rep groups of rows_per output channels, group
        // r holding positions [32 r, 32 r + 32) of the tile
        // (interleaved groups, d.ilv: row 2 o + r = channel o at positions s0 + 2 u + r)
        const int ilv = FHE_ILV_EPI ? d.ilv : 0;
        const int rows_per = kOcTile / d.rep;
        const int grp = ilv ? 0 : (quad * 32 + lane) / rows_per;
        const int orow = ilv ? (quad * 32 + lane) >> 1 : (quad * 32 + lane) % rows_per;
        uint64_t* const dout = d.out;
        const uint8_t* const bmask = d.bmask;
        const uint64_t* const bias = d.bias;
        for (;; ++tl) {  // this CTA's tiles of layer l, in the loader's order
        const int t = (int)(lt & 0xFFFFFFu);
        const Tile T = tile_of(t, d, n);
        const int o = T.ob * kOcTile + orow;
        const bool active = T.ob * kOcTile + (ilv ? quad * 16 : (quad * 32) % rows_per) < c_o;  // warp-uniform
        const uint64_t bd = (active && T.p == 0 && bias && o < c_o) ? bias[o] : 0;
        for (int a = 0; a < nacc; ++a) {
          int buf;
          if (nacc == 1) {
            buf = nb;
            nb ^= 1;
          } else {
            buf = a;
          }
          const int s0 = T.s0 + (a + grp) * npos;
#if FHE_EPI_SLEEP
          mbar_wait_sleep(tfull_bar(buf), (use >> buf) & 1, 64);
#else
          // no nanosleep: a sleeping warp woke up to ~1k cycles after its accumulator was
          // ready, and the slowest epilogue warp sets the tile period (try_wait suspends
          // the warp in hardware between polls)
          mbar_wait(tfull_bar(buf), (use >> buf) & 1);
#endif
          use ^= 1u << buf;
          if (lane == 0 && warp == 2) TC_TRACE(5, tl);
          if (lane == 0) TC_TRACE(9 + warp - 2, tl);  // every epilogue warp: tfull seen
          asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef TC_PROBE_NOEPI  // timing probe only: accumulators released unread
          if (false) {
#else
          if (active) {
#endif
            // lane = output channel within the quadrant; a 32-column TMEM chunk
            // holds 4 positions x 8 planes. lo = q + Σ_{d<4} 2^(8d) P_d and
            // hi = q + Σ_{d>=4} 2^(8(d-4)) P_d lie in (0, 2q) (|P_d| < 2^31,
            // q > 2^56); V = lo + 2^32 hi.
            const uint32_t acc = tmem + buf * kAccCols + ((uint32_t)(quad * 32) << 16);
            uint64_t* orow = dout + ((size_t)(o * F + T.f) * 2 + T.p) * n + s0;
            // each warp of the quadrant takes a contiguous half of the chunks: a
            // lane then writes whole 128-byte lines of its channel row
            // the quadrant's npos/4 chunks split over its kEpiWarps/4 warps (contiguous ranges)
            constexpr int kEpq = kEpiWarps / 4;
            const int k_lo = sub * (npos / 4) / kEpq, k_hi = (sub + 1) * (npos / 4) / kEpq;
            const int kper = k_hi - k_lo;
            // recombine the 4 positions of one 32-column chunk and store them
            auto finish = [&](const uint32_t* v, int k, auto pm_tag) {
              uint64_t r[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int32_t* P = reinterpret_cast<const int32_t*>(v + 8 * j);
                if constexpr (decltype(pm_tag)::value == 2) {
                  r[j] = finish_pm_pair(P, k1, k8, k16, pm_ca, pm_dlo, pm_dhi, q);
                } else if constexpr (decltype(pm_tag)::value == 1) {
                  r[j] = finish_pm(P, k1, k8, k16, k24, pm_ca, pm_dlo, pm_dhi, q);
                } else {
                  const long long lo = mad_wide(P[3], k24, mad_wide(P[2], k16, mad_wide(P[1], k8, mad_wide(P[0], k1, q))));
                  const long long hi = mad_wide(P[7], k24, mad_wide(P[6], k16, mad_wide(P[5], k8, mad_wide(P[4], k1, q))));
                  // 2^32 hi mod q by Shoup (w = 2^32 < q): result in [0, 2q)
                  const uint64_t uh = ((uint64_t)hi << 32) - __umul64hi(A.w32p, (uint64_t)hi) * q;
                  uint64_t val = (uint64_t)lo + uh;  // < 4q
                  val = val >= 2 * q ? val - 2 * q : val;
                  r[j] = val >= q ? val - q : val;
                }
              }
              int kk = 4 * k;  // the lane's 4 consecutive positions within the tile row
              if (ilv) {
                // the lane pair (2 o, 2 o + 1) holds positions 8 k + {0, 2, 4, 6} and 8 k + {1, 3, 5, 7}:
                // exchange two values each so the even lane stores 8 k .. 8 k + 3, the odd one 8 k + 4 .. + 7
                const bool odd = lane & 1;
                const uint64_t g0 = __shfl_xor_sync(0xffffffffu, odd ? r[0] : r[2], 1);
                const uint64_t g1 = __shfl_xor_sync(0xffffffffu, odd ? r[1] : r[3], 1);
                if (odd) {
                  r[0] = g0; r[1] = r[2]; r[2] = g1;
                } else {
                  r[2] = r[1]; r[1] = g0; r[3] = g1;
                }
                kk = 8 * k + (odd ? 4 : 0);
              }
              if (bd) {
                const uint32_t mk = *reinterpret_cast<const uint32_t*>(bmask + (size_t)T.f * n + s0 + kk);
#pragma unroll
                for (int j = 0; j < 4; ++j)
                  if ((mk >> (8 * j)) & 0xff) r[j] = csub(r[j] + bd, q);
              }
#ifdef TC_PROBE_NOSTORE  // timing probe only: results reduced but not stored
              if (o < c_o && (r[0] ^ r[1] ^ r[2] ^ r[3]) == 0x5eed5eedull) orow[0] = 1;
#else
              FHE_CHECK(o >= c_o || ((uint8_t*)(orow + kk + 4) <= (uint8_t*)dout + d.out_bytes &&
                                     s0 + kk + 4 <= n));
              if (o < c_o)  // one 32-byte store per lane: a full sector (STG.256)
                asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(orow + kk), "l"(r[0]), "l"(r[1]),
                             "l"(r[2]), "l"(r[3])
                             : "memory");
#endif
            };
            auto chunks = [&](auto pm_tag) {
              if (FHE_EPI_PAIR && kper % 2 == 0) {
                // two chunks per TMEM round trip: both loads in flight before the
                // one wait (tcgen05.wait::ld covers every outstanding load)
#pragma unroll 1
                for (int k = k_lo; k < k_hi; k += 2) {
                  uint32_t va[32], vb[32];
                  TMEM_LD32(acc + k * 32, va);
                  TMEM_LD32(acc + (k + 1) * 32, vb);
                  asm volatile("tcgen05.wait::ld.sync.aligned;");
                  finish(va, k, pm_tag);
                  finish(vb, k + 1, pm_tag);
                }
              } else {
#if FHE_EPI_PIPE && !defined(TC_PROBE_NOLD) && !defined(TC_PROBE_LDONLY) && !defined(TC_PROBE_Q0LD)
                // software pipeline: chunk k+1's TMEM load is in flight while
                // chunk k is recombined and stored (two register sets, no copies)
                if (decltype(pm_tag)::value == 2 && k_lo < k_hi) {  // (the pair path: fewest temporaries)
                  uint32_t va[32], vb[32];
                  TMEM_LD32(acc + k_lo * 32, va);
                  TMEM_WAIT32(va);
#pragma unroll 1
                  for (int k = k_lo;; k += 2) {
                    const bool m1 = k + 1 < k_hi;
                    if (m1) TMEM_LD32(acc + (k + 1) * 32, vb);
                    finish(va, k, pm_tag);
                    if (!m1) break;
                    TMEM_WAIT32(vb);
                    const bool m2 = k + 2 < k_hi;
                    if (m2) TMEM_LD32(acc + (k + 2) * 32, va);
                    finish(vb, k + 1, pm_tag);
                    if (!m2) break;
                    TMEM_WAIT32(va);
                  }
                }
                if (decltype(pm_tag)::value != 2)
#endif
#pragma unroll 1
                for (int k = k_lo; k < k_hi; ++k) {
                  uint32_t v[32];
#if defined(TC_PROBE_NOLD)  // timing probe only: arithmetic and stores on register garbage, no TMEM loads
#pragma unroll
                  for (int i = 0; i < 32; ++i) v[i] = (uint32_t)opaque(k * 32 + i);
#else
                  TMEM_LD32(acc + k * 32, v);
                  asm volatile("tcgen05.wait::ld.sync.aligned;");
#endif
#if defined(TC_PROBE_LDONLY)  // timing probe only: TMEM loads, no arithmetic or stores
                  if (v[0] == 0x5eed5eedu && v[31] == 0x1234567u) dout[0] = v[7];
#elif defined(TC_PROBE_Q0LD)  // timing probe only: the MMA warp's sub-partition (quadrant 0) skips the arithmetic
                  if (quad == 0) {
                    if (v[0] == 0x5eed5eedu && v[31] == 0x1234567u) dout[0] = v[7];
                  } else {
                    finish(v, k, pm_tag);
                  }
#else
                  finish(v, k, pm_tag);
#endif
                }
              }
            };
            if (pm && pair)
              chunks(std::integral_constant<int, 2>{});
            else if (pm)
              chunks(std::integral_constant<int, 1>{});
            else
              chunks(std::integral_constant<int, 0>{});
          }
          asm volatile("tcgen05.fence::before_thread_sync;");
          mbar_arrive(tempty_bar(buf));
          if (lane == 0 && warp == 2) TC_TRACE(6, tl);
          if (lane == 0) TC_TRACE(9 + kEpiWarps + warp - 2, tl);  // every epilogue warp: done
        }
        lt = tq_get(tq, tl + 1);
        if ((int)(lt >> 24) != l) {
          ++tl;
          break;
        }
        }
      }
      // this CTA consumed all of layer l's X (every tile's MMAs completed). Only the rotating-X mode
      // with more than three layers ever waits for this count; otherwise the epilogue warps move on
      // to the next layer without meeting at a barrier.
      if (FHE_GEM_ALWAYS || (A.xrot && nl > 3)) {
        asm volatile("bar.sync 1, %0;" ::"n"(kEpilogue));
        if (tid == 64) {
          __threadfence();
          atomicAdd(A.sync + kGem + l, 1ull);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * kAccCols));
  if (trc && tid == 0) {  // per-CTA end
    trc[8 * 4096 + 2 * blockIdx.x + 1] = gtime();
    trc[8 * 4096 + 512 + 2 * blockIdx.x + 1] = clock64();
  }
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
  unsigned long long c0 = 0, g0 = 0;
  if (threadIdx.x == 0) {
    c0 = clock64();
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    const uint64_t ad = umma_desc(smem_u32(smem)), bd = umma_desc(smem_u32(smem + 4096));
    constexpr uint32_t idesc = idesc_i8(N);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) mma_i8(tmem + (k & 1) * 256, ad, bd, idesc, 1);
    }
    mma_commit(smem_u32(bar));
  }
  mbar_wait(smem_u32(bar), 0);
  if (threadIdx.x == 0 && blockIdx.x == 0) {  // SM clock of the probe: cycles and ns of CTA 0 (sink[2..5])
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    reinterpret_cast<unsigned long long*>(sink)[1] = clock64() - c0;
    reinterpret_cast<unsigned long long*>(sink)[2] = g1 - g0;
  }
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

static unsigned long long* g_trace_host = nullptr;  // host copy of the trace pointer (launch metadata)

int fhe_debug_trace(void* dev_buf) {
  unsigned long long* p = (unsigned long long*)dev_buf;
  FHE_CUDA(cudaMemcpyToSymbol(tc::g_trace, &p, sizeof(p)));
  g_trace_host = p;
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

// FHE_TC_BALANCE=1: cost-aware dealing of each layer's extra tiles (measured
// 1 % slower than the round-robin continuation on configs 4 and 5: the
// per-tile cost estimate misses the pipeline overlap; kept as an option)
static bool balance_tiles() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_TC_BALANCE");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

static bool pm_allowed() {  // FHE_TC_NO_PM=1: the general (Shoup) epilogue for every modulus (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_TC_NO_PM");
    v = (e && e[0] == '1') ? 0 : 1;
  }
  return v == 1;
}

static bool resident_allowed() {  // FHE_TC_RESIDENT=0: weights streamed with every stage (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_TC_RESIDENT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static bool dynamic_tiles() {  // FHE_TC_DYNAMIC=0: static round-robin tile dealing (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_TC_DYNAMIC");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static bool keep_partition() {  // FHE_TC_KEEP_RING=0: re-partition at every stage-size change (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_TC_KEEP_RING");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int fhe_conv_tc_stack(uint64_t q, int n, const fhe_conv_tc_layer* layers, int nl, uint8_t* X, size_t x_stride,
                      uint64_t* sync, void* stream) {
  if (q < (1ull << 56) || q >= (1ull << 62)) return fail(FHE_ERR_VALUE, "tc path needs 2^56 <= q < 2^62");
  if (n < 64 || (n & (n - 1))) return fail(FHE_ERR_VALUE, "tc path needs a power-of-two n >= 64");
  if (nl < 1 || nl > tc::kMaxLayers) return fail(FHE_ERR_VALUE, "tc stack: 1..%d layers", tc::kMaxLayers);
  if (!layers || !X || !sync) return fail(FHE_ERR_VALUE, "null tc stack operand");
  // large: kept off the stack; per host thread (launches from several threads do not share it)
  static thread_local tc::StackArgs A;
  A.q = q;
  A.w32p = h_shoup(1ull << 32, q);
  A.n = n;
  A.nl = nl;
  A.xrot = x_stride ? 1 : 0;
  A.dyn = dynamic_tiles() ? 1 : 0;
  A.k1 = 1;
  A.k8 = 1 << 8;
  A.k16 = 1 << 16;
  A.k24 = 1 << 24;
  {
    const uint64_t delta = (1ull << 60) - q;  // pseudo-Mersenne fast path (finish_pm)
    A.pm = (q < (1ull << 60) && delta < (1ull << 35) && pm_allowed()) ? 1 : 0;
    A.pm_dlo = (uint32_t)delta;
    A.pm_dhi = (uint32_t)(delta >> 32);
    const unsigned __int128 t88 = (unsigned __int128)1 << 88;
    uint64_t ca = (uint64_t)((q - (uint64_t)(t88 % q)) % q);  // -2^88 mod q
    if (ca < (1ull << 56)) ca += q;
    A.pm_ca = ca;
  }
  size_t xoff = 0;
  A.sync = reinterpret_cast<unsigned long long*>(sync);
  int max_tiles = 0, ring = 0, toff = 0;
  double load[1024] = {0};  // estimated work per CTA (tile dealing, see balance_tiles)
  // per device: the SM count (grid size) and the kernel's shared-memory attribute
  constexpr int kMaxDevices = 64;
  static std::atomic<int> sms_of[kMaxDevices];
  static std::atomic<bool> attr_of[kMaxDevices];
  int dev = 0;
  FHE_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) return fail(FHE_ERR_VALUE, "device index %d out of range", dev);
  int sms_now = sms_of[dev].load(std::memory_order_relaxed);
  if (!sms_now) {
    FHE_CUDA(cudaDeviceGetAttribute(&sms_now, cudaDevAttrMultiProcessorCount, dev));
    sms_of[dev].store(sms_now, std::memory_order_relaxed);
  }
  if (sms_now > 1024) return fail(FHE_ERR_VALUE, "too many SMs");
  for (int l = 0; l < nl; ++l) {
    const fhe_conv_tc_layer& s = layers[l];
    tc::LayerDesc& d = A.L[l];
    if (s.c_i < 1 || s.frags < 1 || s.c_o < 1 || s.taps < 1 || s.taps > tc::kMaxTaps || s.h < 0 || 2 * s.h >= n)
      return fail(FHE_ERR_VALUE, "tc layer %d: bad shape", l);
    if (!s.in || !s.chan || !s.w || !s.out || !s.tap_steps) return fail(FHE_ERR_VALUE, "tc layer %d: null operand", l);
    if (s.n_in < 1) return fail(FHE_ERR_VALUE, "tc layer %d: n_in must be >= 1", l);
    if (s.bias_delta && !s.bias_mask) return fail(FHE_ERR_VALUE, "tc layer %d: bias needs a mask", l);
    if (s.pos_tile != 16 && s.pos_tile != 32 && s.pos_tile != 64)
      return fail(FHE_ERR_VALUE, "tc layer %d: pos_tile must be 16, 32 or 64", l);
    const int rep = s.rep < 1 ? 1 : s.rep;
    if (rep != 1 && rep != 2 && rep != 4) return fail(FHE_ERR_VALUE, "tc layer %d: rep must be 1, 2 or 4", l);
    if (rep > 1 && (s.pos_tile != 32 || s.c_o > tc::kOcTile / rep))
      return fail(FHE_ERR_VALUE, "tc layer %d: rep %d needs pos_tile 32 and c_o <= %d", l, rep, tc::kOcTile / rep);
    // rep 2 with tsplit 2: the two position groups interleave (LayerDesc.ilv); taps / tap_steps / w are
    // then the MERGED taps (distinct window offsets step + r), each one full-height MMA
    const bool ilv = rep == 2 && s.tsplit == 2;
    if (!ilv && s.taps * rep > tc::kMaxTaps)
      return fail(FHE_ERR_VALUE, "tc layer %d: taps x rep above %d", l, tc::kMaxTaps);
    if (127ll * 255 * ((s.c_i + 31) / 32 * 32) * s.taps >= (1ll << 31))
      return fail(FHE_ERR_VALUE, "tc layer %d: plane sums would exceed s32", l);
    d.in = s.in;
    d.chan = reinterpret_cast<const int2*>(s.chan);
    if (x_stride) {
      d.X = X + (size_t)(l % 3) * x_stride;
    } else {  // own region per layer, consecutive, 256-byte aligned
      d.X = X + xoff;
    }
    d.W = reinterpret_cast<const uint8_t*>(s.w);
    d.bias = s.bias_delta;
    d.bmask = s.bias_mask;
    d.out = s.out;
    d.Y = n + 2 * s.h;
    d.JB = (s.c_i + 31) / 32;
    d.F = s.frags;
    d.c_i = s.c_i;
    d.fstride = s.fstride;
    d.c_o = s.c_o;
    d.OB = (s.c_o + tc::kOcTile - 1) / tc::kOcTile;
    d.taps = ilv ? s.taps : s.taps * rep;  // MMAs per 32-channel block: every tap for every stacked position group
    if (s.tsplit > 1 && !ilv) return fail(FHE_ERR_VALUE, "tc layer %d: tsplit is 0, 1, or 2 with rep 2", l);
    d.rep = rep;
    d.ilv = ilv ? 1 : 0;
    // |P_d| <= 127·255·c_i·taps (each accumulator row sums one position group's taps)
    d.pair = 127ll * 255 * 257 * s.c_i * s.taps < (1ll << 31) ? 1 : 0;
    d.h = s.h;
    d.npos = std::min(s.pos_tile, 32);  // positions per MMA (N = 8 npos <= 256)
    d.nacc = s.pos_tile / d.npos;       // 64-position tiles use both TMEM buffers
    d.tpos = s.pos_tile * rep;
    d.in_bytes = (size_t)s.n_in * 2 * n * 8;
    d.w_bytes = (size_t)d.OB * d.JB * d.taps * tc::kWTap;
    d.out_bytes = (size_t)s.c_o * s.frags * 2 * n * 8;
    for (int t = 0; t < s.taps; ++t) {
      const int off = s.tap_steps[t] + s.h;
      if (off < 0 || off > 2 * s.h + (ilv ? 1 : 0))
        return fail(FHE_ERR_VALUE, "tc layer %d: tap step outside the halo", l);
      if (ilv) {  // merged taps: column u reads window position 2 u + off = entry u + (off >> 1) of its parity half
        d.tap_off[t] = (int16_t)((off & 1) * (d.npos + s.h) + (off >> 1));
        continue;
      }
      for (int r = 0; r < rep; ++r) d.tap_off[r * s.taps + t] = (int16_t)(off + r * d.npos);  // group r: +32 r
    }
    d.win_bytes = ((d.tpos + 2 * d.h) * 256 + 1023) / 1024 * 1024;
    d.stage_bytes = d.win_bytes + d.taps * tc::kWTap;
    d.nst = std::min(tc::kMaxStages, tc::kRingBudget / d.stage_bytes);
    if (d.nst < 2) return fail(FHE_ERR_VALUE, "tc layer %d: halo too large for the tc path", l);
    // Keep the previous layer's ring partition when this layer's stages fit its
    // slots without losing depth: the loader then streams on without draining
    // the ring at the layer boundary (s3 -> s4 layers, same-shape layers).
    // Resident weights: a layer with one output-channel block and no tap split
    // reuses one weight slab (JB x taps x 4 KB) in every tile; when it fits
    // beside >= 3 window slots it is loaded once per CTA and a stage is just the
    // window (the 7x7 stem: 74 -> 18 KB per tile, 2 -> 6 stages in flight).
    const int wres = d.JB * d.taps * tc::kWTap;
    d.res_bytes = 0;
    if (d.OB == 1 && resident_allowed() && wres + 3 * d.win_bytes <= tc::kRingBudget) {
      d.res_bytes = wres;
      d.slot_bytes = d.win_bytes;
      d.nslots = std::min(tc::kMaxStages, (tc::kRingBudget - wres) / d.win_bytes);
    } else if (l > 0 && !A.L[l - 1].res_bytes && d.stage_bytes <= A.L[l - 1].slot_bytes &&
               A.L[l - 1].nslots >= d.nst && keep_partition()) {
      d.slot_bytes = A.L[l - 1].slot_bytes;
      d.nslots = A.L[l - 1].nslots;
    } else {
      d.slot_bytes = d.stage_bytes;
      d.nslots = d.nst;
    }
    d.tiles = (n / d.tpos) * d.OB * 2 * d.F;
    const size_t xb = (size_t)2 * d.F * d.JB * d.Y * 256;
    d.x_bytes = xb;
    if (x_stride && nl > 1 && xb > x_stride) return fail(FHE_ERR_VALUE, "tc layer %d: X stride smaller than its operand", l);
    xoff += (xb + 255) / 256 * 256;
    const long long units = 2ll * ((d.Y + 31) / 32) * d.JB * 2 * d.F;
    if (units > (1ll << 30)) return fail(FHE_ERR_VALUE, "tc layer %d too large", l);
    d.units = (int)units;
    max_tiles = std::max(max_tiles, d.tiles);
    if (balance_tiles()) {
      // Cost-aware dealing: every CTA gets tiles/G tiles of this layer, the
      // tiles % G extra ones go to a window of consecutive CTAs; place that
      // window where the CTAs' estimated accumulated work is lowest (tile cost:
      // its MMAs, 128 cycles each, or the epilogue's ~3.4k cycles, whichever
      // binds), so the extra tiles of successive big layers do not pile up on
      // the same CTAs and the stack's slowest CTA finishes earlier.
      const int G = sms_now, extra = d.tiles % G;
      const double cost = std::max(128.0 * d.JB * d.taps, 3400.0) + 600.0;
      int best = toff;
      if (extra > 0 && extra < G) {
        double best_max = 1e300;
        for (int st = 0; st < G; ++st) {  // window [st, st + extra) cyclic: its max load
          double mx = 0;
          for (int k = 0; k < extra; ++k) mx = std::max(mx, load[(st + k) % G]);
          if (mx < best_max - 1e-9) {
            best_max = mx;
            best = st;
          }
        }
      }
      d.toff = best;
      for (int b = 0; b < G; ++b) load[b] += cost * (d.tiles / G + (((b - best + G) % G) < extra ? 1 : 0));
    } else {
      d.toff = toff;
      toff = (toff + d.tiles) % sms_now;
    }
    ring = std::max(ring, d.res_bytes + d.nslots * d.slot_bytes);
  }
  ring = std::max(ring, tc::kEpiWarps * tc::kStg);  // the epilogue warps' layer-0 staging lives in the ring
  const size_t smem = (size_t)ring + tc::kRelWarps * tc::kStg + 8 * (2 * tc::kMaxStages + 4) + 4 * tc::kSlotWords +
                      8 * tc::kTq;
  if (!attr_of[dev].load(std::memory_order_acquire)) {  // idempotent: a racing second set is harmless
    FHE_CUDA(cudaFuncSetAttribute(tc::conv_tc_stack_kernel<tc::kMaxLayers>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    FHE_CUDA(cudaFuncSetAttribute(tc::conv_tc_stack_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  227 * 1024));
    attr_of[dev].store(true, std::memory_order_release);
  }
  // persistent and cooperative: every CTA must be resident for the grid barriers
  (void)max_tiles;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(sms_now);
  cfg.blockDim = dim3(tc::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr_coop;
  attr_coop.id = cudaLaunchAttributeCooperative;
  attr_coop.val.cooperative = 1;
  cfg.attrs = &attr_coop;
  cfg.numAttrs = 1;
  if (g_trace_host) {  // trace mode: the launch's tile dealing offsets for tools/trace_stack.py
    static thread_local unsigned long long toffs[tc::kMaxLayers];
    for (int l = 0; l < nl; ++l) toffs[l] = (unsigned long long)A.L[l].toff;
    FHE_CUDA(cudaMemcpyAsync(g_trace_host + 7 * 4096 + 2048, toffs, sizeof(unsigned long long) * nl,
                             cudaMemcpyHostToDevice, (cudaStream_t)stream));
  }
  if (nl == 1) {
    static thread_local tc::StackArgsT<1> A1;
    A1.L[0] = A.L[0];
    A1.sync = A.sync;
    A1.q = A.q;
    A1.w32p = A.w32p;
    A1.n = A.n;
    A1.nl = 1;
    A1.k1 = A.k1;
    A1.k8 = A.k8;
    A1.k16 = A.k16;
    A1.k24 = A.k24;
    A1.xrot = A.xrot;
    A1.dyn = A.dyn;
    A1.pm = A.pm;
    A1.pm_dlo = A.pm_dlo;
    A1.pm_dhi = A.pm_dhi;
    A1.pm_ca = A.pm_ca;
    FHE_CUDA(cudaLaunchKernelEx(&cfg, tc::conv_tc_stack_kernel<1>, A1));
  } else {
    FHE_CUDA(cudaLaunchKernelEx(&cfg, tc::conv_tc_stack_kernel<tc::kMaxLayers>, A));
  }
  FHE_CHECK_LAUNCH("conv_tc_stack_kernel");
  return FHE_OK;
}

int fhe_conv_stream_job(uint64_t q, int n, const fhe_conv_tc_layer* layer, const void* host_in, size_t in_bytes,
                        void* host_out, size_t out_bytes, uint8_t* X, size_t x_stride, uint64_t* sync, void* up,
                        void* comp, void* down, void* ev_up, void* ev_comp) {
  if (!layer || !host_in || !host_out || !ev_up || !ev_comp)  // streams may be 0 (the legacy default stream)
    return fail(FHE_ERR_VALUE, "null stream-job operand");
  cudaStream_t su = (cudaStream_t)up, sc = (cudaStream_t)comp, sd = (cudaStream_t)down;
  FHE_CUDA(cudaMemcpyAsync((void*)layer->in, host_in, in_bytes, cudaMemcpyHostToDevice, su));
  FHE_CUDA(cudaEventRecord((cudaEvent_t)ev_up, su));
  FHE_CUDA(cudaStreamWaitEvent(sc, (cudaEvent_t)ev_up, 0));
  if (int rc = fhe_conv_tc_stack(q, n, layer, 1, X, x_stride, sync, comp)) return rc;
  FHE_CUDA(cudaEventRecord((cudaEvent_t)ev_comp, sc));
  FHE_CUDA(cudaStreamWaitEvent(sd, (cudaEvent_t)ev_comp, 0));
  FHE_CUDA(cudaMemcpyAsync(host_out, layer->out, out_bytes, cudaMemcpyDeviceToHost, sd));
  return FHE_OK;
}

}  // extern "C"
