// conv.cu — K1: the Flash convolution core on the integer pipes (sm_100a).
//
// Reference: conv.conv_proposed / _proposed_channel (conv.py:326-411) with
// _ExtPoly (conv.py:251-266), _CtAccum (conv.py:269-291) and WidePoly
// (ring.py:347-406). Closed form: for output unit u = o*frags+f,
//   out[u][p][s] = ( Σ_k w[o][k] · (in[src_k + f·fs][p] · x^(-step_k))[s] ) mod q
// i.e. an exact integer GEMM over "negacyclic-shifted" input rows, reduced
// once per output coefficient. The reference realises x^(-step) as a slice
// of [-a | a | -a] (q - a on the wrapped parts) and accumulates two 30-bit
// limbs in int64; here the wrapped coefficient is negated in the signed limb
// domain instead. Both are congruent mod q and the single final reduction
// is canonical, so the result is bit-identical.
//
// Kernel shape: a CTA owns an S_TILE-position x O_CTA-channel tile of one
// (poly, fragment). Input terms are staged KCH at a time into shared memory
// as signed (lo31, hi31) limb pairs with the wrap sign folded in; weights as
// int32. Every thread keeps PP x OPW pairs of int64 accumulators and issues
// 2 IMAD.WIDE (mad.wide.s32) per term·position·channel. Global loads of the
// next chunk are in flight (registers) while the current one is consumed.
// One reduction per output: r = (lo mod q) + 2^31 (hi mod q) (Shoup) mod q.
#include "common.cuh"

namespace fhe {

struct ConvArgs {
  const uint64_t* in;
  const int16_t* w;
  const int32_t* tsrc;
  const int32_t* tstep;
  const uint64_t* bias;
  const uint8_t* bmask;
  uint64_t* out;
  ModDesc m;
  uint64_t w31, w31p;  // 2^31 mod q and its Shoup companion
  int n, K, c_o, frags, fstride;
};

template <int WS, int WO, int OPW, int PP, int KCH>
__global__ void __launch_bounds__(WS* WO * 32) conv_flash_kernel(const ConvArgs a) {
  constexpr int NT = WS * WO * 32;
  constexpr int S_TILE = WS * 32 * PP;
  constexpr int O_CTA = WO * OPW;
  constexpr int DITEMS = KCH * S_TILE / NT;
  constexpr int WITEMS = (KCH * O_CTA + NT - 1) / NT;
  static_assert(KCH * S_TILE % NT == 0, "staging split");

  __shared__ int2 sdat[2][KCH][S_TILE];
  __shared__ __align__(16) int32_t swt[2][KCH][O_CTA];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ws = warp % WS, wo = warp / WS;
  const int s0 = blockIdx.x * S_TILE;
  const int o0 = blockIdx.y * O_CTA;
  const int p = blockIdx.z & 1, f = blockIdx.z >> 1;
  const int n = a.n, K = a.K;

  uint64_t pv[DITEMS];
  uint32_t pneg = 0;
  int32_t pw[WITEMS];

  auto prefetch = [&](int c) {
    pneg = 0;
#pragma unroll
    for (int it = 0; it < DITEMS; ++it) {
      const int item = tid + it * NT;
      const int kk = item / S_TILE, sl = item % S_TILE;
      const int k = c * KCH + kk, s = s0 + sl;
      uint64_t v = 0;
      if (k < K && s < n) {
        const int src = __ldg(&a.tsrc[k]) + f * a.fstride;
        int x = s + __ldg(&a.tstep[k]);  // in (-n, 2n)
        int neg = 0;
        if (x < 0) {
          x += n;
          neg = 1;
        } else if (x >= n) {
          x -= n;
          neg = 1;
        }
        v = __ldg(&a.in[((size_t)src * 2 + p) * n + x]);
        pneg |= (uint32_t)neg << it;
      }
      pv[it] = v;
    }
#pragma unroll
    for (int it = 0; it < WITEMS; ++it) {
      const int item = tid + it * NT;
      int32_t wv = 0;
      if (item < KCH * O_CTA) {
        const int kk = item / O_CTA, oo = item % O_CTA;
        const int k = c * KCH + kk, o = o0 + oo;
        if (k < K && o < a.c_o) wv = (int32_t)a.w[(size_t)o * K + k];
      }
      pw[it] = wv;
    }
  };
  auto stage = [&](int buf) {
#pragma unroll
    for (int it = 0; it < DITEMS; ++it) {
      const int item = tid + it * NT;
      const int kk = item / S_TILE, sl = item % S_TILE;
      int32_t lo = (int32_t)(pv[it] & 0x7fffffffull);
      int32_t hi = (int32_t)(pv[it] >> 31);
      if (pneg >> it & 1) {
        lo = -lo;
        hi = -hi;
      }
      sdat[buf][kk][sl] = make_int2(lo, hi);
    }
#pragma unroll
    for (int it = 0; it < WITEMS; ++it) {
      const int item = tid + it * NT;
      if (item < KCH * O_CTA) swt[buf][item / O_CTA][item % O_CTA] = pw[it];
    }
  };

  long long acc_lo[PP][OPW], acc_hi[PP][OPW];
#pragma unroll
  for (int r = 0; r < PP; ++r)
#pragma unroll
    for (int c = 0; c < OPW; ++c) acc_lo[r][c] = acc_hi[r][c] = 0;

  const int nch = (K + KCH - 1) / KCH;
  prefetch(0);
  stage(0);
  __syncthreads();
  for (int c = 0; c < nch; ++c) {
    const int buf = c & 1;
    if (c + 1 < nch) prefetch(c + 1);
#pragma unroll
    for (int kk = 0; kk < KCH; ++kk) {
      int2 d[PP];
#pragma unroll
      for (int r = 0; r < PP; ++r) d[r] = sdat[buf][kk][ws * 32 * PP + lane + 32 * r];
      int32_t wv[OPW];
      if constexpr (OPW % 4 == 0) {
#pragma unroll
        for (int c4 = 0; c4 < OPW / 4; ++c4) {
          const int4 t = *reinterpret_cast<const int4*>(&swt[buf][kk][wo * OPW + 4 * c4]);
          wv[4 * c4 + 0] = t.x;
          wv[4 * c4 + 1] = t.y;
          wv[4 * c4 + 2] = t.z;
          wv[4 * c4 + 3] = t.w;
        }
      } else {
#pragma unroll
        for (int cc = 0; cc < OPW; ++cc) wv[cc] = swt[buf][kk][wo * OPW + cc];
      }
#pragma unroll
      for (int r = 0; r < PP; ++r)
#pragma unroll
        for (int cc = 0; cc < OPW; ++cc) {
          acc_lo[r][cc] += (long long)wv[cc] * d[r].x;  // mad.wide.s32
          acc_hi[r][cc] += (long long)wv[cc] * d[r].y;
        }
    }
    if (c + 1 < nch) stage(buf ^ 1);
    __syncthreads();
  }

  // epilogue: one canonical reduction per coefficient (WidePoly.finalize)
  const uint64_t q = a.m.q;
#pragma unroll
  for (int cc = 0; cc < OPW; ++cc) {
    const int o = o0 + wo * OPW + cc;
    if (o >= a.c_o) continue;
    const size_t orow = ((size_t)(o * a.frags + f) * 2 + p) * n;
    const uint64_t bd = (p == 0 && a.bias) ? a.bias[o] : 0;
#pragma unroll
    for (int r = 0; r < PP; ++r) {
      const int s = s0 + ws * 32 * PP + lane + 32 * r;
      if (s >= n) continue;
      const uint64_t lo = reduce_i64(acc_lo[r][cc], a.m);
      const uint64_t hi = reduce_i64(acc_hi[r][cc], a.m);
      uint64_t v = csub(lo + csub(shoup_lazy(hi, a.w31, a.w31p, q), q), q);
      if (bd && a.bmask[(size_t)f * n + s]) v = csub(v + bd, q);
      a.out[orow + s] = v;
    }
  }
}

template <int WS, int WO, int OPW, int PP, int KCH>
static int launch_conv(const ConvArgs& a, cudaStream_t st) {
  constexpr int S_TILE = WS * 32 * PP;
  constexpr int O_CTA = WO * OPW;
  dim3 grid((a.n + S_TILE - 1) / S_TILE, (a.c_o + O_CTA - 1) / O_CTA, 2 * a.frags);
  conv_flash_kernel<WS, WO, OPW, PP, KCH><<<grid, WS * WO * 32, 0, st>>>(a);
  FHE_CHECK_LAUNCH("conv_flash_kernel");
  return FHE_OK;
}

}  // namespace fhe

using namespace fhe;

extern "C" int fhe_conv_flash(uint64_t q, int n, const uint64_t* in, int n_in, const int16_t* weights,
                              int c_o, int K, const int32_t* term_src, const int32_t* term_step,
                              int frags, int frag_stride, const uint64_t* bias_delta,
                              const uint8_t* bias_mask, uint64_t* out, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (n < 2 || (n & (n - 1))) return fail(FHE_ERR_VALUE, "n must be a power of two");
  if (c_o < 0 || K < 0 || frags < 1 || n_in < 0) return fail(FHE_ERR_VALUE, "bad conv geometry");
  if (K > 0 && (!in || !weights || !term_src || !term_step)) return fail(FHE_ERR_VALUE, "null conv operand");
  if (bias_delta && !bias_mask) return fail(FHE_ERR_VALUE, "bias needs a mask");
  if ((int64_t)c_o * frags * 2 * n >= ((int64_t)1 << 40)) return fail(FHE_ERR_VALUE, "output too large");
  if (c_o == 0) return FHE_OK;
  ConvArgs a;
  a.in = in;
  a.w = weights;
  a.tsrc = term_src;
  a.tstep = term_step;
  a.bias = bias_delta;
  a.bmask = bias_mask;
  a.out = out;
  a.m = ms.m[0];
  a.w31 = (1ull << 31) % q;
  a.w31p = h_shoup(a.w31, q);
  a.n = n;
  a.K = K;
  a.c_o = c_o;
  a.frags = frags;
  a.fstride = frag_stride;
  cudaStream_t st = (cudaStream_t)stream;
  if (c_o >= 64) return launch_conv<1, 8, 8, 4, 8>(a, st);
  if (c_o >= 16) return launch_conv<4, 2, 8, 4, 4>(a, st);
  if (c_o >= 8) return launch_conv<8, 1, 8, 2, 4>(a, st);
  return launch_conv<8, 1, 1, 2, 4>(a, st);
}

// ---------------------------------------------------------------------------
// K1 pooling: conv.avg_pool (conv.py:604-623) sums the k x k window of every
// slot through k² DRot taps of weight 1. The sum is exact mod q in any order,
// so it is computed separably — k row taps into a staged row sum, then k
// column taps of that sum (2k modular adds per slot instead of k²) — one
// polynomial row per CTA, staged in shared memory. Identical ciphertexts to
// the k²-tap contraction.
namespace fhe {

__global__ void __launch_bounds__(256) avg_pool_kernel(uint64_t q, int n, int k, int w_p,
                                                       const uint64_t* __restrict__ in,
                                                       uint64_t* __restrict__ out) {
  extern __shared__ uint64_t pool_sm[];
  uint64_t* a = pool_sm;      // the row
  uint64_t* hs = pool_sm + n;  // row sums h[i] = Σ_dx A(i + dx), i < n
  const size_t row = blockIdx.x;
  const uint64_t* src = in + row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = src[i];
  __syncthreads();
  // A(j) = a[j] (j < n), -a[j - n] (n <= j < 2n): the negacyclic extension
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint64_t s = 0;
    for (int dx = 0; dx < k; ++dx) {
      const int j = i + dx;
      const uint64_t v = j < n ? a[j] : (a[j - n] ? q - a[j - n] : 0);
      s = csub(s + v, q);
    }
    hs[i] = s;
  }
  __syncthreads();
  uint64_t* dst = out + row * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    uint64_t s = 0;
    for (int dy = 0; dy < k; ++dy) {
      const int j = i + dy * w_p;  // H(j) = h[j] or -h[j - n]: every term of h[j - n + ...] wrapped
      const uint64_t v = j < n ? hs[j] : (hs[j - n] ? q - hs[j - n] : 0);
      s = csub(s + v, q);
    }
    dst[i] = s;
  }
}

}  // namespace fhe

extern "C" int fhe_avg_pool(uint64_t q, int n, int rows, int k, int w_p, const uint64_t* in, uint64_t* out,
                            void* stream) {
  if (n < 2 || (n & (n - 1)) || n > 8192) return fail(FHE_ERR_VALUE, "pool needs a power-of-two n <= 8192");
  if (q < 2 || q >= (1ull << 62)) return fail(FHE_ERR_PARAMETER, "modulus out of range");
  if (rows < 0 || k < 1 || w_p < 1) return fail(FHE_ERR_VALUE, "bad pool geometry");
  if ((int64_t)(k - 1) * (w_p + 1) >= n) return fail(FHE_ERR_VALUE, "pool window must stay within one wrap");
  if (!rows) return FHE_OK;
  if (!in || !out || in == out) return fail(FHE_ERR_VALUE, "bad pool buffers");
  const size_t smem = (size_t)2 * n * sizeof(uint64_t);
  if (smem > 48 * 1024)
    FHE_CUDA(cudaFuncSetAttribute(fhe::avg_pool_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  fhe::avg_pool_kernel<<<rows, 256, smem, (cudaStream_t)stream>>>(q, n, k, w_p, in, out);
  FHE_CHECK_LAUNCH("avg_pool_kernel");
  return FHE_OK;
}
