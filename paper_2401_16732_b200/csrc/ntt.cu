// ntt.cu — K2: batched negacyclic NTT / iNTT over RNS limbs (sm_100a).
//
// Replaces ring.NttPlan.fwd / inv (ring.py:129-162), which run one big-int
// (`object`) butterfly pass per stage. Semantics kept exactly: forward is
// Cooley-Tukey with merged twiddles psi_brv[m + j] (natural order in,
// bit-reversed out), inverse is Gentleman-Sande with ipsi_brv[h + j] then
// x n^-1. Values are canonical [0, q) at the boundary, so the lazy internal
// ranges ([0,4q) forward, [0,2q) inverse, Harvey 2014) are invisible.
//
// One CTA owns one polynomial (n <= 16384 -> <= 139 KB of shared memory).
// Stages are grouped in phases of up to LOGR stages: each thread pulls
// 2^LOGR coefficients (stride t_min) from shared memory into registers, runs
// the phase's butterflies register-resident (one 128-bit twiddle load per
// distinct twiddle), and writes them back — log2(n)/LOGR shared-memory round
// trips instead of log2(n). Global traffic is one coalesced 128-bit read and
// one write per coefficient (the HBM roofline of 16 B/coefficient).
// The padding x + x/16 keeps the 64-bit shared accesses at the 2-wavefront
// minimum for every phase stride.
#include <atomic>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace fhe {

__host__ __device__ __forceinline__ int spad(int x) { return x + (x >> 4); }

struct LoadMap {
  const uint64_t* src;
  int G;        // rows per limb group in the OUTPUT indexing (P, or ndig)
  int ndig;     // 0 = plain (src row == out row); >0 = digit mode
  int T;        // digit width
  int pad_;
  uint64_t mask;
};

template <int I, int N, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < N) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, N>(f);
  }
}

// One forward phase: stages [s, s+R) (half-sizes t_min*2^(R-1) .. t_min).
template <int LOGR, int R>
__device__ __forceinline__ void fwd_phase(uint64_t* sm, const NttDesc& d, int s, int tid, int nthr) {
  const int n = d.n, logn = d.logn;
  const uint64_t q = d.m.q, q2 = 2 * q;
  const int tl = logn - (s + R);  // log2 t_min
  const int items = n >> LOGR;
  for (int w = tid; w < items; w += nthr) {
    const int base = ((w >> tl) << (tl + LOGR)) + (w & ((1 << tl) - 1));
    uint64_t e[1 << LOGR];
#pragma unroll
    for (int i = 0; i < (1 << LOGR); ++i) e[i] = sm[spad(base + (i << tl))];
    static_for<0, R>([&](auto ai) {
      constexpr int a = R - 1 - decltype(ai)::value;  // largest stride first
      constexpr int dd = 1 << a;
      const int sh = tl + a + 1;                      // = logn - stage
#pragma unroll
      for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
        const ulonglong2 tw = __ldg(&d.psi[(n + base + (g << tl)) >> sh]);
#pragma unroll
        for (int u = 0; u < dd; ++u) {
          uint64_t X = e[g + u];
          X = X >= q2 ? X - q2 : X;
          const uint64_t T = shoup_lazy(e[g + u + dd], tw.x, tw.y, q);
          e[g + u] = X + T;
          e[g + u + dd] = X - T + q2;
        }
      }
    });
#pragma unroll
    for (int i = 0; i < (1 << LOGR); ++i) sm[spad(base + (i << tl))] = e[i];
  }
}

// One inverse phase: stages [s, s+R) processed smallest half-size first.
template <int LOGR, int R>
__device__ __forceinline__ void inv_phase(uint64_t* sm, const NttDesc& d, int s, int tid, int nthr) {
  const int n = d.n, logn = d.logn;
  const uint64_t q = d.m.q, q2 = 2 * q;
  const int tl = logn - (s + R);
  const int items = n >> LOGR;
  const bool last = (s == 0);
  for (int w = tid; w < items; w += nthr) {
    const int base = ((w >> tl) << (tl + LOGR)) + (w & ((1 << tl) - 1));
    uint64_t e[1 << LOGR];
#pragma unroll
    for (int i = 0; i < (1 << LOGR); ++i) e[i] = sm[spad(base + (i << tl))];
    static_for<0, R>([&](auto ai) {
      constexpr int a = decltype(ai)::value;
      constexpr int dd = 1 << a;
      const int sh = tl + a + 1;
      if (last && a == R - 1) {  // stage 0: fold n^-1 (ring.py:162)
#pragma unroll
        for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
#pragma unroll
          for (int u = 0; u < dd; ++u) {
            const uint64_t X = e[g + u], Y = e[g + u + dd];
            e[g + u] = shoup_lazy(X + Y, d.ninv.x, d.ninv.y, q);
            e[g + u + dd] = shoup_lazy(X - Y + q2, d.ninv_w1.x, d.ninv_w1.y, q);
          }
        }
      } else {
#pragma unroll
        for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
          const ulonglong2 tw = __ldg(&d.ipsi[(n + base + (g << tl)) >> sh]);
#pragma unroll
          for (int u = 0; u < dd; ++u) {
            const uint64_t X = e[g + u], Y = e[g + u + dd];
            const uint64_t S = X + Y;
            e[g + u] = S >= q2 ? S - q2 : S;
            e[g + u + dd] = shoup_lazy(X - Y + q2, tw.x, tw.y, q);
          }
        }
      }
    });
#pragma unroll
    for (int i = 0; i < (1 << LOGR); ++i) sm[spad(base + (i << tl))] = e[i];
  }
}

template <int LOGR, bool INV, int R>
__device__ __forceinline__ void run_phase(uint64_t* sm, const NttDesc& d, int s, int tid, int nthr) {
  if constexpr (INV)
    inv_phase<LOGR, R>(sm, d, s, tid, nthr);
  else
    fwd_phase<LOGR, R>(sm, d, s, tid, nthr);
}

template <int LOGR, bool INV>
__device__ __forceinline__ void run_partial(uint64_t* sm, const NttDesc& d, int s, int r, int tid,
                                            int nthr) {
  static_for<1, LOGR>([&](auto ri) {
    constexpr int R = decltype(ri)::value;
    if (r == R) run_phase<LOGR, INV, R>(sm, d, s, tid, nthr);
  });
}

template <int LOGR, bool INV>
__global__ void __launch_bounds__(512) ntt_kernel(const LimbSet ls, const LoadMap lm,
                                                  uint64_t* __restrict__ dst) {
  extern __shared__ uint64_t sm[];
  const int row = blockIdx.x;
  const int limb = (row / lm.G) % ls.L;
  const NttDesc d = ls.d[limb];
  const int n = d.n, logn = d.logn;
  const int tid = threadIdx.x, nthr = blockDim.x;

  const uint64_t* srow;
  int shift = 0;
  if (lm.ndig > 0) {
    srow = lm.src + (size_t)(row / lm.ndig) * n;
    shift = lm.T * (row % lm.ndig);
  } else {
    srow = lm.src + (size_t)row * n;
  }
  const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(srow);
  for (int i = tid; i < (n >> 1); i += nthr) {
    ulonglong2 v = s2[i];
    if (lm.ndig > 0) {
      v.x = (v.x >> shift) & lm.mask;
      v.y = (v.y >> shift) & lm.mask;
    }
    sm[spad(2 * i)] = v.x;
    sm[spad(2 * i + 1)] = v.y;
  }
  __syncthreads();

  const int nfull = logn / LOGR, rem = logn - nfull * LOGR;
  if (!INV) {
    for (int p = 0; p < nfull; ++p) {
      run_phase<LOGR, false, LOGR>(sm, d, p * LOGR, tid, nthr);
      __syncthreads();
    }
    if (rem) {
      run_partial<LOGR, false>(sm, d, nfull * LOGR, rem, tid, nthr);
      __syncthreads();
    }
  } else {
    if (rem) {
      run_partial<LOGR, true>(sm, d, nfull * LOGR, rem, tid, nthr);
      __syncthreads();
    }
    for (int p = nfull - 1; p >= 0; --p) {
      run_phase<LOGR, true, LOGR>(sm, d, p * LOGR, tid, nthr);
      __syncthreads();
    }
  }

  const uint64_t q = d.m.q, q2 = 2 * q;
  ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst + (size_t)row * n);
  for (int i = tid; i < (n >> 1); i += nthr) {
    uint64_t x = sm[spad(2 * i)], y = sm[spad(2 * i + 1)];
    if (!INV) {
      x = x >= q2 ? x - q2 : x;
      y = y >= q2 ? y - q2 : y;
    }
    d2[i] = make_ulonglong2(csub(x, q), csub(y, q));
  }
}

// ---------------------------------------------------------------------------
// Split transform for n >= 8192 (n = 2^a · 2^b): the first a Cooley-Tukey
// stages only mix elements i = i1·2^b + i2 with equal i2 (length-2^a
// transforms down the columns), the last b stages only mix elements of one
// contiguous 2^b block. With the merged twiddles psi_brv the column transforms
// all use psi[(2^a + i1) >> (a - s)] and block k's use
// psi[(((2^a + k) << b) + i2) >> (b - s')], so the transform splits into two
// launches with no twiddle pass and no transpose — each over small CTAs
// (16 columns or 16 blocks, ~17 KB of shared memory) that keep every SM busy
// and overlap memory with butterflies. The inverse runs the same two
// launches in the opposite order (GS, n^-1 folded into stage 0). Values stay
// lazy ([0,4q) / [0,2q)) between the launches; the second one canonicalises.
constexpr int kSplitW = 16;  // columns (first launch) or blocks (second launch) per CTA
constexpr int kSplitMinLog = 13;

static bool split_enabled() {  // FHE_NTT_SPLIT=0 selects the one-CTA-per-row kernel (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_NTT_SPLIT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Register budget of the split kernels: __launch_bounds__(256, MINB) caps them
// at 64K / (256 MINB) registers. MINB = 3 (85 registers, 6 resident 128-thread
// CTAs = 24 warps per SM) measured 7 % faster than the unconstrained 106-120
// registers (4 CTAs) on N = 16384; FHE_NTT_MINB = 1 selects the unconstrained
// variant for A/B checks.
static int split_minb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_NTT_MINB");
    v = e ? atoi(e) : 3;
  }
  return v;
}

// Element i of a phase item sits at a compile-time offset from the item's
// base slot: columns are interleaved (slot = e * kSplitW + v), blocks are
// padded (slot = v * (len + len/16) + e + e/16, 2-wavefront 64-bit accesses
// for every stride); with B the item's first element and (i << TL) a multiple
// of 2^TL, spad(B + (i << TL)) = spad(B) + (i << TL) + ((i << TL) >> 4).
template <bool COLS, int TL>
__device__ __forceinline__ constexpr int elem_off(int i) {
  return COLS ? (i << TL) * kSplitW : (i << TL) + ((i << TL) >> 4);
}

// One phase of R stages on 2^LOGR register-resident elements. tb = O + B: the
// merged-twiddle index of the item's first element; the group of g reads
// psi[(tb + (g << TL)) >> (TL + a + 1)] = psi[(tb >> sh) + (g >> (a + 1))]
// (g << TL is a multiple of 2^sh), so every index is one shift plus a constant.
template <int LOGR, int R, bool INV, bool COLS, int TL>
__device__ __forceinline__ void split_phase(uint64_t* __restrict__ p, const NttDesc& d, uint32_t tb,
                                            bool fold_ninv) {
  const uint64_t q = d.m.q, q2 = 2 * q;
  uint64_t e[1 << LOGR];
#pragma unroll
  for (int i = 0; i < (1 << LOGR); ++i) e[i] = p[elem_off<COLS, TL>(i)];
  if constexpr (!INV) {
    static_for<0, R>([&](auto ai) {
      constexpr int a = R - 1 - decltype(ai)::value;  // largest stride first
      constexpr int dd = 1 << a;
      const uint32_t t0 = tb >> (TL + a + 1);
#pragma unroll
      for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
        const ulonglong2 tw = __ldg(&d.psi[t0 + (g >> (a + 1))]);
#pragma unroll
        for (int u = 0; u < dd; ++u) {
          uint64_t X = e[g + u];
          X = X >= q2 ? X - q2 : X;
          const uint64_t T = shoup_lazy(e[g + u + dd], tw.x, tw.y, q);
          e[g + u] = X + T;
          e[g + u + dd] = X - T + q2;
        }
      }
    });
  } else {
    static_for<0, R>([&](auto ai) {
      constexpr int a = decltype(ai)::value;  // smallest stride first
      constexpr int dd = 1 << a;
      if (fold_ninv && a == R - 1) {  // global stage 0: fold n^-1 (ring.py:162)
#pragma unroll
        for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
#pragma unroll
          for (int u = 0; u < dd; ++u) {
            const uint64_t X = e[g + u], Y = e[g + u + dd];
            e[g + u] = shoup_lazy(X + Y, d.ninv.x, d.ninv.y, q);
            e[g + u + dd] = shoup_lazy(X - Y + q2, d.ninv_w1.x, d.ninv_w1.y, q);
          }
        }
      } else {
        const uint32_t t0 = tb >> (TL + a + 1);
#pragma unroll
        for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
          const ulonglong2 tw = __ldg(&d.ipsi[t0 + (g >> (a + 1))]);
#pragma unroll
          for (int u = 0; u < dd; ++u) {
            const uint64_t X = e[g + u], Y = e[g + u + dd];
            const uint64_t S = X + Y;
            e[g + u] = S >= q2 ? S - q2 : S;
            e[g + u + dd] = shoup_lazy(X - Y + q2, tw.x, tw.y, q);
          }
        }
      }
    });
  }
#pragma unroll
  for (int i = 0; i < (1 << LOGR); ++i) p[elem_off<COLS, TL>(i)] = e[i];
}

// all LG stages of this thread's sub-transform v (LOGR-stage phases)
template <int LOGR, bool INV, bool COLS, int LG>
__device__ __forceinline__ void split_sub(uint64_t* sm, int v, int item, const NttDesc& d, uint32_t O, bool fold_ninv) {
  constexpr int nfull = LG / LOGR, rem = LG - nfull * LOGR;
  constexpr int len = 1 << LG;
  auto phase = [&](auto s_c, auto r_c) {
    constexpr int S = decltype(s_c)::value, R = decltype(r_c)::value;
    constexpr int TL = LG - (S + R);
    const int B = ((item >> TL) << (TL + LOGR)) + (item & ((1 << TL) - 1));
    uint64_t* p = COLS ? sm + B * kSplitW + v : sm + v * (len + len / 16) + spad(B);
    split_phase<LOGR, R, INV, COLS, TL>(p, d, O + (uint32_t)B, fold_ninv && S == 0);
  };
  if constexpr (!INV) {
    static_for<0, nfull>([&](auto pi) {
      phase(std::integral_constant<int, decltype(pi)::value * LOGR>{}, std::integral_constant<int, LOGR>{});
      __syncthreads();
    });
    if constexpr (rem > 0) {
      phase(std::integral_constant<int, nfull * LOGR>{}, std::integral_constant<int, rem>{});
      __syncthreads();
    }
  } else {
    if constexpr (rem > 0) {
      phase(std::integral_constant<int, nfull * LOGR>{}, std::integral_constant<int, rem>{});
      __syncthreads();
    }
    static_for<0, nfull>([&](auto pi) {
      phase(std::integral_constant<int, (nfull - 1 - decltype(pi)::value) * LOGR>{},
            std::integral_constant<int, LOGR>{});
      __syncthreads();
    });
  }
}

// COLS: this CTA = row, columns [c0, c0 + 16): stages [0, a), LG = a.
// !COLS: this CTA = row, blocks [k0, k0 + 16): stages [a, a + b), LG = b.
// from_src: read through the LoadMap (first launch) else read dst in place;
// final: canonical [0,q) output (second launch).
template <int LOGR, bool INV, bool COLS, int MINB, int LG>
__global__ void __launch_bounds__(256, MINB) ntt_split_kernel(const LimbSet ls, const LoadMap lm, uint64_t* __restrict__ dst,
                                                              int a, int b, int from_src, int final_) {
  extern __shared__ uint64_t sm[];
  constexpr int len = 1 << LG;
  const int per_row = COLS ? (1 << b) / kSplitW : (1 << a) / kSplitW;
  const int row = blockIdx.x / per_row, part = blockIdx.x % per_row;
  const int limb = (row / lm.G) % ls.L;
  const NttDesc d = ls.d[limb];
  const int n = d.n;
  const int tid = threadIdx.x;
  const uint64_t* srow;
  int shift = 0;
  if (from_src) {
    if (lm.ndig > 0) {
      srow = lm.src + (size_t)(row / lm.ndig) * n;
      shift = lm.T * (row % lm.ndig);
    } else {
      srow = lm.src + (size_t)row * n;
    }
  } else {
    srow = dst + (size_t)row * n;
  }
  uint64_t* drow = dst + (size_t)row * n;
  const uint64_t mask = (from_src && lm.ndig > 0) ? lm.mask : ~0ull;
  // element (e, v): e = position in the sub-transform, v = column / block in this CTA
  auto gidx = [&](int e, int v) -> size_t {
    return COLS ? (size_t)e * (1 << b) + part * kSplitW + v : (size_t)(part * kSplitW + v) * len + e;
  };
  auto sidx = [&](int e, int v) -> int { return COLS ? e * kSplitW + v : v * (len + len / 16) + spad(e); };
  // load (pairs of consecutive elements: columns for COLS, positions for blocks):
  // the thread count is a compile-time constant (kSplitW sub-transforms x
  // len / 2^LOGR items), so all NP pair loads are issued before the first
  // shared-memory store
  constexpr int NT = kSplitW * (len >> LOGR), NP = (len * kSplitW / 2) / NT;
  ulonglong2 xin[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int i = tid + k * NT;
    const int e = COLS ? (2 * i) / kSplitW : (2 * i) % len, v = COLS ? (2 * i) % kSplitW : (2 * i) / len;
    xin[k] = *reinterpret_cast<const ulonglong2*>(srow + gidx(e, v));
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int i = tid + k * NT;
    const int e = COLS ? (2 * i) / kSplitW : (2 * i) % len, v = COLS ? (2 * i) % kSplitW : (2 * i) / len;
    ulonglong2 x = xin[k];
    if (from_src && lm.ndig > 0) {
      x.x = (x.x >> shift) & mask;
      x.y = (x.y >> shift) & mask;
    }
    if (COLS) {
      sm[sidx(e, v)] = x.x;
      sm[sidx(e, v + 1)] = x.y;
    } else {
      sm[sidx(e, v)] = x.x;
      sm[sidx(e + 1, v)] = x.y;
    }
  }
  __syncthreads();
  // one item per thread: (v, phase item)
  constexpr int ipv = len >> LOGR;  // phase items per sub-transform
  const int v = COLS ? tid % kSplitW : tid / ipv;
  const int item = COLS ? tid / kSplitW : tid % ipv;
  const uint32_t O = COLS ? (uint32_t)len : (uint32_t)((1 << a) + part * kSplitW + v) << b;
  split_sub<LOGR, INV, COLS, LG>(sm, v, item, d, O, INV && COLS);
  // store: all NP pairs read from shared memory, then written
  const uint64_t q = d.m.q, q2 = 2 * q;
  ulonglong2 xo[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int i = tid + k * NT;
    const int e = COLS ? (2 * i) / kSplitW : (2 * i) % len, vv = COLS ? (2 * i) % kSplitW : (2 * i) / len;
    uint64_t x = sm[sidx(e, vv)];
    uint64_t y = COLS ? sm[sidx(e, vv + 1)] : sm[sidx(e + 1, vv)];
    if (final_) {
      if (!INV) {
        x = x >= q2 ? x - q2 : x;
        y = y >= q2 ? y - q2 : y;
      }
      x = csub(x, q);
      y = csub(y, q);
    }
    xo[k] = make_ulonglong2(x, y);
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int i = tid + k * NT;
    const int e = COLS ? (2 * i) / kSplitW : (2 * i) % len, vv = COLS ? (2 * i) % kSplitW : (2 * i) / len;
    *reinterpret_cast<ulonglong2*>(drow + gidx(e, vv)) = xo[k];
  }
}

template <int LOGR, bool INV, bool COLS, int MINB, int LG>
static void launch_split_k(const LimbSet& ls, const LoadMap& lm, uint64_t* dst, int grid, int threads, size_t smem,
                           int a, int b, int from_src, int final_, cudaStream_t st) {
  ntt_split_kernel<LOGR, INV, COLS, MINB, LG><<<grid, threads, smem, st>>>(ls, lm, dst, a, b, from_src, final_);
}

// One CTA per row for 2^LOGN <= 4096 with the split kernels' compile-time
// phase geometry (the whole row is one "block": O = n, v = 0): one item per
// thread per phase, element slots and twiddle indices as base + constant.
template <bool INV, int LOGN, int LOGR>
__global__ void __launch_bounds__((1 << LOGN) >> LOGR) ntt_row_kernel(const LimbSet ls, const LoadMap lm,
                                                                   uint64_t* __restrict__ dst) {
  extern __shared__ uint64_t sm[];
  constexpr int n = 1 << LOGN;
  const int row = blockIdx.x;
  const NttDesc d = ls.d[(row / lm.G) % ls.L];
  const int tid = threadIdx.x;
  const uint64_t* srow;
  int shift = 0;
  if (lm.ndig > 0) {
    srow = lm.src + (size_t)(row / lm.ndig) * n;
    shift = lm.T * (row % lm.ndig);
  } else {
    srow = lm.src + (size_t)row * n;
  }
  const ulonglong2* s2 = reinterpret_cast<const ulonglong2*>(srow);
  constexpr int NT = n >> LOGR, NP = (n / 2) / NT;  // n/2 pairs over n/2^LOGR threads
  ulonglong2 xin[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) xin[k] = s2[tid + k * NT];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int i = tid + k * NT;
    ulonglong2 v = xin[k];
    if (lm.ndig > 0) {
      v.x = (v.x >> shift) & lm.mask;
      v.y = (v.y >> shift) & lm.mask;
    }
    sm[spad(2 * i)] = v.x;
    sm[spad(2 * i + 1)] = v.y;
  }
  __syncthreads();
  split_sub<LOGR, INV, false, LOGN>(sm, 0, tid, d, (uint32_t)n, INV);
  const uint64_t q = d.m.q, q2 = 2 * q;
  ulonglong2* d2 = reinterpret_cast<ulonglong2*>(dst + (size_t)row * n);
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    const int i = tid + k * NT;
    uint64_t x = sm[spad(2 * i)], y = sm[spad(2 * i + 1)];
    if (!INV) {
      x = x >= q2 ? x - q2 : x;
      y = y >= q2 ? y - q2 : y;
    }
    xin[k] = make_ulonglong2(csub(x, q), csub(y, q));
  }
#pragma unroll
  for (int k = 0; k < NP; ++k) d2[tid + k * NT] = xin[k];
}

// Butterflies of one phase on register-resident elements (the math of
// split_phase without its shared-memory load / store).
template <int LOGR, int R, bool INV, int TL>
__device__ __forceinline__ void phase_math(uint64_t (&e)[1 << LOGR], const NttDesc& d, uint32_t tb, bool fold_ninv) {
  const uint64_t q = d.m.q, q2 = 2 * q;
  if constexpr (!INV) {
    static_for<0, R>([&](auto ai) {
      constexpr int a = R - 1 - decltype(ai)::value;  // largest stride first
      constexpr int dd = 1 << a;
      const uint32_t t0 = tb >> (TL + a + 1);
#pragma unroll
      for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
        const ulonglong2 tw = __ldg(&d.psi[t0 + (g >> (a + 1))]);
#pragma unroll
        for (int u = 0; u < dd; ++u) {
          uint64_t X = e[g + u];
          X = X >= q2 ? X - q2 : X;
          const uint64_t T = shoup_lazy(e[g + u + dd], tw.x, tw.y, q);
          e[g + u] = X + T;
          e[g + u + dd] = X - T + q2;
        }
      }
    });
  } else {
    static_for<0, R>([&](auto ai) {
      constexpr int a = decltype(ai)::value;  // smallest stride first
      constexpr int dd = 1 << a;
      if (fold_ninv && a == R - 1) {  // global stage 0: fold n^-1 (ring.py:162)
#pragma unroll
        for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
#pragma unroll
          for (int u = 0; u < dd; ++u) {
            const uint64_t X = e[g + u], Y = e[g + u + dd];
            e[g + u] = shoup_lazy(X + Y, d.ninv.x, d.ninv.y, q);
            e[g + u + dd] = shoup_lazy(X - Y + q2, d.ninv_w1.x, d.ninv_w1.y, q);
          }
        }
      } else {
        const uint32_t t0 = tb >> (TL + a + 1);
#pragma unroll
        for (int g = 0; g < (1 << LOGR); g += 2 * dd) {
          const ulonglong2 tw = __ldg(&d.ipsi[t0 + (g >> (a + 1))]);
#pragma unroll
          for (int u = 0; u < dd; ++u) {
            const uint64_t X = e[g + u], Y = e[g + u + dd];
            const uint64_t S = X + Y;
            e[g + u] = S >= q2 ? S - q2 : S;
            e[g + u + dd] = shoup_lazy(X - Y + q2, tw.x, tw.y, q);
          }
        }
      }
    });
  }
}

// Phase K of a LOGN-point transform in execution order: forward runs the
// stage groups [0, LOGR), [LOGR, 2 LOGR), ..., [nfull LOGR, LOGN); the inverse
// runs them in reverse.
template <int LOGN, int LOGR, bool INV, int K>
struct RowPhase {
  static constexpr int nfull = LOGN / LOGR, rem = LOGN - nfull * LOGR, count = nfull + (rem > 0);
  static constexpr int fk = INV ? count - 1 - K : K;
  static constexpr int S = fk * LOGR;
  static constexpr int R = fk < nfull ? LOGR : rem;
  static constexpr int TL = LOGN - (S + R);
};

// One CTA per row, the first phase's elements loaded straight from global
// memory into registers (a warp's load i reads 32 consecutive words, or each
// thread's 2^LOGR contiguous words as 128-bit loads when the phase's stride is
// 1) and the last phase's results stored straight from registers: two
// shared-memory passes and two barriers fewer than staging the row through
// shared memory at both ends. n = 2048: 3 phases, 2 shared-memory exchanges.
// Row kernels: enough resident CTAs per SM for 1024 threads, i.e. a 64-register cap
// (n = 2048: 4 CTAs; fused decryption of 5120 rows 254 -> 228 us, row NTT unchanged)
// (radix 16 keeps 16 values per thread: half the CTAs, a 128-register cap)
#define FHE_ROW_MINB(T, LOGR) ((LOGR) >= 4 ? ((T) < 512 ? 512 / (T) : 1) : ((T) < 1024 ? 1024 / (T) : 1))
template <bool INV, int LOGN, int LOGR>
__global__ void __launch_bounds__((1 << LOGN) >> LOGR, FHE_ROW_MINB((1 << LOGN) >> LOGR, LOGR)) ntt_row_direct_kernel(const LimbSet ls, const LoadMap lm,
                                                                          uint64_t* __restrict__ dst) {
  extern __shared__ uint64_t sm[];
  constexpr int n = 1 << LOGN, E = 1 << LOGR;
  constexpr int NPH = RowPhase<LOGN, LOGR, INV, 0>::count;
  const int row = blockIdx.x;
  const NttDesc d = ls.d[(row / lm.G) % ls.L];
  const int item = threadIdx.x;
  const uint64_t* srow;
  int shift = 0;
  uint64_t mask = ~0ull;
  if (lm.ndig > 0) {
    srow = lm.src + (size_t)(row / lm.ndig) * n;
    shift = lm.T * (row % lm.ndig);
    mask = lm.mask;
  } else {
    srow = lm.src + (size_t)row * n;
  }
  uint64_t* drow = dst + (size_t)row * n;
  const uint64_t q = d.m.q, q2 = 2 * q;
  static_for<0, NPH>([&](auto kc) {
    constexpr int K = decltype(kc)::value;
    using Ph = RowPhase<LOGN, LOGR, INV, K>;
    constexpr int TL = Ph::TL;
    const int B = ((item >> TL) << (TL + LOGR)) + (item & ((1 << TL) - 1));
    uint64_t e[E];
    if constexpr (K == 0) {
      if constexpr (TL == 0) {
#pragma unroll
        for (int i = 0; i < E; i += 2) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(srow + B + i);
          e[i] = (v.x >> shift) & mask;
          e[i + 1] = (v.y >> shift) & mask;
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) e[i] = (srow[B + (i << TL)] >> shift) & mask;
      }
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) e[i] = sm[spad(B) + (i << TL) + ((i << TL) >> 4)];
    }
    phase_math<LOGR, Ph::R, INV, TL>(e, d, (uint32_t)(n + B), INV && Ph::S == 0);
    if constexpr (K == NPH - 1) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        uint64_t x = e[i];
        if (!INV) x = x >= q2 ? x - q2 : x;
        e[i] = csub(x, q);
      }
      if constexpr (TL == 0) {
#pragma unroll
        for (int i = 0; i < E; i += 2)
          *reinterpret_cast<ulonglong2*>(drow + B + i) = make_ulonglong2(e[i], e[i + 1]);
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) drow[B + (i << TL)] = e[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) sm[spad(B) + (i << TL) + ((i << TL) >> 4)] = e[i];
      __syncthreads();
    }
  });
}

// K6 fused (the client's decryption of a batch, bfv.py:278-293): one CTA per
// ciphertext computes [c1·s + c0]_q and rounds it to the message in one pass —
// NTT(c1) (forward phases), · s in registers, the inverse phases (the forward
// transform's last phase and the inverse's first share their register
// positions, so no shared-memory trip between them), + c0, then round(u/Δ)
// mod p with the residual folded into max_all. EVAL ciphertexts skip the
// forward transform: (c1·s + c0) is formed in registers before the inverse.
// Replaces the 7-launch chain (two column copies, NTT, ·s, iNTT, + c0, round)
// with one launch; values are identical (every step is exact mod q).
template <int LOGN, int LOGR, bool EVAL>
__global__ void __launch_bounds__((1 << LOGN) >> LOGR, FHE_ROW_MINB((1 << LOGN) >> LOGR, LOGR)) decrypt_fused_kernel(
    const NttDesc d, const uint64_t* __restrict__ cts, const uint64_t* __restrict__ s_eval, uint64_t p,
    uint64_t delta, uint64_t magic, uint64_t* __restrict__ mout, unsigned long long* __restrict__ max_all) {
  extern __shared__ uint64_t sm[];
  constexpr int n = 1 << LOGN, E = 1 << LOGR;
  constexpr int NPH = RowPhase<LOGN, LOGR, false, 0>::count;
  const int row = blockIdx.x, item = threadIdx.x;
  const uint64_t* c0 = cts + (size_t)row * 2 * n;
  const uint64_t* c1 = c0 + n;
  const uint64_t q = d.m.q, q2 = 2 * q;
  uint64_t e[E];
  if constexpr (!EVAL) {
    static_for<0, NPH>([&](auto kc) {  // forward transform of c1
      constexpr int K = decltype(kc)::value;
      using Ph = RowPhase<LOGN, LOGR, false, K>;
      constexpr int TL = Ph::TL;
      const int B = ((item >> TL) << (TL + LOGR)) + (item & ((1 << TL) - 1));
      if constexpr (K == 0) {
#pragma unroll
        for (int i = 0; i < E; ++i) e[i] = c1[B + (i << TL)];
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) e[i] = sm[spad(B) + (i << TL) + ((i << TL) >> 4)];
      }
      phase_math<LOGR, Ph::R, false, TL>(e, d, (uint32_t)(n + B), false);
      if constexpr (K < NPH - 1) {
#pragma unroll
        for (int i = 0; i < E; ++i) sm[spad(B) + (i << TL) + ((i << TL) >> 4)] = e[i];
        __syncthreads();
      }
    });
  }
  // the forward's last phase positions = the inverse's first: · s (+ c0 for EVAL input)
  {
    using Ph = RowPhase<LOGN, LOGR, true, 0>;
    constexpr int TL = Ph::TL;
    const int B = ((item >> TL) << (TL + LOGR)) + (item & ((1 << TL) - 1));
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const int pos = B + (i << TL);
      uint64_t x;
      if constexpr (EVAL) {
        x = c1[pos];
      } else {
        x = e[i] >= q2 ? e[i] - q2 : e[i];
        x = csub(x, q);
      }
      x = mulmod(x, s_eval[pos], d.m);
      if constexpr (EVAL) x = csub(x + c0[pos], q);
      e[i] = x;
    }
  }
  uint64_t local = 0;
  static_for<0, NPH>([&](auto kc) {  // inverse transform, then + c0 and the rounding
    constexpr int K = decltype(kc)::value;
    using Ph = RowPhase<LOGN, LOGR, true, K>;
    constexpr int TL = Ph::TL;
    const int B = ((item >> TL) << (TL + LOGR)) + (item & ((1 << TL) - 1));
    if constexpr (K > 0) {
#pragma unroll
      for (int i = 0; i < E; ++i) e[i] = sm[spad(B) + (i << TL) + ((i << TL) >> 4)];
    }
    phase_math<LOGR, Ph::R, true, TL>(e, d, (uint32_t)(n + B), Ph::S == 0);
    if constexpr (K < NPH - 1) {
      // (a thread stores exactly the positions it loaded for this phase: no barrier before)
#pragma unroll
      for (int i = 0; i < E; ++i) sm[spad(B) + (i << TL) + ((i << TL) >> 4)] = e[i];
      __syncthreads();
    } else {
      const uint64_t half = delta / 2;
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int pos = B + (i << TL);
        uint64_t u = csub(e[i], q);
        if constexpr (!EVAL) u = csub(u + c0[pos], q);
        const uint64_t x = u + half;  // (u + Δ//2) // Δ  (bfv.py:288)
        uint64_t mq = __umul64hi(x, magic);
        uint64_t rem = x - mq * delta;
        if (rem >= delta) {
          ++mq;
          rem -= delta;
        }
        const uint64_t aw = rem >= half ? rem - half : half - rem;  // |u - Δ m_raw|
        local = aw > local ? aw : local;
        while (mq >= p) mq -= p;
        mout[(size_t)row * n + pos] = mq;
      }
    }
  });
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t v = __shfl_xor_sync(0xffffffffu, local, o);
    local = v > local ? v : local;
  }
  if ((item & 31) == 0) atomicMax(max_all, (unsigned long long)local);
}

// The server's second round of the layer exchange (bfv.to_eval + pmult +
// plain_add, bfv.py:359-372, 503-512) in one launch: the forward transform of
// every row of ct [k][2][n] (one CTA per row), then out = NTT(row) ⊙ pt[ct]
// (+ add[ct] on c0 rows) before the store — the transformed ciphertext is
// never written. Values identical to fhe_ntt_forward + fhe_ct_pmult_add.
template <int LOGN, int LOGR>
__global__ void __launch_bounds__((1 << LOGN) >> LOGR, FHE_ROW_MINB((1 << LOGN) >> LOGR, LOGR))
    ntt_pmult_add_kernel(const NttDesc d, const uint64_t* __restrict__ ct, const uint64_t* __restrict__ pt,
                         const uint64_t* __restrict__ add, uint64_t* __restrict__ out) {
  extern __shared__ uint64_t sm[];
  constexpr int n = 1 << LOGN, E = 1 << LOGR;
  constexpr int NPH = RowPhase<LOGN, LOGR, false, 0>::count;
  const int row = blockIdx.x, item = threadIdx.x;
  const int c = row >> 1;
  const bool c0 = (row & 1) == 0;
  const uint64_t* srow = ct + (size_t)row * n;
  const uint64_t q = d.m.q, q2 = 2 * q;
  uint64_t e[E];
  static_for<0, NPH>([&](auto kc) {
    constexpr int K = decltype(kc)::value;
    using Ph = RowPhase<LOGN, LOGR, false, K>;
    constexpr int TL = Ph::TL;
    const int B = ((item >> TL) << (TL + LOGR)) + (item & ((1 << TL) - 1));
    if constexpr (K == 0) {
#pragma unroll
      for (int i = 0; i < E; ++i) e[i] = srow[B + (i << TL)];
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) e[i] = sm[spad(B) + (i << TL) + ((i << TL) >> 4)];
    }
    phase_math<LOGR, Ph::R, false, TL>(e, d, (uint32_t)(n + B), false);
    if constexpr (K == NPH - 1) {
#pragma unroll
      for (int i = 0; i < E; ++i) {
        const int pos = B + (i << TL);
        uint64_t x = e[i] >= q2 ? e[i] - q2 : e[i];
        x = mulmod(csub(x, q), pt[(size_t)c * n + pos], d.m);
        if (c0 && add) x = csub(x + add[(size_t)c * n + pos], q);
        out[(size_t)row * n + pos] = x;
      }
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) sm[spad(B) + (i << TL) + ((i << TL) >> 4)] = e[i];
      __syncthreads();
    }
  });
}

static bool row_direct_enabled() {  // FHE_NTT_ROW_DIRECT=0 selects the staged row kernel (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_NTT_ROW_DIRECT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Radix of the row kernels' register phases (2^LOGR elements per thread,
// n / 2^LOGR threads per row). Measured on the B200 at 512 rows: n = 4096
// radix 8 (512 threads) 32.8 us vs radix 16 34.8 us forward; n = 2048 with
// the direct kernel radix 8 13.4 us vs radix 16 14.2 us. FHE_NTT_ROW_LOGR
// overrides it for A/B checks.
static int row_logr(int logn) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FHE_NTT_ROW_LOGR");
    v = e ? atoi(e) : 0;
    if (v < 2 || v > 4) v = 0;
  }
  return v ? v : 3;  // n = 2048: radix 8 (256 threads, direct first/last phases) 13.4 vs 14.2 us at 512 rows
}

template <bool INV, int LOGN>
static void launch_row(const LimbSet& ls, const LoadMap& lm, uint64_t* dst, int rows, cudaStream_t st) {
  constexpr int n = 1 << LOGN;
  const size_t smem = (size_t)(n + (n >> 4) + 1) * sizeof(uint64_t);
  if (row_direct_enabled()) {
    switch (row_logr(LOGN)) {
      case 2: ntt_row_direct_kernel<INV, LOGN, 2><<<rows, n >> 2, smem, st>>>(ls, lm, dst); break;
      case 3: ntt_row_direct_kernel<INV, LOGN, 3><<<rows, n >> 3, smem, st>>>(ls, lm, dst); break;
      default: ntt_row_direct_kernel<INV, LOGN, 4><<<rows, n >> 4, smem, st>>>(ls, lm, dst); break;
    }
    return;
  }
  switch (row_logr(LOGN)) {
    case 2: ntt_row_kernel<INV, LOGN, 2><<<rows, n >> 2, smem, st>>>(ls, lm, dst); break;
    case 3: ntt_row_kernel<INV, LOGN, 3><<<rows, n >> 3, smem, st>>>(ls, lm, dst); break;
    default: ntt_row_kernel<INV, LOGN, 4><<<rows, n >> 4, smem, st>>>(ls, lm, dst); break;
  }
}

template <int LOGR, bool INV, bool COLS>
static int launch_split_one(const LimbSet& ls, const LoadMap& lm, uint64_t* dst, int rows, int a, int b,
                            int from_src, int final_, cudaStream_t st) {
  const int Lg = COLS ? a : b;
  const int len = 1 << Lg;
  const int per_row = COLS ? (1 << b) / kSplitW : (1 << a) / kSplitW;
  const int threads = kSplitW * (len >> LOGR);
  const size_t smem = COLS ? (size_t)len * kSplitW * 8 : (size_t)(spad(len * kSplitW) + 1) * 8;
  const int grid = rows * per_row;
  const bool capped = split_minb() != 1;
  if (Lg == 6) {
    if (capped) launch_split_k<LOGR, INV, COLS, 3, 6>(ls, lm, dst, grid, threads, smem, a, b, from_src, final_, st);
    else launch_split_k<LOGR, INV, COLS, 1, 6>(ls, lm, dst, grid, threads, smem, a, b, from_src, final_, st);
  } else if (Lg == 7) {
    if (capped) launch_split_k<LOGR, INV, COLS, 3, 7>(ls, lm, dst, grid, threads, smem, a, b, from_src, final_, st);
    else launch_split_k<LOGR, INV, COLS, 1, 7>(ls, lm, dst, grid, threads, smem, a, b, from_src, final_, st);
  } else {
    return fail(FHE_ERR_VALUE, "split NTT sub-transform length 2^%d unsupported", Lg);
  }
  FHE_CHECK_LAUNCH("ntt_split_kernel");
  return FHE_OK;
}

template <bool INV>
static int launch_split(const LimbSet& ls, const LoadMap& lm, uint64_t* dst, int rows, int logn, cudaStream_t st) {
  const int a = logn / 2, b = logn - a;  // a <= b <= 7 for n <= 16384
  if (!INV) {
    if (int rc = launch_split_one<4, false, true>(ls, lm, dst, rows, a, b, 1, 0, st)) return rc;
    return launch_split_one<4, false, false>(ls, lm, dst, rows, a, b, 0, 1, st);
  }
  if (int rc = launch_split_one<4, true, false>(ls, lm, dst, rows, a, b, 1, 0, st)) return rc;
  return launch_split_one<4, true, true>(ls, lm, dst, rows, a, b, 0, 1, st);
}

static int build_limbset(const fhe_plan* const* plans, int L, LimbSet* ls, int* n_out) {
  if (L < 1 || L > FHE_MAX_LIMBS) return fail(FHE_ERR_VALUE, "limb count %d out of range", L);
  if (!plans) return fail(FHE_ERR_VALUE, "null plans");
  ls->L = L;
  ls->pad_ = 0;
  int n = -1;
  for (int l = 0; l < L; ++l) {
    if (!plans[l]) return fail(FHE_ERR_VALUE, "null plan %d", l);
    if (n >= 0 && plans[l]->n != n) return fail(FHE_ERR_PARAMETER, "limb plans disagree on n");
    n = plans[l]->n;
    ls->d[l] = plans[l]->desc;
  }
  if (n > 16384) return fail(FHE_ERR_PARAMETER, "NTT supports n <= 16384 (got %d)", n);
  *n_out = n;
  return FHE_OK;
}

template <int LOGR, bool INV>
static int launch_t(const LimbSet& ls, const LoadMap& lm, uint64_t* dst, int rows, int n,
                    cudaStream_t st) {
  const size_t smem = (size_t)(n + (n >> 4) + 1) * sizeof(uint64_t);
  static std::atomic<uint64_t> attr_set{0};  // one bit per device (cudaFuncSetAttribute is per device)
  int dev = 0;
  FHE_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    FHE_CUDA(cudaFuncSetAttribute(ntt_kernel<LOGR, INV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  150 * 1024));
    attr_set.fetch_or(bit, std::memory_order_release);
  }
  int items = n >> LOGR;
  int threads = items < 512 ? items : 512;
  if (threads < 1) threads = 1;
  ntt_kernel<LOGR, INV><<<rows, threads, smem, st>>>(ls, lm, dst);
  FHE_CHECK_LAUNCH("ntt_kernel");
  return FHE_OK;
}

template <bool INV>
static int launch(const LimbSet& ls, const LoadMap& lm, uint64_t* dst, int rows, int n,
                  cudaStream_t st) {
  if (rows == 0) return FHE_OK;
  int logn = 0;
  while ((1 << logn) < n) ++logn;
  if (logn >= kSplitMinLog && split_enabled()) return launch_split<INV>(ls, lm, dst, rows, logn, st);
  if ((logn == 11 || logn == 12) && split_enabled()) {  // FHE_NTT_SPLIT=0 also selects the generic row kernel
    if (logn == 11)
      launch_row<INV, 11>(ls, lm, dst, rows, st);
    else
      launch_row<INV, 12>(ls, lm, dst, rows, st);
    FHE_CHECK_LAUNCH("ntt_row_kernel");
    return FHE_OK;
  }
  switch (logn < 4 ? logn : 4) {
    case 1: return launch_t<1, INV>(ls, lm, dst, rows, n, st);
    case 2: return launch_t<2, INV>(ls, lm, dst, rows, n, st);
    case 3: return launch_t<3, INV>(ls, lm, dst, rows, n, st);
    default: return launch_t<4, INV>(ls, lm, dst, rows, n, st);
  }
}

}  // namespace fhe

using namespace fhe;

extern "C" {

int fhe_ntt_forward(const fhe_plan* const* plans, int L, int B, int P, const uint64_t* src,
                    uint64_t* dst, void* stream) {
  LimbSet ls;
  int n;
  if (int rc = build_limbset(plans, L, &ls, &n)) return rc;
  if (B < 0 || P < 1) return fail(FHE_ERR_VALUE, "bad batch arguments");
  if (!B) return FHE_OK;  // empty batch: nothing to transform
  if (!src || !dst) return fail(FHE_ERR_VALUE, "null NTT buffer");
  LoadMap lm{src, P, 0, 0, 0, ~0ull};
  return launch<false>(ls, lm, dst, B * L * P, n, (cudaStream_t)stream);
}

int fhe_ntt_inverse(const fhe_plan* const* plans, int L, int B, int P, const uint64_t* src,
                    uint64_t* dst, void* stream) {
  LimbSet ls;
  int n;
  if (int rc = build_limbset(plans, L, &ls, &n)) return rc;
  if (B < 0 || P < 1) return fail(FHE_ERR_VALUE, "bad batch arguments");
  if (!B) return FHE_OK;  // empty batch: nothing to transform
  if (!src || !dst) return fail(FHE_ERR_VALUE, "null NTT buffer");
  LoadMap lm{src, P, 0, 0, 0, ~0ull};
  return launch<true>(ls, lm, dst, B * L * P, n, (cudaStream_t)stream);
}

int fhe_decrypt_fused(const fhe_plan* plan, int k, int eval, const uint64_t* cts, const uint64_t* s_eval,
                      uint64_t p, uint64_t delta, uint64_t* m_out, uint64_t* max_all, void* stream) {
  if (!plan || !cts || !s_eval || !m_out || !max_all) return fail(FHE_ERR_VALUE, "null decrypt operand");
  if (k < 0 || delta < 2 || p < 2) return fail(FHE_ERR_VALUE, "bad decrypt arguments");
  if (plan->desc.m.q >= (1ull << 62)) return fail(FHE_ERR_PARAMETER, "modulus too large");
  if (!k) return FHE_OK;
  const uint64_t magic = ~0ull / delta;
  cudaStream_t st = (cudaStream_t)stream;
  auto* mx = reinterpret_cast<unsigned long long*>(max_all);
#define FHE_DECRYPT_N(LOGN)                                                                                    \
  case (1 << LOGN): {                                                                                        \
    constexpr int LOGR = 3;                                                                                  \
    const size_t smem = (size_t)((1 << LOGN) + ((1 << LOGN) >> 4) + 1) * sizeof(uint64_t);                   \
    if (eval)                                                                                                \
      decrypt_fused_kernel<LOGN, LOGR, true><<<k, (1 << LOGN) >> LOGR, smem, st>>>(plan->desc, cts, s_eval, p, \
                                                                                  delta, magic, m_out, mx);  \
    else                                                                                                     \
      decrypt_fused_kernel<LOGN, LOGR, false><<<k, (1 << LOGN) >> LOGR, smem, st>>>(plan->desc, cts, s_eval, \
                                                                                   p, delta, magic, m_out, mx); \
    break;                                                                                                   \
  }
  switch (plan->n) {
    FHE_DECRYPT_N(10)
    FHE_DECRYPT_N(11)
    FHE_DECRYPT_N(12)
    default:
      return fail(FHE_ERR_PARAMETER, "fused decryption supports n = 1024, 2048, 4096 (got %d)", plan->n);
  }
#undef FHE_DECRYPT_N
  FHE_CHECK_LAUNCH("decrypt_fused_kernel");
  return FHE_OK;
}

int fhe_ntt_pmult_add(const fhe_plan* plan, int k, const uint64_t* ct, const uint64_t* pt, const uint64_t* add,
                      uint64_t* out, void* stream) {
  if (!plan || !ct || !pt || !out) return fail(FHE_ERR_VALUE, "null ntt-pmult operand");
  if (k < 0) return fail(FHE_ERR_VALUE, "bad ciphertext count");
  if (ct == out) return fail(FHE_ERR_VALUE, "ntt-pmult cannot run in place");
  if (!k) return FHE_OK;
  cudaStream_t st = (cudaStream_t)stream;
#define FHE_NTT_PMULT_N(LOGN)                                                                                \
  case (1 << LOGN): {                                                                                      \
    const size_t smem = (size_t)((1 << LOGN) + ((1 << LOGN) >> 4) + 1) * sizeof(uint64_t);                 \
    ntt_pmult_add_kernel<LOGN, 3><<<2 * k, (1 << LOGN) >> 3, smem, st>>>(plan->desc, ct, pt, add, out);    \
    break;                                                                                                 \
  }
  switch (plan->n) {
    FHE_NTT_PMULT_N(10)
    FHE_NTT_PMULT_N(11)
    FHE_NTT_PMULT_N(12)
    default:
      return fail(FHE_ERR_PARAMETER, "ntt-pmult supports n = 1024, 2048, 4096 (got %d)", plan->n);
  }
#undef FHE_NTT_PMULT_N
  FHE_CHECK_LAUNCH("ntt_pmult_add_kernel");
  return FHE_OK;
}

int fhe_ntt_forward_digits(const fhe_plan* const* plans, int L, int B, const uint64_t* src,
                           uint64_t* dst, int T, int ndig, void* stream) {
  LimbSet ls;
  int n;
  if (int rc = build_limbset(plans, L, &ls, &n)) return rc;
  if (B < 0 || ndig < 1 || T < 1 || T > 63) return fail(FHE_ERR_VALUE, "bad digit arguments");
  if (!B) return FHE_OK;
  if (!src || !dst) return fail(FHE_ERR_VALUE, "null digit buffer");
  if (src == dst) return fail(FHE_ERR_VALUE, "digit NTT cannot run in place");
  LoadMap lm{src, ndig, ndig, T, 0, (1ull << T) - 1};
  return launch<false>(ls, lm, dst, B * L * ndig, n, (cudaStream_t)stream);
}

}  // extern "C"
