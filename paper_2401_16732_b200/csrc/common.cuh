// common.cuh — shared types, modular arithmetic and error plumbing of libflashhe.
//
// Modular arithmetic for 60-bit-class primes (q < 2^62) on the integer pipes:
//   * Shoup multiplication by precomputed constants (twiddles, scalars),
//     result in [0, 2q) — Harvey lazy butterflies keep NTT values in [0, 4q).
//   * Barrett reduction of a full 128-bit product (general a*b, both < q).
//   * Montgomery REDC for lazily accumulated sums < q * 2^64 (key switching).
// All reductions end canonical in [0, q), which is what the reference's
// `% q` on Python ints yields (ring.py:144,162,197,243,403-405), so any
// correct schedule of these operations is bit-exact with it.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/flashhe.h"

namespace fhe {

// ------------------------------------------------------------------ errors
void set_error(int code, const char* fmt, ...);
int fail(int code, const char* fmt, ...);
extern std::atomic<uint64_t> g_launches;

#define FHE_CHECK_LAUNCH(what)                                                  \
  do {                                                                          \
    ::fhe::g_launches.fetch_add(1, std::memory_order_relaxed);                  \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess)                                                      \
      return ::fhe::fail(FHE_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e_)); \
  } while (0)

#define FHE_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return ::fhe::fail(FHE_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------ host helpers
typedef unsigned __int128 u128_t;

static inline uint64_t h_mulmod(uint64_t a, uint64_t b, uint64_t q) {
  return (uint64_t)(((u128_t)a * b) % q);
}
static inline uint64_t h_powmod(uint64_t b, uint64_t e, uint64_t q) {
  uint64_t r = 1 % q;
  b %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, b, q);
    b = h_mulmod(b, b, q);
    e >>= 1;
  }
  return r;
}
static inline uint64_t h_invmod(uint64_t a, uint64_t q) {  // a^-1 mod q (extended Euclid)
  __int128 t = 0, nt = 1, r = q, nr = a % q;
  while (nr) {
    __int128 qq = r / nr, tmp;
    tmp = t - qq * nt; t = nt; nt = tmp;
    tmp = r - qq * nr; r = nr; nr = tmp;
  }
  if (t < 0) t += q;
  return (uint64_t)t;
}
static inline uint64_t h_shoup(uint64_t w, uint64_t q) {  // floor(w * 2^64 / q)
  return (uint64_t)(((u128_t)w << 64) / q);
}
static inline int h_bitlen(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 0; }

// Per-modulus constants, passed to kernels by value.
struct ModDesc {
  uint64_t q;
  uint64_t mu;        // floor(2^(2k) / q)           (Barrett)
  uint64_t qinv_neg;  // -q^{-1} mod 2^64            (Montgomery)
  uint64_t r2;        // 2^128 mod q                 (to Montgomery form)
  uint64_t inv64;     // floor((2^64-1) / q)         (64-bit reduction)
  uint32_t k;         // bit length of q
  uint32_t pad_;
};

static inline ModDesc make_mod(uint64_t q) {
  ModDesc m;
  m.q = q;
  m.k = (uint32_t)h_bitlen(q);
  m.mu = (uint64_t)(((u128_t)1 << (2 * m.k)) / q);
  // Newton iteration for q^{-1} mod 2^64 (q odd)
  uint64_t inv = q;  // correct to 3 bits
  for (int i = 0; i < 6; ++i) inv *= 2 - q * inv;
  m.qinv_neg = (uint64_t)(0 - inv);
  uint64_t r = (uint64_t)(((u128_t)1 << 64) % q);  // 2^64 mod q
  m.r2 = h_mulmod(r, r, q);
  m.inv64 = ~0ull / q;
  m.pad_ = 0;
  return m;
}

// NTT descriptor of one limb (device tables + constants).
struct NttDesc {
  ModDesc m;
  const ulonglong2* psi;   // [n] (psi_brv[i], shoup)        forward CT twiddles
  const ulonglong2* ipsi;  // [n] (ipsi_brv[i], shoup)       inverse GS twiddles
  ulonglong2 ninv;         // (n^-1, shoup)
  ulonglong2 ninv_w1;      // (n^-1 * ipsi_brv[1], shoup)    folded last GS stage
  int n, logn;
};

struct LimbSet {
  int L;
  int pad_;
  NttDesc d[FHE_MAX_LIMBS];
};

struct ModSet {
  int L;
  int pad_;
  ModDesc m[FHE_MAX_LIMBS];
};

int make_modset(const uint64_t* moduli, int L, ModSet* out);

}  // namespace fhe

struct fhe_plan {
  int n, logn;
  uint64_t q, psi;
  fhe::NttDesc desc;  // device pointers inside
  void* dev_mem;      // owns psi/ipsi tables
};

namespace fhe {

// ---------------------------------------------------------- device arith
__device__ __forceinline__ uint64_t shoup_lazy(uint64_t y, uint64_t w, uint64_t wp, uint64_t q) {
  // w * y mod q in [0, 2q) for any y < 2^64, w < q, wp = floor(w 2^64 / q)
  uint64_t qt = __umul64hi(wp, y);
  return w * y - qt * q;
}

__device__ __forceinline__ uint64_t csub(uint64_t x, uint64_t q) { return x >= q ? x - q : x; }

// Barrett: x = hi:lo < 2^(2k)  ->  x mod q
__device__ __forceinline__ uint64_t barrett128(uint64_t lo, uint64_t hi, const ModDesc& m) {
  const uint32_t k = m.k;
  uint64_t q1 = (hi << (65 - k)) | (lo >> (k - 1));
  uint64_t q2lo = q1 * m.mu;
  uint64_t q2hi = __umul64hi(q1, m.mu);
  uint64_t q3 = (q2hi << (63 - k)) | (q2lo >> (k + 1));
  uint64_t r = lo - q3 * m.q;
  r = csub(r, m.q);
  return csub(r, m.q);
}

__device__ __forceinline__ uint64_t mulmod(uint64_t a, uint64_t b, const ModDesc& m) {
  return barrett128(a * b, __umul64hi(a, b), m);
}

// Montgomery REDC of x = hi:lo < q 2^64 -> x 2^-64 mod q, canonical.
__device__ __forceinline__ uint64_t redc(uint64_t lo, uint64_t hi, const ModDesc& m) {
  uint64_t mm = lo * m.qinv_neg;
  uint64_t t = hi + __umul64hi(mm, m.q) + (lo != 0 ? 1ull : 0ull);
  return csub(t, m.q);
}

// 128-bit accumulate: (hi:lo) += a*b
__device__ __forceinline__ void mac128(uint64_t& lo, uint64_t& hi, uint64_t a, uint64_t b) {
  uint64_t pl = a * b, ph = __umul64hi(a, b);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;" : "+l"(lo), "+l"(hi) : "l"(pl), "l"(ph));
}

// Column-split 128-bit accumulator for sums of up to 8 products of 60-bit
// operands (u, v < 2^60): the 32x32 partial products go to separate columns —
// lo*lo into a 96-bit carry chain, both cross products into one 64-bit word
// (16 terms < 2^60 each), hi*hi into another (< 2^56 each) — so no 128-bit
// carry propagation per product; acc60_get combines the columns once.
struct Acc60 {
  uint32_t s0, s1, s2;
  uint64_t x, h;
};
__device__ __forceinline__ void acc60_zero(Acc60& a) {
  a.s0 = a.s1 = a.s2 = 0;
  a.x = a.h = 0;
}
__device__ __forceinline__ void mac60(Acc60& a, uint64_t u, uint64_t v) {
  const uint32_t ul = (uint32_t)u, uh = (uint32_t)(u >> 32), vl = (uint32_t)v, vh = (uint32_t)(v >> 32);
  asm("mad.lo.cc.u32 %0, %3, %4, %0;\n\tmadc.hi.cc.u32 %1, %3, %4, %1;\n\taddc.u32 %2, %2, 0;"
      : "+r"(a.s0), "+r"(a.s1), "+r"(a.s2)
      : "r"(ul), "r"(vl));
  a.x += (uint64_t)ul * vh;
  a.x += (uint64_t)uh * vl;
  a.h += (uint64_t)uh * vh;
}
__device__ __forceinline__ void acc60_get(const Acc60& a, uint64_t& lo, uint64_t& hi) {
  const uint64_t l = ((uint64_t)a.s1 << 32) | a.s0;
  lo = l + (a.x << 32);
  hi = a.h + a.s2 + (a.x >> 32) + (lo < l ? 1ull : 0ull);
}

// Karatsuba accumulator for sums of up to 4 products of operands below 2^60:
// u = u0 + 2^30 u1 with 30-bit limbs, u0 v0 and u1 v1 accumulate directly and
// the cross term through (u0 + u1)(v0 + v1) (< 2^62 each, four sum below 2^64),
// so a product costs three 32x32 -> 64 multiply-accumulates (IMAD.WIDE.U32
// with a 64-bit addend) and no carry handling; acc30_get recombines once.
struct Split30 {
  uint32_t l, h, s;  // low 30 bits, high 30 bits, their sum (< 2^31)
};
__device__ __forceinline__ Split30 split30(uint64_t u) {
  Split30 r;
  r.l = (uint32_t)u & 0x3fffffffu;
  r.h = (uint32_t)(u >> 30);
  r.s = r.l + r.h;
  return r;
}
struct Acc30 {
  uint64_t s00, smid, s11;
};
__device__ __forceinline__ void acc30_zero(Acc30& a) { a.s00 = a.smid = a.s11 = 0; }
__device__ __forceinline__ void mac30(Acc30& a, const Split30& u, const Split30& v) {
  a.s00 += (uint64_t)u.l * v.l;
  a.s11 += (uint64_t)u.h * v.h;
  a.smid += (uint64_t)u.s * v.s;
}
// T = s00 + 2^30 (smid - s00 - s11) + 2^60 s11 as hi:lo
__device__ __forceinline__ void acc30_get(const Acc30& a, uint64_t& lo, uint64_t& hi) {
  const uint64_t m = a.smid - a.s00 - a.s11;
  const uint64_t x = m << 30, y = a.s11 << 60;
  asm("add.cc.u64 %0, %2, %3;\n\t"
      "addc.u64 %1, %4, %5;\n\t"
      "add.cc.u64 %0, %0, %6;\n\t"
      "addc.u64 %1, %1, 0;"
      : "=l"(lo), "=l"(hi)
      : "l"(a.s00), "l"(x), "l"(m >> 34), "l"(a.s11 >> 4), "l"(y));
}

// x mod q for any x < 2^64 (q < 2^63): quotient estimate off by at most 1
__device__ __forceinline__ uint64_t reduce_u64(uint64_t x, const ModDesc& m) {
  uint64_t qt = __umul64hi(x, m.inv64);
  return csub(x - qt * m.q, m.q);
}

// canonical residue of a signed 64-bit value
__device__ __forceinline__ uint64_t reduce_i64(int64_t x, const ModDesc& m) {
  uint64_t mag = x < 0 ? (uint64_t)(-(x + 1)) + 1 : (uint64_t)x;  // |x|, no UB at INT64_MIN
  uint64_t r = reduce_u64(mag, m);
  return (x < 0 && r) ? m.q - r : r;
}

__device__ __forceinline__ uint32_t brev_bits(uint32_t x, int bits) {
  return bits ? (__brev(x) >> (32 - bits)) : 0u;
}

}  // namespace fhe
