// elementwise.cu — K3 (pointwise ring ops), K4 apply (hoisted key switch),
// K5 (x^2+x share arithmetic) and K6 (decryption rounding).
// All HBM-bound single passes: 128-bit coalesced rows where the access is
// affine, scalar 64-bit gathers where it is a permutation (DRot, automorphism,
// eval-domain Galois map).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace fhe {

static constexpr int kThreads = 256;

static inline unsigned grid_for(int64_t work) {
  int64_t g = (work + kThreads - 1) / kThreads;
  return (unsigned)(g < 1 ? 1 : g);
}

// row r of [B][L][P] -> (b, l, p)
struct RowGeom {
  int L, P, logn;
  __device__ __forceinline__ void split(int64_t r, int64_t& b, int& l, int& p) const {
    p = (int)(r % P);
    int64_t t = r / P;
    l = (int)(t % L);
    b = t / L;
  }
};

static int log2i(int n) {
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  return lg;
}

static int check_rows(int L, int B, int P, int n) {
  if (L < 1 || L > FHE_MAX_LIMBS || B < 0 || P < 1 || n < 2 || (n & (n - 1)))
    return fail(FHE_ERR_VALUE, "bad row geometry (L=%d B=%d P=%d n=%d)", L, B, P, n);
  return FHE_OK;
}

// ------------------------------------------------------------- binary ops
__global__ void binary_kernel(int op, const ModSet ms, RowGeom g, int B, int Bb, int Pb,
                              const uint64_t* __restrict__ a, const uint64_t* __restrict__ b,
                              uint64_t* __restrict__ out, int64_t total2) {
  int64_t i2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pair index
  if (i2 >= total2) return;
  const int64_t idx = 2 * i2;
  const int64_t r = idx >> g.logn;
  const int col = (int)(idx & ((1 << g.logn) - 1));
  int64_t bb;
  int l, p;
  g.split(r, bb, l, p);
  const int64_t rb = ((bb % Bb) * g.L + l) * Pb + (p % Pb);
  const ModDesc& m = ms.m[l];
  const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(a + idx);
  const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(b + (rb << g.logn) + col);
  ulonglong2 z;
  if (op == FHE_OP_ADD) {
    z.x = csub(x.x + y.x, m.q);
    z.y = csub(x.y + y.y, m.q);
  } else if (op == FHE_OP_SUB) {
    z.x = x.x >= y.x ? x.x - y.x : x.x + m.q - y.x;
    z.y = x.y >= y.y ? x.y - y.y : x.y + m.q - y.y;
  } else {
    z.x = mulmod(x.x, y.x, m);
    z.y = mulmod(x.y, y.y, m);
  }
  *reinterpret_cast<ulonglong2*>(out + idx) = z;
}

// pmult with a prepared plaintext: Shoup multiplication by the plaintext word
// and its companion w' = floor(w 2^64 / q) — 2 high/low products per element
// instead of the generic 128-bit Barrett reduction; identical canonical result.
__global__ void mul_shoup_kernel(const ModSet ms, RowGeom g, int Bb, int Pb, const uint64_t* __restrict__ a,
                                 const uint64_t* __restrict__ w, const uint64_t* __restrict__ wp,
                                 uint64_t* __restrict__ out, int64_t total2) {
  const int64_t i2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pair index
  if (i2 >= total2) return;
  const int64_t idx = 2 * i2;
  const int r = (int)(idx >> g.logn);  // rows < 2^31 (checked on the host)
  const int col = (int)(idx & ((1 << g.logn) - 1));
  const int p = r % g.P, t = r / g.P, l = t % g.L, bb = t / g.L;
  const int64_t rb = ((int64_t)(bb % Bb) * g.L + l) * Pb + (p % Pb);
  const uint64_t q = ms.m[l].q;
  const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(a + idx);
  const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(w + (rb << g.logn) + col);
  const ulonglong2 yp = *reinterpret_cast<const ulonglong2*>(wp + (rb << g.logn) + col);
  ulonglong2 z;
  z.x = csub(shoup_lazy(x.x, y.x, yp.x, q), q);
  z.y = csub(shoup_lazy(x.y, y.y, yp.y, q), q);
  *reinterpret_cast<ulonglong2*>(out + idx) = z;
}

// pmult with one plaintext broadcast over the batch (Bb = 1, the common
// case): each thread keeps its plaintext pair and companions in registers and
// applies them to BCH ciphertexts, whose loads are all issued first — the
// plaintext is read once per chunk and the row decomposition is done once.
template <int BCH>
__global__ void mul_shoup_bcast_kernel(const ModSet ms, int logn, int L, int P, int Pb, int B,
                                       const uint64_t* __restrict__ a, const uint64_t* __restrict__ w,
                                       const uint64_t* __restrict__ wp, uint64_t* __restrict__ out, int64_t inner2) {
  const int64_t j2 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pair index inside one batch slice
  if (j2 >= inner2) return;
  const int64_t j = 2 * j2;
  const int rr = (int)(j >> logn);  // l * P + p
  const int col = (int)(j & ((1 << logn) - 1));
  const int p = rr % P, l = rr / P;
  const int64_t rb = (int64_t)l * Pb + (p % Pb);
  const uint64_t q = ms.m[l].q;
  const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(w + (rb << logn) + col);
  const ulonglong2 yp = *reinterpret_cast<const ulonglong2*>(wp + (rb << logn) + col);
  const int b0 = blockIdx.y * BCH;
  const int64_t slice = (int64_t)L * P << logn;  // words per batch entry
  ulonglong2 x[BCH];
#pragma unroll
  for (int k = 0; k < BCH; ++k)
    if (b0 + k < B) x[k] = *reinterpret_cast<const ulonglong2*>(a + (b0 + k) * slice + j);
#pragma unroll
  for (int k = 0; k < BCH; ++k) {
    if (b0 + k < B) {
      ulonglong2 z;
      z.x = csub(shoup_lazy(x[k].x, y.x, yp.x, q), q);
      z.y = csub(shoup_lazy(x[k].y, y.y, yp.y, q), q);
      *reinterpret_cast<ulonglong2*>(out + (b0 + k) * slice + j) = z;
    }
  }
}

// w' = floor(w 2^64 / q_l) per word (one-time, when a plaintext is prepared)
__global__ void shoup_companion_kernel(const ModSet ms, RowGeom g, const uint64_t* __restrict__ w,
                                       uint64_t* __restrict__ wp, int64_t total) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int r = (int)(idx >> g.logn);
  const int l = (r / g.P) % g.L;
  wp[idx] = (uint64_t)(((unsigned __int128)w[idx] << 64) / ms.m[l].q);
}

__global__ void neg_kernel(const ModSet ms, RowGeom g, const uint64_t* __restrict__ a,
                           uint64_t* __restrict__ out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int64_t bb;
  int l, p;
  g.split(idx >> g.logn, bb, l, p);
  const uint64_t v = a[idx];
  out[idx] = v ? ms.m[l].q - v : 0;
}

struct Scalars {
  uint64_t k[FHE_MAX_LIMBS];
  uint64_t kp[FHE_MAX_LIMBS];  // Shoup companions
};

__global__ void scalar_kernel(const ModSet ms, RowGeom g, Scalars sc, const uint64_t* __restrict__ a,
                              uint64_t* __restrict__ out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int64_t bb;
  int l, p;
  g.split(idx >> g.logn, bb, l, p);
  const uint64_t q = ms.m[l].q;
  out[idx] = csub(shoup_lazy(a[idx], sc.k[l], sc.kp[l], q), q);
}

// out = a * x^(-shift) mod x^n + 1 (ring.monomial_mul, ring.py:279-299)
__global__ void monomial_kernel(const ModSet ms, RowGeom g, int64_t s, int flip,
                                const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                                int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int n = 1 << g.logn;
  const int64_t r = idx >> g.logn;
  const int i = (int)(idx & (n - 1));
  int64_t bb;
  int l, p;
  g.split(r, bb, l, p);
  int j = i + (int)s;
  int neg = flip;
  if (j >= n) {
    j -= n;
    neg ^= 1;
  }
  const uint64_t v = a[(r << g.logn) + j];
  out[idx] = (neg && v) ? ms.m[l].q - v : v;
}

// ResNet shortcut in the conv output layout (one channel per ciphertext):
// out[j] = y[j] + a[j / c_n] * x^(-tile*(j mod c_n)) for both polynomials of
// ciphertext j. The DRot (ring.monomial_mul, ring.py:279-299) moves channel j's
// tile of the packed block input to slot 0, where conv_proposed writes channel
// j; c_n = 1 is a plain hadd (bfv.py:316-320). In place on y is allowed.
__global__ void residual_add_kernel(uint64_t q, int logn, int c_n, int tile,
                                    const uint64_t* y, const uint64_t* __restrict__ a,
                                    uint64_t* out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int n = 1 << logn;
  const int64_t r = idx >> logn;  // output row: ciphertext j = r / 2, polynomial r % 2
  const int i = (int)(idx & (n - 1));
  const int64_t j = r >> 1;
  int src = i + tile * (int)(j % c_n);
  const bool neg = src >= n;
  if (neg) src -= n;
  uint64_t v = a[(((j / c_n) << 1) + (r & 1)) * n + src];
  if (neg && v) v = q - v;
  uint64_t s = y[idx] + v;
  out[idx] = s >= q ? s - q : s;
}

// out(x) = a(x^gpow) (ring.apply_galois, ring.py:326-334), scatter form
__global__ void automorphism_kernel(const ModSet ms, RowGeom g, uint64_t gpow,
                                    const uint64_t* __restrict__ a, uint64_t* __restrict__ out,
                                    int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const int n = 1 << g.logn;
  const int64_t r = idx >> g.logn;
  const uint64_t i = (uint64_t)(idx & (n - 1));
  int64_t bb;
  int l, p;
  g.split(r, bb, l, p);
  const uint64_t mask2n = 2ull * n - 1;  // mod 2n as a mask (n is a power of two)
  const uint64_t e = (i * (gpow & mask2n)) & mask2n;
  const uint64_t v = a[idx];
  const bool neg = e >= (uint64_t)n;
  out[(r << g.logn) + (e & (n - 1))] = (neg && v) ? ms.m[l].q - v : v;
}

__global__ void add_delta_kernel(ModDesc mq, uint64_t p, uint64_t delta, const uint64_t* __restrict__ base,
                                 const int64_t* __restrict__ m, uint64_t* __restrict__ out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int64_t v = m[idx] % (int64_t)p;
  if (v < 0) v += (int64_t)p;
  uint64_t dm = delta * (uint64_t)v;  // Δ (p-1) < q (bfv.py:167)
  uint64_t b = base ? base[idx] : 0;
  out[idx] = csub(b + dm, mq.q);
}

// c0 = (Δ (m mod p) - as - e) mod q   (bfv.encrypt_private, bfv.py:181)
__global__ void encrypt_combine_kernel(ModDesc mq, uint64_t p, uint64_t delta, const int64_t* __restrict__ m,
                                       const uint64_t* __restrict__ as, const int64_t* __restrict__ e,
                                       uint64_t* __restrict__ out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int64_t v = m ? m[idx] % (int64_t)p : 0;  // m == NULL: encryptions of zero
  if (v < 0) v += (int64_t)p;
  const uint64_t q = mq.q;
  uint64_t t = csub(delta * (uint64_t)v, q);
  t = csub(t + q - as[idx], q);
  const uint64_t er = reduce_i64(e[idx], mq);
  out[idx] = csub(t + q - er, q);
}

__global__ void lift_centered_kernel(uint64_t p, uint64_t q, const int64_t* __restrict__ v,
                                     uint64_t* __restrict__ out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int64_t x = v[idx] % (int64_t)p;
  if (x < 0) x += (int64_t)p;
  if (x > (int64_t)(p / 2)) x -= (int64_t)p;  // bfv.centered (bfv.py:156-159)
  out[idx] = x < 0 ? q - (uint64_t)(-x) : (uint64_t)x;
}

__global__ void to_mont_kernel(const ModSet ms, RowGeom g, const uint64_t* __restrict__ a,
                               uint64_t* __restrict__ out, int64_t total) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  int64_t bb;
  int l, p;
  g.split(idx >> g.logn, bb, l, p);
  const ModDesc& m = ms.m[l];
  const uint64_t x = a[idx];
  out[idx] = redc(x * m.r2, __umul64hi(x, m.r2), m);
}

// ------------------------------------------------- WidePoly (ring.py:347-406)
__global__ void wide_acc_kernel(int n, const uint64_t* __restrict__ f, const int64_t* __restrict__ flo,
                                const int64_t* __restrict__ fhi, int64_t scalar, int64_t* lo, int64_t* hi) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t a, b;
  if (f) {
    a = (int64_t)(f[i] & ((1ull << 30) - 1));
    b = (int64_t)(f[i] >> 30);
  } else {
    a = flo[i];
    b = fhi[i];
  }
  // int64 wrap-around like numpy (the budget guard keeps it from happening)
  lo[i] = (int64_t)((uint64_t)lo[i] + (uint64_t)a * (uint64_t)scalar);
  hi[i] = (int64_t)((uint64_t)hi[i] + (uint64_t)b * (uint64_t)scalar);
}

__global__ void wide_rot_kernel(int n, const int64_t* __restrict__ olo, const int64_t* __restrict__ ohi,
                                int s, int flip, int64_t* lo, int64_t* hi) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int j = i + s, neg = flip;
  if (j >= n) {
    j -= n;
    neg ^= 1;
  }
  const uint64_t a = (uint64_t)olo[j], b = (uint64_t)ohi[j];
  lo[i] = (int64_t)(neg ? (uint64_t)lo[i] - a : (uint64_t)lo[i] + a);
  hi[i] = (int64_t)(neg ? (uint64_t)hi[i] - b : (uint64_t)hi[i] + b);
}

__global__ void wide_fin_kernel(int n, ModDesc m, uint64_t w30, uint64_t w30p, const int64_t* __restrict__ lo,
                                const int64_t* __restrict__ hi, uint64_t* __restrict__ out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t l = reduce_i64(lo[i], m), h = reduce_i64(hi[i], m);
  out[i] = csub(l + csub(shoup_lazy(h, w30, w30p, m.q), m.q), m.q);
}

// ------------------------------------------------------- K6 decrypt round
__global__ void decrypt_round_kernel(uint64_t p, uint64_t delta, uint64_t magic, int n,
                                     const uint64_t* __restrict__ u, uint64_t* __restrict__ mout,
                                     uint64_t* __restrict__ maxw, unsigned long long* __restrict__ max_all) {
  const int64_t r = blockIdx.x;
  const uint64_t half = delta / 2;
  uint64_t local = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint64_t x = u[r * n + i] + half;  // (u + Δ//2) // Δ  (bfv.py:288)
    uint64_t mq = __umul64hi(x, magic);
    uint64_t rem = x - mq * delta;
    if (rem >= delta) {
      ++mq;
      rem -= delta;
    }
    // w = u - Δ m_raw = rem - Δ//2
    const uint64_t aw = rem >= half ? rem - half : half - rem;
    local = aw > local ? aw : local;
    while (mq >= p) mq -= p;  // m_raw <= p + 1 since Δ = q // p
    mout[r * n + i] = mq;
  }
  __shared__ uint64_t red[32];
  for (int o = 16; o > 0; o >>= 1) {
    uint64_t v = __shfl_xor_sync(0xffffffffu, local, o);
    local = v > local ? v : local;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t mx = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) mx = red[w] > mx ? red[w] : mx;
    if (maxw) maxw[r] = mx;
    if (max_all) atomicMax(max_all, (unsigned long long)mx);
  }
}

// ------------------------------------------------------- row plumbing
constexpr int kCopyMany = 8;
struct CopyTable {
  const uint64_t* src[kCopyMany];
  uint64_t* dst[kCopyMany];
  unsigned long long start[kCopyMany + 1];  // word offsets of each copy in the concatenation
  int count;
};

// grid-stride over the concatenated words of all copies; the copy of word w is
// found by a short scan of the (<= 8) start offsets
__global__ void copy_many_kernel(const CopyTable t) {
  const unsigned long long total = t.start[t.count];
  for (unsigned long long w = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; w < total;
       w += (unsigned long long)gridDim.x * blockDim.x) {
    int c = 0;
    while (w >= t.start[c + 1]) ++c;
    const unsigned long long i = w - t.start[c];
    t.dst[c][i] = t.src[c][i];
  }
}
// Gather k device rows of n words (arbitrary addresses) into one contiguous
// stack: the list form of a ciphertext batch (bfv.cts_rows of separate
// Ciphertext objects) becomes one [k][n] operand without a torch kernel.
constexpr int kGatherPtrs = 64;
struct GatherPtrs {
  const uint64_t* src[kGatherPtrs];
};

__global__ void gather_rows_kernel(const __grid_constant__ GatherPtrs P, int n, uint64_t* __restrict__ dst) {
  const int r = blockIdx.y;
  const uint64_t* s = P.src[r];
  uint64_t* d = dst + (size_t)r * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[i] = s[i];
}

// ------------------------------------------------------------ K5 shares
__global__ void act_client_kernel(ModDesc mp, uint64_t two_f, const uint64_t* __restrict__ w,
                                  uint64_t* __restrict__ y, int64_t count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t x = reduce_u64(w[i], mp);
  const uint64_t sq = mulmod(x, x, mp);
  const uint64_t lin = mulmod(x, two_f, mp);
  y[i] = csub(sq + lin, mp.q);
}

__global__ void act_server_kernel(ModDesc mp, uint64_t two_f, const uint64_t* __restrict__ r,
                                  const uint64_t* __restrict__ rsq, const uint64_t* __restrict__ v,
                                  uint64_t* __restrict__ c, int64_t count) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t p = mp.q;
  const uint64_t rr = reduce_u64(r[i], mp);
  const uint64_t lin = mulmod(rr, two_f, mp);
  uint64_t t = reduce_u64(rsq[i], mp);
  t = csub(t + p - lin, p);
  c[i] = csub(t + reduce_u64(v[i], mp), p);
}

// ------------------------------------------------ K4 hoisted key switching
// One thread per (position x, limb l, batch chunk): the 2*ndig key words of x
// stay in registers and are reused by every ciphertext of the chunk (the key
// is read from HBM once per chunk, not once per ciphertext).
template <int MAXD, int BCH, bool W60>
__global__ void __launch_bounds__(128) keyswitch_kernel(const ModSet ms, int logn, int L, int B, int ndig,
                                                        uint64_t gpow, const uint64_t* __restrict__ ct,
                                                        const uint64_t* __restrict__ dig,
                                                        const uint64_t* __restrict__ keys,
                                                        uint64_t* __restrict__ out) {
  const int n = 1 << logn;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int l = blockIdx.y;
  const int b0 = blockIdx.z * BCH;
  const ModDesc m = ms.m[l];
  // eval_perm (ring.py:199-202): exp_at_index[x] = 2 bitrev(x) + 1. A warp's 32
  // consecutive x gather from 32 distinct slots of two aligned 128-byte lines
  // (the map permutes within blocks), so the gathers stay coalesced.
  const uint32_t e = 2u * brev_bits((uint32_t)x, logn) + 1u;
  const uint32_t mask2n = 2u * (uint32_t)n - 1u;  // 2n is a power of two: mod 2n is a mask
  const uint32_t e2 = (uint32_t)(((uint64_t)e * (gpow & mask2n)) & mask2n);
  const int src = (int)brev_bits((e2 - 1u) >> 1, logn);
  uint64_t k0[MAXD], k1[MAXD];
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    if (i < ndig) {
      k0[i] = keys[((size_t)(l * ndig + i) * 2 + 0) * n + x];
      k1[i] = keys[((size_t)(l * ndig + i) * 2 + 1) * n + x];
    }
  }
  // BCH ciphertexts per thread: every gather of the chunk (BCH x (ndig + 1)
  // words) is issued as a predicated load before the first multiply, so they
  // are all in flight together (memory-level parallelism); the key words stay
  // in registers for all of them
  uint64_t dv[BCH][MAXD], c0v[BCH];
#pragma unroll
  for (int bb = 0; bb < BCH; ++bb) {
    const bool ok = b0 + bb < B;
    const size_t crow = ((size_t)(b0 + bb) * L + l) * 2;
    const size_t drow = ((size_t)(b0 + bb) * L + l) * ndig;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) dv[bb][i] = (ok && i < ndig) ? __ldg(&dig[(drow + i) * n + src]) : 0;
    c0v[bb] = ok ? __ldg(&ct[crow * n + src]) : 0;
  }
  constexpr bool KARA = W60 && MAXD <= 4;  // q < 2^60, <= 4 digits: Karatsuba 30-bit limbs
  Split30 sk0[KARA ? MAXD : 1], sk1[KARA ? MAXD : 1];
  if constexpr (KARA) {
#pragma unroll
    for (int i = 0; i < MAXD; ++i) {
      sk0[i] = split30(k0[i]);
      sk1[i] = split30(k1[i]);
    }
  }
#pragma unroll
  for (int bb = 0; bb < BCH; ++bb) {
    const int b = b0 + bb;
    if (b < B) {
      const size_t crow = ((size_t)b * L + l) * 2;
      uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0;
      if constexpr (KARA) {
        Acc30 s0, s1;
        acc30_zero(s0);
        acc30_zero(s1);
#pragma unroll
        for (int i = 0; i < MAXD; ++i) {
          if (i < ndig) {
            const Split30 u = split30(dv[bb][i]);
            mac30(s0, u, sk0[i]);
            mac30(s1, u, sk1[i]);
          }
        }
        acc30_get(s0, a0l, a0h);
        acc30_get(s1, a1l, a1h);
      } else if constexpr (W60) {  // q < 2^60, ndig <= 8: column-split accumulation
        Acc60 s0, s1;
        acc60_zero(s0);
        acc60_zero(s1);
#pragma unroll
        for (int i = 0; i < MAXD; ++i) {
          if (i < ndig) {
            mac60(s0, dv[bb][i], k0[i]);
            mac60(s1, dv[bb][i], k1[i]);
          }
        }
        acc60_get(s0, a0l, a0h);
        acc60_get(s1, a1l, a1h);
      } else {
#pragma unroll
        for (int i = 0; i < MAXD; ++i) {
          if (i < ndig) {
            mac128(a0l, a0h, dv[bb][i], k0[i]);
            mac128(a1l, a1h, dv[bb][i], k1[i]);
          }
        }
      }
      // Σ_i D_i swk_i < ndig q^2 < q 2^64 (ndig < 2^64/q): one REDC each
      out[crow * n + x] = csub(redc(a0l, a0h, m) + c0v[bb], m.q);
      out[(crow + 1) * n + x] = redc(a1l, a1h, m);
    }
  }
}

// K4 over a whole rotation sweep (bfv.hrot over several steps, bfv.py:467-500,
// with the step-independent digit NTTs of :485-497 hoisted): one launch writes
// every step's rotated ciphertexts. A thread owns one coefficient x of one limb
// for BCH ciphertexts and walks the steps; its ciphertexts' c0 and digit rows
// are fetched from HBM by the first step and re-gathered from L2 by the others
// (blocks are ordered x-fastest, then chunk, then limb, so the resident CTAs
// work on a few chunks of ONE limb: their digit rows and that limb's keys stay
// L2-resident). Step s+1's key words and gathers are issued before step s's
// multiply-accumulates (software pipelining keeps two steps of loads in flight).
constexpr int kKsMaxSteps = 32;
struct KsSteps {
  const uint64_t* keys[kKsMaxSteps];  // [L][ndig][2][n] Montgomery form, per step
  uint64_t* out[kKsMaxSteps];         // [B][L][2][n] per step
  uint32_t gpow[kKsMaxSteps];         // Galois element mod 2n per step
  int S;
};

template <int MAXD, int BCH>
struct KsLoads {
  uint64_t k0[MAXD], k1[MAXD], dv[BCH][MAXD], c0[BCH];
};

template <int MAXD, int BCH>
__device__ __forceinline__ void ks_issue(KsLoads<MAXD, BCH>& v, const KsSteps& A, int s, int logn, int L, int B,
                                         int ndig, int l, int b0, int x, uint32_t e,
                                         const uint64_t* __restrict__ ct, const uint64_t* __restrict__ dig) {
  const int n = 1 << logn;
  const uint32_t mask2n = 2u * (uint32_t)n - 1u;
  const uint32_t e2 = (e * A.gpow[s]) & mask2n;
  const int src = (int)brev_bits((e2 - 1u) >> 1, logn);
  const uint64_t* keys = A.keys[s];
#pragma unroll
  for (int i = 0; i < MAXD; ++i) {
    v.k0[i] = i < ndig ? __ldg(&keys[((size_t)(l * ndig + i) * 2 + 0) * n + x]) : 0;
    v.k1[i] = i < ndig ? __ldg(&keys[((size_t)(l * ndig + i) * 2 + 1) * n + x]) : 0;
  }
#pragma unroll
  for (int bb = 0; bb < BCH; ++bb) {
    const bool ok = b0 + bb < B;
    const size_t drow = ((size_t)(b0 + bb) * L + l) * ndig;
#pragma unroll
    for (int i = 0; i < MAXD; ++i) v.dv[bb][i] = (ok && i < ndig) ? __ldg(&dig[(drow + i) * n + src]) : 0;
    v.c0[bb] = ok ? __ldg(&ct[((size_t)(b0 + bb) * L + l) * 2 * n + src]) : 0;
  }
}

template <int MAXD, int BCH, bool W60>
__device__ __forceinline__ void ks_finish(const KsLoads<MAXD, BCH>& v, uint64_t* __restrict__ out, int logn, int L,
                                          int B, int ndig, int l, int b0, int x, const ModDesc& m) {
  const int n = 1 << logn;
#pragma unroll
  for (int bb = 0; bb < BCH; ++bb) {
    const int b = b0 + bb;
    if (b >= B) continue;
    uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0;
    if constexpr (W60 && MAXD <= 4) {  // Karatsuba 30-bit limbs (see Acc30)
      Acc30 s0, s1;
      acc30_zero(s0);
      acc30_zero(s1);
#pragma unroll
      for (int i = 0; i < MAXD; ++i) {
        if (i < ndig) {
          const Split30 u = split30(v.dv[bb][i]);
          mac30(s0, u, split30(v.k0[i]));
          mac30(s1, u, split30(v.k1[i]));
        }
      }
      acc30_get(s0, a0l, a0h);
      acc30_get(s1, a1l, a1h);
    } else if constexpr (W60) {
      Acc60 s0, s1;
      acc60_zero(s0);
      acc60_zero(s1);
#pragma unroll
      for (int i = 0; i < MAXD; ++i) {
        if (i < ndig) {
          mac60(s0, v.dv[bb][i], v.k0[i]);
          mac60(s1, v.dv[bb][i], v.k1[i]);
        }
      }
      acc60_get(s0, a0l, a0h);
      acc60_get(s1, a1l, a1h);
    } else {
#pragma unroll
      for (int i = 0; i < MAXD; ++i) {
        if (i < ndig) {
          mac128(a0l, a0h, v.dv[bb][i], v.k0[i]);
          mac128(a1l, a1h, v.dv[bb][i], v.k1[i]);
        }
      }
    }
    const size_t crow = ((size_t)b * L + l) * 2;
    out[crow * n + x] = csub(redc(a0l, a0h, m) + v.c0[bb], m.q);
    out[(crow + 1) * n + x] = redc(a1l, a1h, m);
  }
}

template <int MAXD, int BCH, bool W60>
__global__ void __launch_bounds__(128) keyswitch_multi_kernel(const ModSet ms, int logn, int L, int B, int ndig,
                                                              const __grid_constant__ KsSteps A,
                                                              const uint64_t* __restrict__ ct,
                                                              const uint64_t* __restrict__ dig) {
  const int n = 1 << logn;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int b0 = blockIdx.y * BCH;
  const int l = blockIdx.z;
  const ModDesc m = ms.m[l];
  const uint32_t e = 2u * brev_bits((uint32_t)x, logn) + 1u;  // exp_at_index[x] (ring.py:114-116)
  KsLoads<MAXD, BCH> cur, nxt;
  ks_issue<MAXD, BCH>(cur, A, 0, logn, L, B, ndig, l, b0, x, e, ct, dig);
  for (int s = 0; s < A.S; ++s) {
    if (s + 1 < A.S) ks_issue<MAXD, BCH>(nxt, A, s + 1, logn, L, B, ndig, l, b0, x, e, ct, dig);
    ks_finish<MAXD, BCH, W60>(cur, A.out[s], logn, L, B, ndig, l, b0, x, m);
    cur = nxt;
  }
}

// The default configuration (T = 16: four digits, every modulus below 2^60)
// of keyswitch_multi_kernel with the digit count and the Karatsuba MAC form
// fixed at compile time: no per-digit predicates, no load-buffer copies
// between steps (the generic kernel spent most of its issue slots on those),
// occupancy instead of software pipelining for the gather latency.
template <int BCH>
__global__ void __launch_bounds__(128) keyswitch_multi4_kernel(const ModSet ms, int logn, int L, int B,
                                                               const __grid_constant__ KsSteps A,
                                                               const uint64_t* __restrict__ ct,
                                                               const uint64_t* __restrict__ dig) {
  const uint32_t n = 1u << logn;
  const uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n) return;
  const int b0 = blockIdx.y * BCH;
  const int l = blockIdx.z;
  const ModDesc m = ms.m[l];
  const uint32_t e = 2u * brev_bits(x, logn) + 1u, mask2n = 2u * n - 1u;
  const uint64_t* drow[BCH];
  const uint64_t* crow[BCH];
  size_t orow[BCH];
#pragma unroll
  for (int bb = 0; bb < BCH; ++bb) {
    const size_t b = (size_t)min(b0 + bb, B - 1);  // clamped: loads stay in bounds, stores are guarded
    drow[bb] = dig + (b * L + l) * 4 * n;
    crow[bb] = ct + (b * L + l) * 2 * n;
    orow[bb] = (b * L + l) * 2 * n + x;
  }
  const size_t krow = (size_t)l * 8 * n + x;
#pragma unroll 1
  for (int s = 0; s < A.S; ++s) {
    const uint32_t e2 = (e * A.gpow[s]) & mask2n;
    const uint32_t src = brev_bits((e2 - 1u) >> 1, logn);
    const uint64_t* K = A.keys[s] + krow;
    uint64_t kv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) kv[i] = __ldg(K + (size_t)i * n);  // swk0_0, swk1_0, swk0_1, ...
    uint64_t dv[BCH][4], c0[BCH];
#pragma unroll
    for (int bb = 0; bb < BCH; ++bb) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dv[bb][i] = __ldg(drow[bb] + (size_t)i * n + src);
      c0[bb] = __ldg(crow[bb] + src);
    }
    Split30 k0[4], k1[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      k0[i] = split30(kv[2 * i]);
      k1[i] = split30(kv[2 * i + 1]);
    }
    uint64_t* out = A.out[s];
#pragma unroll
    for (int bb = 0; bb < BCH; ++bb) {
      Acc30 s0, s1;
      acc30_zero(s0);
      acc30_zero(s1);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const Split30 u = split30(dv[bb][i]);
        mac30(s0, u, k0[i]);
        mac30(s1, u, k1[i]);
      }
      uint64_t a0l, a0h, a1l, a1h;
      acc30_get(s0, a0l, a0h);
      acc30_get(s1, a1l, a1h);
      if (b0 + bb < B) {
        out[orow[bb]] = csub(redc(a0l, a0h, m) + c0[bb], m.q);
        out[orow[bb] + n] = redc(a1l, a1h, m);
      }
    }
  }
}

// ---------------------------------------------------------------- K4b
// Fused PMult-accumulate of the conventional convolution (conv.py:457-564):
// out[o][p] = Σ_{(r, w) in terms(o)} R[r][p] ⊙ PT[w]   (mod q, EVAL domain)
// One thread per (output ciphertext, slot): plaintexts are in Montgomery
// form, so each term is one 64x64 product and one REDC (canonical), both
// polys share the plaintext load, the sum stays in 128 bits and is reduced
// once — the per-term pmult/hadd ciphertexts of the reference never exist.
__global__ void __launch_bounds__(256) pmac_kernel(const ModDesc m, int n, const uint64_t* __restrict__ R,
                                                   const uint64_t* __restrict__ PT, const int* __restrict__ off,
                                                   const int2* __restrict__ terms, uint64_t* __restrict__ out) {
  const int o = blockIdx.y;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
  const int k0 = __ldg(&off[o]), k1 = __ldg(&off[o + 1]);
  for (int k = k0; k < k1; ++k) {
    const int2 t = __ldg(&terms[k]);
    const uint64_t w = __ldg(&PT[(size_t)t.y * n + i]);
    const uint64_t a = __ldg(&R[((size_t)t.x * 2) * n + i]), b = __ldg(&R[((size_t)t.x * 2 + 1) * n + i]);
    const uint64_t r0 = redc(a * w, __umul64hi(a, w), m), r1 = redc(b * w, __umul64hi(b, w), m);
    lo0 += r0;
    hi0 += lo0 < r0;
    lo1 += r1;
    hi1 += lo1 < r1;
  }
  out[((size_t)o * 2) * n + i] = barrett128(lo0, hi0, m);
  out[((size_t)o * 2 + 1) * n + i] = barrett128(lo1, hi1, m);
}

// ------------------------------------- K4c fused HRot x PMult x HAdd (north_star b)
// The conventional convolution's whole chain for one block of slots: each
// rotation group g (source ciphertext, Galois step) is key-switched in
// registers from the hoisted digits (bfv.hrot, bfv.py:467-500), multiplied by
// every encoded-weight plaintext that uses it and accumulated into the
// outputs' shared-memory accumulators — rotated ciphertexts never reach HBM.
// blockIdx.x: 64 slots; blockIdx.y: a tile of kRotOT outputs; blockIdx.z: a
// chunk of groups (partial sums into part[z] when gridDim.z > 1).
constexpr int kRotOT = 16, kRotX = 64, kRotMaxDig = 16;

__global__ void __launch_bounds__(kRotX) rot_pmac_kernel(const ModDesc m, int logn, int ndig, int G, int n_out,
                                                          int gchunk, const uint64_t* __restrict__ C,
                                                          const uint64_t* __restrict__ D,
                                                          const uint64_t* __restrict__ K,
                                                          const int2* __restrict__ groups,
                                                          const uint64_t* __restrict__ gpow,
                                                          const int* __restrict__ toff,
                                                          const int2* __restrict__ terms,
                                                          const uint64_t* __restrict__ PT, uint64_t* __restrict__ out) {
  __shared__ uint64_t acc[kRotOT][2][kRotX];
  const int n = 1 << logn;
  const int tid = threadIdx.x, x = blockIdx.x * kRotX + tid;
  const int tile = blockIdx.y, o0 = tile * kRotOT;
  const int g0 = blockIdx.z * gchunk, g1 = min(G, g0 + gchunk);
#pragma unroll
  for (int o = 0; o < kRotOT; ++o) acc[o][0][tid] = acc[o][1][tid] = 0;
  const uint64_t q = m.q;
  const int* offs = toff + (size_t)tile * (G + 1);
  for (int g = g0; g < g1; ++g) {
    const int t0 = __ldg(&offs[g]), t1 = __ldg(&offs[g + 1]);
    if (t0 == t1) continue;  // no output of this tile uses the rotation (block-uniform)
    const int2 gi = __ldg(&groups[g]);
    const uint64_t* c = C + (size_t)gi.x * 2 * n;
    uint64_t r0, r1;
    if (gi.y < 0) {  // step 0: the ciphertext itself
      r0 = c[x];
      r1 = c[n + x];
    } else {
      // eval_perm (ring.py:199-202): exp_at_index[x] = 2 bitrev(x) + 1
      const uint64_t mask2n = 2ull * n - 1;  // mod 2n as a mask (n is a power of two)
      const uint64_t gp = __ldg(&gpow[g]) & mask2n;
      const uint32_t e = 2u * brev_bits((uint32_t)x, logn) + 1u;
      const uint32_t e2 = (uint32_t)(((uint64_t)e * gp) & mask2n);
      const int src = (int)brev_bits((e2 - 1u) >> 1, logn);
      const uint64_t* dg = D + (size_t)gi.x * ndig * n;
      const uint64_t* kk = K + (size_t)gi.y * ndig * 2 * n;
      uint64_t a0l = 0, a0h = 0, a1l = 0, a1h = 0;
#pragma unroll 4
      for (int i = 0; i < ndig; ++i) {
        const uint64_t dv = __ldg(&dg[(size_t)i * n + src]);
        mac128(a0l, a0h, dv, __ldg(&kk[((size_t)i * 2) * n + x]));
        mac128(a1l, a1h, dv, __ldg(&kk[((size_t)i * 2 + 1) * n + x]));
      }
      r0 = csub(redc(a0l, a0h, m) + c[src], q);  // ndig q^2 < q 2^64: one REDC each
      r1 = redc(a1l, a1h, m);
    }
    for (int t = t0; t < t1; ++t) {
      const int2 tm = __ldg(&terms[t]);  // (output within the tile, plaintext row)
      const uint64_t w = __ldg(&PT[(size_t)tm.y * n + x]);  // Montgomery form: redc(r w) = r w_plain
      acc[tm.x][0][tid] = csub(acc[tm.x][0][tid] + redc(r0 * w, __umul64hi(r0, w), m), q);
      acc[tm.x][1][tid] = csub(acc[tm.x][1][tid] + redc(r1 * w, __umul64hi(r1, w), m), q);
    }
  }
  uint64_t* dst = out + (size_t)blockIdx.z * n_out * 2 * n;
  for (int o = 0; o < kRotOT && o0 + o < n_out; ++o) {
    dst[((size_t)(o0 + o) * 2) * n + x] = acc[o][0][tid];
    dst[((size_t)(o0 + o) * 2 + 1) * n + x] = acc[o][1][tid];
  }
}

// out = Σ_z part[z] mod q (partial sums of the group chunks)
__global__ void rot_pmac_reduce_kernel(uint64_t q, int Z, int64_t total, const uint64_t* __restrict__ part,
                                       uint64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  uint64_t s = 0;
  for (int z = 0; z < Z; ++z) s = csub(s + part[(size_t)z * total + i], q);
  out[i] = s;
}

}  // namespace fhe

using namespace fhe;

extern "C" {

int fhe_poly_binary(int op, const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a,
                    const uint64_t* b, int Bb, int Pb, uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  if (op < 0 || op > 2) return fail(FHE_ERR_VALUE, "bad op %d", op);
  if (!(Bb == 1 || Bb == B) || !(Pb == 1 || Pb == P) || Bb < 1) return fail(FHE_ERR_VALUE, "bad broadcast");
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  const int64_t total2 = (int64_t)B * L * P * n / 2;
  if (!total2) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  binary_kernel<<<grid_for(total2), kThreads, 0, (cudaStream_t)stream>>>(op, ms, g, B, Bb, Pb, a, b, out, total2);
  FHE_CHECK_LAUNCH("binary_kernel");
  return FHE_OK;
}

int fhe_poly_mul_shoup(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a, const uint64_t* w,
                       const uint64_t* w_shoup, int Bb, int Pb, uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  if (!(Bb == 1 || Bb == B) || !(Pb == 1 || Pb == P) || Bb < 1) return fail(FHE_ERR_VALUE, "bad broadcast");
  if ((int64_t)B * L * P >= ((int64_t)1 << 31)) return fail(FHE_ERR_VALUE, "too many rows");
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  for (int l = 0; l < L; ++l)
    if (ms.m[l].q >= (1ull << 63)) return fail(FHE_ERR_PARAMETER, "Shoup multiply needs q < 2^63");
  const int64_t total2 = (int64_t)B * L * P * n / 2;
  if (!total2) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  if (Bb == 1 && B > 1 && (B + 3) / 4 <= 65535) {
    constexpr int bch = 4;
    const int64_t inner2 = (int64_t)L * P * n / 2;
    dim3 grid((unsigned)((inner2 + kThreads - 1) / kThreads), (unsigned)((B + bch - 1) / bch));
    mul_shoup_bcast_kernel<bch><<<grid, kThreads, 0, (cudaStream_t)stream>>>(ms, g.logn, L, P, Pb, B, a, w, w_shoup,
                                                                             out, inner2);
    FHE_CHECK_LAUNCH("mul_shoup_bcast_kernel");
    return FHE_OK;
  }
  mul_shoup_kernel<<<grid_for(total2), kThreads, 0, (cudaStream_t)stream>>>(ms, g, Bb, Pb, a, w, w_shoup, out,
                                                                             total2);
  FHE_CHECK_LAUNCH("mul_shoup_kernel");
  return FHE_OK;
}

int fhe_shoup_companions(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* w, uint64_t* w_shoup,
                         void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  const int64_t total = (int64_t)B * L * P * n;
  if (!total) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  shoup_companion_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms, g, w, w_shoup, total);
  FHE_CHECK_LAUNCH("shoup_companion_kernel");
  return FHE_OK;
}

int fhe_poly_neg(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a, uint64_t* out,
                 void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  const int64_t total = (int64_t)B * L * P * n;
  if (!total) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  neg_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms, g, a, out, total);
  FHE_CHECK_LAUNCH("neg_kernel");
  return FHE_OK;
}

int fhe_poly_scalar_mul(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a,
                        const uint64_t* k_per_limb, uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  Scalars sc;
  for (int l = 0; l < L; ++l) {
    uint64_t k = k_per_limb[l] % ms.m[l].q;
    sc.k[l] = k;
    sc.kp[l] = h_shoup(k, ms.m[l].q);
  }
  const int64_t total = (int64_t)B * L * P * n;
  if (!total) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  scalar_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms, g, sc, a, out, total);
  FHE_CHECK_LAUNCH("scalar_kernel");
  return FHE_OK;
}

int fhe_poly_monomial(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a,
                      int64_t shift, uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  if (a == out) return fail(FHE_ERR_VALUE, "monomial_mul cannot run in place");
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  int64_t s = shift % (2 * (int64_t)n);
  if (s < 0) s += 2 * (int64_t)n;
  int flip = s >= n;
  if (flip) s -= n;
  const int64_t total = (int64_t)B * L * P * n;
  if (!total) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  monomial_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms, g, s, flip, a, out, total);
  FHE_CHECK_LAUNCH("monomial_kernel");
  return FHE_OK;
}

int fhe_residual_add(uint64_t q, int count, int c_n, int tile, int n, const uint64_t* y, const uint64_t* a,
                     uint64_t* out, void* stream) {
  if (n <= 0 || (n & (n - 1)) || count < 0 || c_n < 1 || tile < 0 || (int64_t)tile * c_n > n)
    return fail(FHE_ERR_VALUE, "residual_add: bad geometry");
  if (!q || q >= (1ull << 62)) return fail(FHE_ERR_VALUE, "residual_add: modulus out of range");
  if (a == out) return fail(FHE_ERR_VALUE, "residual_add: the shortcut cannot alias the output");
  const int64_t total = (int64_t)count * 2 * n;
  if (!total) return FHE_OK;
  residual_add_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(q, log2i(n), c_n, tile, y, a, out,
                                                                              total);
  FHE_CHECK_LAUNCH("residual_add_kernel");
  return FHE_OK;
}

int fhe_poly_automorphism(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a,
                          uint64_t gpow, uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  if (!(gpow & 1)) return fail(FHE_ERR_PARAMETER, "Galois element must be odd");
  if (a == out) return fail(FHE_ERR_VALUE, "automorphism cannot run in place");
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  const int64_t total = (int64_t)B * L * P * n;
  if (!total) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  automorphism_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms, g, gpow, a, out, total);
  FHE_CHECK_LAUNCH("automorphism_kernel");
  return FHE_OK;
}

int fhe_poly_add_delta(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const uint64_t* base,
                       const int64_t* m, uint64_t* out, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (p < 2 || (u128_t)delta * (p - 1) >= q) return fail(FHE_ERR_PARAMETER, "delta*(p-1) must be < q");
  const int64_t total = (int64_t)R * n;
  if (total <= 0) return FHE_OK;
  add_delta_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms.m[0], p, delta, base, m, out, total);
  FHE_CHECK_LAUNCH("add_delta_kernel");
  return FHE_OK;
}

int fhe_encrypt_combine(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const int64_t* m,
                        const uint64_t* as, const int64_t* e, uint64_t* out, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (p < 2 || (u128_t)delta * (p - 1) >= q) return fail(FHE_ERR_PARAMETER, "delta*(p-1) must be < q");
  const int64_t total = (int64_t)R * n;
  if (total <= 0) return FHE_OK;
  encrypt_combine_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms.m[0], p, delta, m, as, e,
                                                                                   out, total);
  FHE_CHECK_LAUNCH("encrypt_combine_kernel");
  return FHE_OK;
}

int fhe_poly_lift_centered(uint64_t p, uint64_t q, int R, int n, const int64_t* v, uint64_t* out,
                           void* stream) {
  if (p < 2 || q < p) return fail(FHE_ERR_PARAMETER, "bad moduli for lift");
  const int64_t total = (int64_t)R * n;
  if (total <= 0) return FHE_OK;
  lift_centered_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(p, q, v, out, total);
  FHE_CHECK_LAUNCH("lift_centered_kernel");
  return FHE_OK;
}

int fhe_to_montgomery(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a,
                      uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, P, n)) return rc;
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  const int64_t total = (int64_t)B * L * P * n;
  if (!total) return FHE_OK;
  RowGeom g{L, P, log2i(n)};
  to_mont_kernel<<<grid_for(total), kThreads, 0, (cudaStream_t)stream>>>(ms, g, a, out, total);
  FHE_CHECK_LAUNCH("to_mont_kernel");
  return FHE_OK;
}

int fhe_wide_accumulate(int n, const uint64_t* f, int64_t scalar, int64_t* lo, int64_t* hi, void* stream) {
  if (n < 1 || !f || !lo || !hi) return fail(FHE_ERR_VALUE, "bad wide accumulate arguments");
  wide_acc_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, f, nullptr, nullptr, scalar, lo, hi);
  FHE_CHECK_LAUNCH("wide_acc_kernel");
  return FHE_OK;
}

int fhe_wide_accumulate_split(int n, const int64_t* flo, const int64_t* fhi, int64_t scalar, int64_t* lo,
                              int64_t* hi, void* stream) {
  if (n < 1 || !flo || !fhi || !lo || !hi) return fail(FHE_ERR_VALUE, "bad wide accumulate arguments");
  wide_acc_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, nullptr, flo, fhi, scalar, lo, hi);
  FHE_CHECK_LAUNCH("wide_acc_kernel");
  return FHE_OK;
}

int fhe_wide_add_rotated(int n, const int64_t* olo, const int64_t* ohi, int64_t shift, int64_t* lo, int64_t* hi,
                         void* stream) {
  if (n < 1 || !olo || !ohi || !lo || !hi) return fail(FHE_ERR_VALUE, "bad wide rotate arguments");
  if (olo == lo || ohi == hi) return fail(FHE_ERR_VALUE, "add_rotated source must not alias the accumulator");
  int64_t s = shift % (2 * (int64_t)n);
  if (s < 0) s += 2 * (int64_t)n;
  int flip = s >= n;
  if (flip) s -= n;
  wide_rot_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, olo, ohi, (int)s, flip, lo, hi);
  FHE_CHECK_LAUNCH("wide_rot_kernel");
  return FHE_OK;
}

int fhe_wide_finalize(int n, uint64_t q, const int64_t* lo, const int64_t* hi, uint64_t* out, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (n < 1 || !lo || !hi || !out) return fail(FHE_ERR_VALUE, "bad wide finalize arguments");
  const uint64_t w30 = (1ull << 30) % q;
  wide_fin_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(n, ms.m[0], w30, h_shoup(w30, q), lo, hi,
                                                                        out);
  FHE_CHECK_LAUNCH("wide_fin_kernel");
  return FHE_OK;
}

int fhe_decrypt_round(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const uint64_t* u,
                      uint64_t* m_out, uint64_t* maxw_out, void* stream) {
  if (R < 0 || n < 1 || delta < 2 || p < 2) return fail(FHE_ERR_VALUE, "bad decrypt arguments");
  if (q >= (1ull << 62)) return fail(FHE_ERR_PARAMETER, "modulus too large");
  if (!R) return FHE_OK;
  const uint64_t magic = ~0ull / delta;
  decrypt_round_kernel<<<R, 256, 0, (cudaStream_t)stream>>>(p, delta, magic, n, u, m_out, maxw_out, nullptr);
  FHE_CHECK_LAUNCH("decrypt_round_kernel");
  return FHE_OK;
}

int fhe_decrypt_round_max(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const uint64_t* u,
                          uint64_t* m_out, uint64_t* max_all, void* stream) {
  if (R < 0 || n < 1 || delta < 2 || p < 2 || !max_all) return fail(FHE_ERR_VALUE, "bad decrypt arguments");
  if (q >= (1ull << 62)) return fail(FHE_ERR_PARAMETER, "modulus too large");
  if (!R) return FHE_OK;
  const uint64_t magic = ~0ull / delta;
  decrypt_round_kernel<<<R, 256, 0, (cudaStream_t)stream>>>(p, delta, magic, n, u, m_out, nullptr,
                                                            reinterpret_cast<unsigned long long*>(max_all));
  FHE_CHECK_LAUNCH("decrypt_round_kernel");
  return FHE_OK;
}

int fhe_act_client_square(uint64_t p, int f, int64_t count, const uint64_t* w, uint64_t* y, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&p, 1, &ms)) return rc;
  if (f < 0 || f > 62) return fail(FHE_ERR_VALUE, "bad fraction bits %d", f);
  if (count <= 0) return FHE_OK;
  const uint64_t two_f = h_powmod(2, (uint64_t)f, p);
  act_client_kernel<<<grid_for(count), kThreads, 0, (cudaStream_t)stream>>>(ms.m[0], two_f, w, y, count);
  FHE_CHECK_LAUNCH("act_client_kernel");
  return FHE_OK;
}

int fhe_act_server_const(uint64_t p, int f, int64_t count, const uint64_t* r, const uint64_t* r_sq,
                         const uint64_t* v, uint64_t* c, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&p, 1, &ms)) return rc;
  if (f < 0 || f > 62) return fail(FHE_ERR_VALUE, "bad fraction bits %d", f);
  if (count <= 0) return FHE_OK;
  const uint64_t two_f = h_powmod(2, (uint64_t)f, p);
  act_server_kernel<<<grid_for(count), kThreads, 0, (cudaStream_t)stream>>>(ms.m[0], two_f, r, r_sq, v, c,
                                                                              count);
  FHE_CHECK_LAUNCH("act_server_kernel");
  return FHE_OK;
}

int fhe_keyswitch_apply(const uint64_t* moduli, int L, int B, int n, const uint64_t* ct,
                        const uint64_t* digits, const uint64_t* keys_mont, int ndig, uint64_t gpow,
                        uint64_t* out, void* stream) {
  if (int rc = check_rows(L, B, 2, n)) return rc;
  if (ndig < 1 || ndig > 64) return fail(FHE_ERR_VALUE, "bad digit count %d", ndig);
  if (!(gpow & 1)) return fail(FHE_ERR_PARAMETER, "Galois element must be odd");
  if (ct == out) return fail(FHE_ERR_VALUE, "keyswitch cannot run in place");
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  for (int l = 0; l < L; ++l)
    if ((u128_t)ndig * ms.m[l].q >= ((u128_t)1 << 64))
      return fail(FHE_ERR_PARAMETER, "too many digits for one lazy REDC");
  if (!B) return FHE_OK;
#ifndef FHE_KS_BCH
#define FHE_KS_BCH 2
#endif
  // key words reused by bchunk ciphertexts; bchunk x (ndig + 1) gathers in flight
  // per thread (chunk shrinks with the digit count to bound registers)
  constexpr int bchunk = FHE_KS_BCH;
  constexpr int bch8 = bchunk > 2 ? bchunk / 2 : 1, bch16 = bchunk > 4 ? bchunk / 4 : 1;
  const int bch = ndig <= 4 ? bchunk : ndig <= 8 ? bch8 : bch16;
  dim3 grid((n + 127) / 128, L, (B + bch - 1) / bch);
  const int logn = log2i(n);
  cudaStream_t st = (cudaStream_t)stream;
  bool w60 = ndig <= 8;  // column-split MACs need every modulus below 2^60
  for (int l = 0; l < L; ++l) w60 = w60 && ms.m[l].q < (1ull << 60);
  if (ndig <= 4 && w60)
    keyswitch_kernel<4, bchunk, true><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, gpow, ct, digits, keys_mont, out);
  else if (ndig <= 4)
    keyswitch_kernel<4, bchunk, false><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, gpow, ct, digits, keys_mont, out);
  else if (ndig <= 8 && w60)
    keyswitch_kernel<8, bch8, true><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, gpow, ct, digits, keys_mont, out);
  else if (ndig <= 8)
    keyswitch_kernel<8, bch8, false><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, gpow, ct, digits, keys_mont, out);
  else if (ndig <= 16)
    keyswitch_kernel<16, bch16, false><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, gpow, ct, digits, keys_mont, out);
  else
    return fail(FHE_ERR_VALUE, "more than 16 digits unsupported");
  FHE_CHECK_LAUNCH("keyswitch_kernel");
  return FHE_OK;
}

static bool ks_multi4() {  // FHE_KS_MULTI4=0 selects the generic multi-step kernel (A/B checks)
  static int v = -1;
  if (v < 0) {
    const char* s = getenv("FHE_KS_MULTI4");
    v = (s && s[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int fhe_keyswitch_multi(const uint64_t* moduli, int L, int B, int n, const uint64_t* ct, const uint64_t* digits,
                        int ndig, int S, const uint64_t* const* keys_mont, const uint64_t* gpows,
                        uint64_t* const* outs, void* stream) {
  if (int rc = check_rows(L, B, 2, n)) return rc;
  if (ndig < 1 || ndig > 8) return fail(FHE_ERR_VALUE, "multi-step key switch takes 1..8 digits, got %d", ndig);
  if (S < 0 || (S && (!keys_mont || !gpows || !outs))) return fail(FHE_ERR_VALUE, "bad step list");
  ModSet ms;
  if (int rc = make_modset(moduli, L, &ms)) return rc;
  for (int l = 0; l < L; ++l)
    if ((u128_t)ndig * ms.m[l].q >= ((u128_t)1 << 64))
      return fail(FHE_ERR_PARAMETER, "too many digits for one lazy REDC");
  for (int s = 0; s < S; ++s) {
    if (!(gpows[s] & 1)) return fail(FHE_ERR_PARAMETER, "Galois element must be odd");
    if (!keys_mont[s] || !outs[s]) return fail(FHE_ERR_VALUE, "null key or output of step %d", s);
    if (outs[s] == ct) return fail(FHE_ERR_VALUE, "keyswitch cannot run in place");
  }
  if (!B || !S) return FHE_OK;
  bool w60 = true;  // column-split MACs need every modulus below 2^60
  for (int l = 0; l < L; ++l) w60 = w60 && ms.m[l].q < (1ull << 60);
  const int logn = log2i(n);
  cudaStream_t st = (cudaStream_t)stream;
#ifndef FHE_KSM_BCH
#define FHE_KSM_BCH 2
#endif
  constexpr int bch = FHE_KSM_BCH;
  const dim3 grid((n + 127) / 128, (B + bch - 1) / bch, L);
  for (int s0 = 0; s0 < S; s0 += kKsMaxSteps) {
    KsSteps A;
    A.S = std::min(kKsMaxSteps, S - s0);
    for (int s = 0; s < A.S; ++s) {
      A.keys[s] = keys_mont[s0 + s];
      A.out[s] = outs[s0 + s];
      A.gpow[s] = (uint32_t)(gpows[s0 + s] & (2ull * n - 1));
    }
    if (ndig == 4 && w60 && ks_multi4())
      keyswitch_multi4_kernel<bch><<<grid, 128, 0, st>>>(ms, logn, L, B, A, ct, digits);
    else if (ndig <= 4 && w60)
      keyswitch_multi_kernel<4, bch, true><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, A, ct, digits);
    else if (ndig <= 4)
      keyswitch_multi_kernel<4, bch, false><<<grid, 128, 0, st>>>(ms, logn, L, B, ndig, A, ct, digits);
    else if (w60)
      keyswitch_multi_kernel<8, 1, true><<<dim3((n + 127) / 128, B, L), 128, 0, st>>>(ms, logn, L, B, ndig, A, ct,
                                                                                       digits);
    else
      keyswitch_multi_kernel<8, 1, false><<<dim3((n + 127) / 128, B, L), 128, 0, st>>>(ms, logn, L, B, ndig, A, ct,
                                                                                        digits);
    FHE_CHECK_LAUNCH("keyswitch_multi_kernel");
  }
  return FHE_OK;
}

int fhe_pmac(uint64_t q, int n, const uint64_t* R, const uint64_t* pt_mont, const int32_t* term_off,
             const int32_t* terms, int n_out, uint64_t* out, void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (n < 1 || n_out < 0 || !R || !pt_mont || !term_off || !terms || !out) return fail(FHE_ERR_VALUE, "bad pmac arguments");
  if (!n_out) return FHE_OK;
  dim3 grid((n + 255) / 256, n_out);
  pmac_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ms.m[0], n, R, pt_mont, term_off,
                                                       reinterpret_cast<const int2*>(terms), out);
  FHE_CHECK_LAUNCH("pmac_kernel");
  return FHE_OK;
}

int fhe_rot_pmac(uint64_t q, int n, int ndig, const uint64_t* C, const uint64_t* D, const uint64_t* K_mont,
                 int G, const int32_t* groups, const uint64_t* gpow, int n_out, const int32_t* tile_off,
                 const int32_t* terms, const uint64_t* pt_mont, int gchunks, uint64_t* partial, uint64_t* out,
                 void* stream) {
  ModSet ms;
  if (int rc = make_modset(&q, 1, &ms)) return rc;
  if (n < kRotX || (n & (n - 1)) || ndig < 1 || ndig > kRotMaxDig || G < 0 || n_out < 0 || gchunks < 1)
    return fail(FHE_ERR_VALUE, "bad rot_pmac geometry");
  if ((u128_t)ndig * q >= ((u128_t)1 << 64)) return fail(FHE_ERR_PARAMETER, "too many digits for one lazy REDC");
  if (!n_out) return FHE_OK;
  if (!C || !groups || !gpow || !tile_off || !terms || !pt_mont || !out || (G && (!D || !K_mont)))
    return fail(FHE_ERR_VALUE, "null rot_pmac operand");
  if (gchunks > 1 && !partial) return fail(FHE_ERR_VALUE, "rot_pmac with group chunks needs a partial buffer");
  const int tiles = (n_out + kRotOT - 1) / kRotOT;
  const int gchunk = G ? (G + gchunks - 1) / gchunks : 1;
  const int Z = G ? (G + gchunk - 1) / gchunk : 1;
  dim3 grid(n / kRotX, tiles, Z);
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t* dst = Z > 1 ? partial : out;
  rot_pmac_kernel<<<grid, kRotX, 0, st>>>(ms.m[0], log2i(n), ndig, G, n_out, gchunk, C, D, K_mont,
                                          reinterpret_cast<const int2*>(groups), gpow, tile_off,
                                          reinterpret_cast<const int2*>(terms), pt_mont, dst);
  FHE_CHECK_LAUNCH("rot_pmac_kernel");
  if (Z > 1) {
    const int64_t total = (int64_t)n_out * 2 * n;
    rot_pmac_reduce_kernel<<<grid_for(total), kThreads, 0, st>>>(q, Z, total, partial, out);
    FHE_CHECK_LAUNCH("rot_pmac_reduce_kernel");
  }
  return FHE_OK;
}

int fhe_gather_rows(const uint64_t* const* srcs, int k, int n, uint64_t* dst, void* stream) {
  if (k < 0 || n < 1 || (k && (!srcs || !dst))) return fail(FHE_ERR_VALUE, "bad gather arguments");
  for (int r0 = 0; r0 < k; r0 += kGatherPtrs) {
    GatherPtrs P;
    const int cnt = std::min(kGatherPtrs, k - r0);
    for (int r = 0; r < cnt; ++r) {
      if (!srcs[r0 + r]) return fail(FHE_ERR_VALUE, "null source row %d", r0 + r);
      P.src[r] = srcs[r0 + r];
    }
    const int bx = std::min(8, (n + 255) / 256);
    gather_rows_kernel<<<dim3(bx, cnt), 256, 0, (cudaStream_t)stream>>>(P, n, dst + (size_t)r0 * n);
    FHE_CHECK_LAUNCH("gather_rows_kernel");
  }
  return FHE_OK;
}

int fhe_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                void* stream) {
  if (!height || !width) return FHE_OK;
  if (!dst || !src) return fail(FHE_ERR_VALUE, "null copy operand");
  FHE_CUDA(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, cudaMemcpyDeviceToDevice,
                             (cudaStream_t)stream));
  return FHE_OK;
}

int fhe_copy_many(int count, const void* const* srcs, void* const* dsts, const size_t* bytes, void* stream) {
  // several device-to-device copies (8-byte multiples, 8-byte aligned) in ONE launch: the
  // act2pc layer graph's operand refill (seven buffers) costs one kernel instead of seven
  // memcpy nodes
  if (count < 0 || count > fhe::kCopyMany) return fail(FHE_ERR_VALUE, "copy count %d out of range", count);
  if (!count) return FHE_OK;
  if (!srcs || !dsts || !bytes) return fail(FHE_ERR_VALUE, "null copy table");
  fhe::CopyTable t{};
  t.count = count;
  unsigned long long total = 0;
  for (int i = 0; i < count; ++i) {
    if (bytes[i] % 8 || ((uintptr_t)srcs[i] | (uintptr_t)dsts[i]) % 8) return fail(FHE_ERR_VALUE, "unaligned copy %d", i);
    if (bytes[i] && (!srcs[i] || !dsts[i])) return fail(FHE_ERR_VALUE, "null copy operand %d", i);
    t.src[i] = static_cast<const uint64_t*>(srcs[i]);
    t.dst[i] = static_cast<uint64_t*>(dsts[i]);
    t.start[i] = total;
    total += bytes[i] / 8;
  }
  t.start[count] = total;
  if (!total) return FHE_OK;
  const int threads = 256;
  const unsigned long long blocks = std::min<unsigned long long>((total + threads - 1) / threads, 148ull * 16);
  fhe::copy_many_kernel<<<(unsigned)blocks, threads, 0, (cudaStream_t)stream>>>(t);
  FHE_CHECK_LAUNCH("copy_many_kernel");
  return FHE_OK;
}

int fhe_zero(void* dst, size_t bytes, void* stream) {
  if (!bytes) return FHE_OK;
  if (!dst) return fail(FHE_ERR_VALUE, "null zero operand");
  FHE_CUDA(cudaMemsetAsync(dst, 0, bytes, (cudaStream_t)stream));
  return FHE_OK;
}

}  // extern "C"
