// act.cu — K5 over a whole layer: the x^2+x share protocol (SPEC.md:304-331,
// PAPER.md:873-895) on row stacks [k][2][n], plus the client-side repack of a
// conv output into the next layer's tile layout (conv.py:148-197).
//
// Every step is one HBM pass over the layer's ciphertexts; the repack and the
// batch-slot permutation are index gathers (precomputed public maps), so the
// client's decrypt -> square -> encrypt chain never leaves the device.
#include "common.cuh"

namespace fhe {

static constexpr int kActThreads = 256;

static inline unsigned act_grid(int64_t work) {
  int64_t g = (work + kActThreads - 1) / kActThreads;
  return (unsigned)(g < 1 ? 1 : g);
}

static int act_logn(int n) {
  if (n < 2 || (n & (n - 1)) || n > (1 << FHE_MAX_LOGN)) return -1;
  int lg = 0;
  while ((1 << lg) < n) ++lg;
  return lg;
}

// out[i] = src[idx[i]] (0 where idx < 0): the repack map composes
// channel_positions of the conv output (stride applied) with pack_vectors of
// the next layout, so zero borders / halos come out right in one pass.
__global__ void act_gather_kernel(const int32_t* __restrict__ idx, const uint64_t* __restrict__ src,
                                  uint64_t* __restrict__ out, int64_t total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int32_t s = idx[i];
  out[i] = s >= 0 ? src[s] : 0;
}

// encrypt_online over rows (bfv.py:248-263), optional client square
// (SPEC.md:313-316): v = m[r][perm ? perm[s] : s]; v <- v^2 + v 2^f (square);
// c0 = zero.c0 + Δ v mod q, c1 = zero.c1.
__global__ void act_encrypt_kernel(ModDesc mq, ModDesc mp, uint64_t delta, uint64_t two_f, int square, int logn,
                                   const uint64_t* __restrict__ zero, const uint64_t* __restrict__ m,
                                   const int32_t* __restrict__ perm, uint64_t* __restrict__ out, int64_t total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t r = i >> logn;
  const int n = 1 << logn, s = (int)(i & (n - 1));
  uint64_t v = reduce_u64(m[(r << logn) + (perm ? perm[s] : s)], mp);
  if (square) v = csub(mulmod(v, v, mp) + mulmod(v, two_f, mp), mp.q);
  const int64_t base = r << (logn + 1);
  out[base + s] = csub(zero[base + s] + delta * v, mq.q);  // Δ (p-1) < q
  out[base + n + s] = zero[base + n + s];
}

// pmult + plain_add in EVAL (bfv.py:330-372): out.c0 = c0 ⊙ pt + add, out.c1 = c1 ⊙ pt.
__global__ void ct_pmult_add_kernel(ModDesc mq, int logn, const uint64_t* __restrict__ ct,
                                    const uint64_t* __restrict__ pt, const uint64_t* __restrict__ add,
                                    uint64_t* __restrict__ out, int64_t total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t r = i >> logn;
  const int n = 1 << logn, s = (int)(i & (n - 1));
  const int64_t base = r << (logn + 1);
  const uint64_t b = pt[i];
  uint64_t o0 = mulmod(ct[base + s], b, mq);
  if (add) o0 = csub(o0 + add[i], mq.q);
  out[base + s] = o0;
  out[base + n + s] = mulmod(ct[base + n + s], b, mq);
}

// server_finalize: psub(ct1, ct2) then plain_add(Δ c).
__global__ void act_finalize_kernel(ModDesc mq, ModDesc mp, uint64_t delta, int logn, const uint64_t* __restrict__ a,
                                    const uint64_t* __restrict__ b, const uint64_t* __restrict__ c,
                                    uint64_t* __restrict__ out, int64_t total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t r = i >> logn;
  const int n = 1 << logn, s = (int)(i & (n - 1));
  const int64_t base = r << (logn + 1);
  const uint64_t q = mq.q;
  const uint64_t d0 = csub(a[base + s] + q - b[base + s], q);
  out[base + s] = csub(d0 + delta * reduce_u64(c[i], mp), q);
  out[base + n + s] = csub(a[base + n + s] + q - b[base + n + s], q);
}

// act_encrypt_kernel with the message gathered by a full index map
// (m_val = m[gidx[i]]): the client's repack gather and the encryption of the
// repacked values in one pass (no gathered intermediate)
__global__ void act_encrypt_gather_kernel(ModDesc mq, ModDesc mp, uint64_t delta, uint64_t two_f, int square,
                                          int logn, const uint64_t* __restrict__ zero,
                                          const uint64_t* __restrict__ m, const int32_t* __restrict__ gidx,
                                          uint64_t* __restrict__ out, int64_t total) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t r = i >> logn;
  const int n = 1 << logn, s = (int)(i & (n - 1));
  const int32_t g = gidx[i];
  uint64_t v = reduce_u64(g >= 0 ? m[g] : 0, mp);  // (act_gather: a slot with no source reads 0)
  if (square) v = csub(mulmod(v, v, mp) + mulmod(v, two_f, mp), mp.q);
  const int64_t base = r << (logn + 1);
  out[base + s] = csub(zero[base + s] + delta * v, mq.q);  // Δ (p-1) < q
  out[base + n + s] = zero[base + n + s];
}

}  // namespace fhe

using namespace fhe;

static int act_moduli(uint64_t q, uint64_t p, uint64_t delta, ModSet* mq, ModSet* mp) {
  if (int rc = make_modset(&q, 1, mq)) return rc;
  if (int rc = make_modset(&p, 1, mp)) return rc;
  if ((u128_t)delta * (p - 1) >= q) return fail(FHE_ERR_PARAMETER, "delta*(p-1) must be < q");
  return FHE_OK;
}

extern "C" {

int fhe_act_gather(int64_t count, const int32_t* idx, const uint64_t* src, uint64_t* out, void* stream) {
  if (count < 0) return fail(FHE_ERR_VALUE, "negative gather count");
  if (!count) return FHE_OK;
  if (!idx || !src || !out) return fail(FHE_ERR_VALUE, "null gather pointer");
  act_gather_kernel<<<act_grid(count), kActThreads, 0, (cudaStream_t)stream>>>(idx, src, out, count);
  FHE_CHECK_LAUNCH("act_gather_kernel");
  return FHE_OK;
}

int fhe_act_encrypt_rows(uint64_t q, uint64_t p, uint64_t delta, int f, int square, int R, int n,
                         const uint64_t* zero, const uint64_t* m, const int32_t* perm, uint64_t* out,
                         void* stream) {
  ModSet mq, mp;
  if (int rc = act_moduli(q, p, delta, &mq, &mp)) return rc;
  const int logn = act_logn(n);
  if (logn < 0 || R < 0) return fail(FHE_ERR_VALUE, "bad row geometry (R=%d n=%d)", R, n);
  if (f < 0 || f > 62) return fail(FHE_ERR_VALUE, "bad fraction bits %d", f);
  if (!R) return FHE_OK;
  if (!zero || !m || !out) return fail(FHE_ERR_VALUE, "null encrypt pointer");
  if (out == zero) return fail(FHE_ERR_VALUE, "encrypt output must not alias the zero ciphertexts");
  const int64_t total = (int64_t)R << logn;
  act_encrypt_kernel<<<act_grid(total), kActThreads, 0, (cudaStream_t)stream>>>(
      mq.m[0], mp.m[0], delta, h_powmod(2, (uint64_t)f, p), square, logn, zero, m, perm, out, total);
  FHE_CHECK_LAUNCH("act_encrypt_kernel");
  return FHE_OK;
}

int fhe_act_encrypt_gather(uint64_t q, uint64_t p, uint64_t delta, int f, int square, int R, int n,
                           const uint64_t* zero, const uint64_t* m, const int32_t* gidx, uint64_t* out,
                           void* stream) {
  ModSet mq, mp;
  if (int rc = act_moduli(q, p, delta, &mq, &mp)) return rc;
  const int logn = act_logn(n);
  if (logn < 0 || R < 0) return fail(FHE_ERR_VALUE, "bad row geometry (R=%d n=%d)", R, n);
  if (f < 0 || f > 62) return fail(FHE_ERR_VALUE, "bad fraction bits %d", f);
  if (!R) return FHE_OK;
  if (!zero || !m || !gidx || !out) return fail(FHE_ERR_VALUE, "null encrypt pointer");
  if (out == zero) return fail(FHE_ERR_VALUE, "encrypt output must not alias the zero ciphertexts");
  const int64_t total = (int64_t)R << logn;
  act_encrypt_gather_kernel<<<act_grid(total), kActThreads, 0, (cudaStream_t)stream>>>(
      mq.m[0], mp.m[0], delta, h_powmod(2, (uint64_t)f, p), square, logn, zero, m, gidx, out, total);
  FHE_CHECK_LAUNCH("act_encrypt_gather_kernel");
  return FHE_OK;
}

int fhe_ct_pmult_add(uint64_t q, int R, int n, const uint64_t* ct, const uint64_t* pt, const uint64_t* add,
                     uint64_t* out, void* stream) {
  ModSet mq;
  if (int rc = make_modset(&q, 1, &mq)) return rc;
  const int logn = act_logn(n);
  if (logn < 0 || R < 0) return fail(FHE_ERR_VALUE, "bad row geometry (R=%d n=%d)", R, n);
  if (!R) return FHE_OK;
  if (!ct || !pt || !out) return fail(FHE_ERR_VALUE, "null pmult pointer");
  const int64_t total = (int64_t)R << logn;
  ct_pmult_add_kernel<<<act_grid(total), kActThreads, 0, (cudaStream_t)stream>>>(mq.m[0], logn, ct, pt, add, out,
                                                                                   total);
  FHE_CHECK_LAUNCH("ct_pmult_add_kernel");
  return FHE_OK;
}

int fhe_act_finalize(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const uint64_t* a, const uint64_t* b,
                     const uint64_t* c, uint64_t* out, void* stream) {
  ModSet mq, mp;
  if (int rc = act_moduli(q, p, delta, &mq, &mp)) return rc;
  const int logn = act_logn(n);
  if (logn < 0 || R < 0) return fail(FHE_ERR_VALUE, "bad row geometry (R=%d n=%d)", R, n);
  if (!R) return FHE_OK;
  if (!a || !b || !c || !out) return fail(FHE_ERR_VALUE, "null finalize pointer");
  const int64_t total = (int64_t)R << logn;
  act_finalize_kernel<<<act_grid(total), kActThreads, 0, (cudaStream_t)stream>>>(mq.m[0], mp.m[0], delta, logn, a,
                                                                                   b, c, out, total);
  FHE_CHECK_LAUNCH("act_finalize_kernel");
  return FHE_OK;
}

}  // extern "C"
