/*
 * conv_oracle.c — CPU oracle / CPU baseline of the Flash convolution core.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/ and bench.py (cpu_baseline and
 * `--impl reference` legs), never by the product package.
 *
 * A C restatement of privinfer's lazy-reduction convolution
 * (conv._proposed_channel conv.py:326-352, _ExtPoly conv.py:251-266,
 * WidePoly.accumulate_split / finalize ring.py:379-406): per output unit,
 * every (input row, DRot step) term is accumulated as two 30-bit limbs in
 * int64 over the [-a | a | -a] extension, then reduced once mod q.
 * Output units are spread over `threads` POSIX threads (the reference's
 * fork-pool over output channels, conv.py:389-395).
 *
 * out[(o*frags+f)][p][s] = ( Σ_k w[o][k] · ext(in[src_k + f*fstride][p])[n + step_k + s] ) mod q
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LIMB 30
#define LMASK ((1ull << LIMB) - 1)

typedef struct {
  uint64_t q;
  int n, n_in, c_o, K, frags, fstride;
  const uint64_t* in;
  const int16_t* w;
  const int32_t* src;
  const int32_t* step;
  uint64_t* out;
  int64_t* ext_lo; /* [n_in][2][3n] */
  int64_t* ext_hi;
  const int32_t* sel; /* optional list of output units to compute (NULL: 0..total-1) */
  int next, total;
  pthread_mutex_t mu;
} job_t;

static void build_ext(job_t* J, int r) {
  const int n = J->n;
  for (int p = 0; p < 2; ++p) {
    const uint64_t* a = J->in + ((size_t)r * 2 + p) * n;
    int64_t* lo = J->ext_lo + ((size_t)r * 2 + p) * 3 * n;
    int64_t* hi = J->ext_hi + ((size_t)r * 2 + p) * 3 * n;
    for (int i = 0; i < n; ++i) {
      uint64_t v = a[i], neg = v ? J->q - v : 0;
      lo[i] = lo[2 * n + i] = (int64_t)(neg & LMASK);
      hi[i] = hi[2 * n + i] = (int64_t)(neg >> LIMB);
      lo[n + i] = (int64_t)(v & LMASK);
      hi[n + i] = (int64_t)(v >> LIMB);
    }
  }
}

static void do_unit(job_t* J, int u, int row, int64_t* alo, int64_t* ahi) {
  const int n = J->n, o = u / J->frags, f = u % J->frags;
  for (int p = 0; p < 2; ++p) {
    memset(alo, 0, sizeof(int64_t) * n);
    memset(ahi, 0, sizeof(int64_t) * n);
    for (int k = 0; k < J->K; ++k) {
      const int64_t w = J->w[(size_t)o * J->K + k];
      if (!w) continue;
      const int r = J->src[k] + f * J->fstride;
      const int64_t* lo = J->ext_lo + ((size_t)r * 2 + p) * 3 * n + n + J->step[k];
      const int64_t* hi = J->ext_hi + ((size_t)r * 2 + p) * 3 * n + n + J->step[k];
      for (int s = 0; s < n; ++s) {
        alo[s] += lo[s] * w;
        ahi[s] += hi[s] * w;
      }
    }
    uint64_t* dst = J->out + ((size_t)row * 2 + p) * n;
    for (int s = 0; s < n; ++s) {
      __int128 t = ((__int128)ahi[s] << LIMB) + alo[s];
      __int128 r = t % (__int128)J->q;
      if (r < 0) r += J->q;
      dst[s] = (uint64_t)r;
    }
  }
}

static void* worker(void* arg) {
  job_t* J = (job_t*)arg;
  int64_t* alo = (int64_t*)malloc(sizeof(int64_t) * J->n);
  int64_t* ahi = (int64_t*)malloc(sizeof(int64_t) * J->n);
  for (;;) {
    pthread_mutex_lock(&J->mu);
    int u = J->next++;
    pthread_mutex_unlock(&J->mu);
    if (u >= J->total) break;
    do_unit(J, J->sel ? J->sel[u] : u, u, alo, ahi); /* row u of `out` */
  }
  free(alo);
  free(ahi);
  return NULL;
}

static int run(uint64_t q, int n, const uint64_t* in, int n_in, const int16_t* w, int c_o, int K,
               const int32_t* src, const int32_t* step, int frags, int fstride, uint64_t* out, int threads,
               int total, const int32_t* sel) {
  job_t J;
  J.q = q;
  J.n = n;
  J.n_in = n_in;
  J.c_o = c_o;
  J.K = K;
  J.frags = frags;
  J.fstride = fstride;
  J.in = in;
  J.w = w;
  J.src = src;
  J.step = step;
  J.out = out;
  J.sel = sel;
  J.next = 0;
  J.total = total;
  for (int k = 0; k < K; ++k)
    if (step[k] <= -n || step[k] >= n) return 1;
  for (int k = 0; k < K; ++k)
    if (src[k] < 0 || src[k] + (frags - 1) * fstride >= n_in) return 3;
  if (sel)
    for (int i = 0; i < total; ++i)
      if (sel[i] < 0 || sel[i] >= c_o * frags) return 4;
  J.ext_lo = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_in * 2 * 3 * n);
  J.ext_hi = (int64_t*)malloc(sizeof(int64_t) * (size_t)n_in * 2 * 3 * n);
  if (!J.ext_lo || !J.ext_hi) return 2;
  for (int r = 0; r < n_in; ++r) build_ext(&J, r);
  pthread_mutex_init(&J.mu, NULL);
  if (threads < 1) threads = 1;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, &J);
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&J.mu);
  free(J.ext_lo);
  free(J.ext_hi);
  return 0;
}

/* Returns 0 on success. `units` limits the computation to the first `units`
 * output units (a bounded sample); pass c_o*frags (or -1) for all. */
int oracle_conv(uint64_t q, int n, const uint64_t* in, int n_in, const int16_t* w, int c_o, int K,
                const int32_t* src, const int32_t* step, int frags, int fstride, uint64_t* out,
                int threads, int units) {
  int total = c_o * frags;
  if (units >= 0 && units < total) total = units;
  return run(q, n, in, n_in, w, c_o, K, src, step, frags, fstride, out, threads, total, NULL);
}

/* The output units listed in `sel` (n_sel of them, any order): unit sel[i]
 * is written to row i of `out` ([n_sel][2][n]). Used by the stacked-launch
 * parity tests and the strided CPU-baseline sample. */
int oracle_conv_units(uint64_t q, int n, const uint64_t* in, int n_in, const int16_t* w, int c_o, int K,
                      const int32_t* src, const int32_t* step, int frags, int fstride, uint64_t* out,
                      int threads, const int32_t* sel, int n_sel) {
  if (!sel || n_sel < 0) return 4;
  return run(q, n, in, n_in, w, c_o, K, src, step, frags, fstride, out, threads, n_sel, sel);
}
