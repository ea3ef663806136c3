/*
 * flashhe.h — C ABI of libflashhe.so, the B200 (sm_100a) hot path of the
 * Flash HE-convolution protocol (arxiv 2401.16732).
 *
 * The reference (`/root/reference/pkg/src/privinfer`, pure Python + numpy) has
 * no FFI layer: its boundary is the Python module API. Each entry point below
 * replaces one numpy hot loop of that API and is what a maintainer would bind
 * from `privinfer` (ctypes / cffi) — see INTEGRATION.md. The Python package
 * `paper_2401_16732_b200` is exactly such a binding.
 *
 * Conventions
 *   - All data pointers are DEVICE pointers (cudaMalloc / torch CUDA memory)
 *     unless a parameter says "host". Coefficients are uint64 holding the
 *     reference's int64 values in [0, modulus) bit-for-bit.
 *   - A "row" is one polynomial of n coefficients, contiguous. Batched calls
 *     take rows laid out [B][L][P][n]: B ciphertexts, L RNS limbs (independent
 *     moduli — the reference is single-modulus), P polys per
 *     ciphertext (2: c0, c1). Row r uses limb (r / P) % L.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream). Every call is
 *     asynchronous on that stream; errors of the launch itself are reported.
 *   - Return value: FHE_OK or an FHE_ERR_* code; fhe_last_error() gives the
 *     message (thread-local). The codes map 1:1 onto the exception types the
 *     reference raises (errors.py:1-25).
 *   - No entry point falls back to the CPU.
 */
#ifndef FLASHHE_H
#define FLASHHE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library builds with -fvisibility=hidden */
#endif

#define FHE_OK 0
#define FHE_ERR_PARAMETER 1 /* privinfer.errors.ParameterError          (errors.py:4)  */
#define FHE_ERR_ENCODING 2  /* privinfer.errors.EncodingError           (errors.py:8)  */
#define FHE_ERR_BUDGET 3    /* privinfer.errors.AccumulatorBudgetError  (errors.py:12) */
#define FHE_ERR_PROTOCOL 4  /* privinfer.errors.ProtocolError           (errors.py:16) */
#define FHE_ERR_VALUE 5     /* ValueError: malformed sizes / pointers               */
#define FHE_ERR_CUDA 6      /* RuntimeError: CUDA launch / runtime failure          */

#define FHE_MAX_LIMBS 8
#define FHE_MAX_LOGN 17

typedef struct fhe_plan fhe_plan; /* opaque: negacyclic NTT tables of one (n, q) */

/* ---------------------------------------------------------------- misc */
const char* fhe_last_error(void);
int fhe_abi_version(void);
/* number of kernel launches issued by this library since load (instrumentation) */
uint64_t fhe_launch_count(void);
/* cudaEventRecord that stays timeable inside a CUDA-graph capture
 * (external event node); used by the benchmark's kernel-level timing. */
int fhe_record_event(void* event, void* stream);
/* Timeline instrumentation of the K1-TC pipeline: CTA 0 records clock64() at
 * its pipeline events into dev_buf, which must hold 25 x 4096 uint64 (kinds 0-7:
 * pipeline events, 7 also the tile sequence; 8: per-CTA start/end and relayout
 * completion times; 9-24: per-epilogue-warp events); NULL disables. The default build
 * records only the per-CTA start/end stamps (kind 8: globaltimer at [2b], [2b+1],
 * clock64 at [512+2b], [512+2b+1] for CTA b); the per-event points inside the role
 * loops need a -DFHE_TC_TRACE=1 build (tools/build_probe.py trace -DFHE_TC_TRACE=1,
 * loaded with FLASHHE_LIB): they cost instruction-cache space in the hot loops. */
int fhe_debug_trace(void* dev_buf);

/* Roofline micro-benchmarks (register-resident, no memory traffic):
 * blocks*threads*iters*16 IMAD.WIDE (mad.wide.s32), and
 * blocks*threads*iters*8 Harvey/Shoup forward butterflies mod q. */
int fhe_peak_imad_wide(int blocks, int threads, int iters, int64_t* sink, void* stream);
int fhe_peak_butterfly(int blocks, int threads, int iters, uint64_t q, uint64_t* sink,
                       void* stream);
/* blocks*iters*8 dense tcgen05.mma.kind::i8 (M=128, N=n_tile, K=32; n_tile
 * 64, 128 or 256) on resident shared-memory operands: 2*128*n_tile*32 int8
 * ops each. sink: DEVICE >= 6 uint32; words [2,4) / [4,6) receive CTA 0's
 * SM cycles / nanoseconds of the MMA loop (its clock = cycles / ns). */
int fhe_peak_tc_i8(int blocks, int n_tile, int iters, uint32_t* sink, void* stream);

/* ------------------------------------------------- plans (ring.NttPlan) */
/* Host-only (no GPU needed). ring.NttPlan._find_root (ring.py:121-127):
 * first g in [2, 10000) with psi = g^((q-1)/2n), psi^n == q-1. */
int fhe_find_root(int n, uint64_t q, uint64_t* psi_out);
/* Host-only: psi_brv / ipsi_brv / n_inv exactly as ring.NttPlan.__init__
 * (ring.py:96-113). Outputs are host arrays of n entries (n_inv: 1 entry). */
int fhe_plan_tables_host(int n, uint64_t q, uint64_t* psi_brv, uint64_t* ipsi_brv,
                         uint64_t* n_inv);
/* Device plan: tables (value + Shoup companion) uploaded to HBM.
 * Replaces ring.get_plan / NttPlan.__init__ (ring.py:96-119, 205-212).
 * Requires q ≡ 1 mod 2n (else FHE_ERR_PARAMETER, ring.py:97-98), q < 2^62. */
int fhe_plan_create(int n, uint64_t q, fhe_plan** out);
int fhe_plan_destroy(fhe_plan* plan);
int fhe_plan_query(const fhe_plan* plan, int* n, uint64_t* q, uint64_t* psi);

/* --------------------------------------------- K2: batched NTT / iNTT */
/* ring.NttPlan.fwd (ring.py:129-144): natural order in, bit-reversed order
 * out (out[i] = f(psi^(2*bitrev(i)+1))), canonical [0,q). src may equal dst.
 * plans: host array of L plan pointers (same n). Rows [B][L][P][n]. */
int fhe_ntt_forward(const fhe_plan* const* plans, int L, int B, int P,
                    const uint64_t* src, uint64_t* dst, void* stream);
/* ring.NttPlan.inv (ring.py:146-162), n^-1 folded into the last stage. */
int fhe_ntt_inverse(const fhe_plan* const* plans, int L, int B, int P,
                    const uint64_t* src, uint64_t* dst, void* stream);
/* Key-switch digit planes, hoisted (bfv.hrot, bfv.py:485-491):
 * src rows [B][L][n] canonical coefficients; dst rows [B][L][ndig][n] with
 * dst[b][l][i] = NTT((src[b][l] >> (T*i)) & (2^T - 1)). */
int fhe_ntt_forward_digits(const fhe_plan* const* plans, int L, int B,
                           const uint64_t* src, uint64_t* dst, int T, int ndig,
                           void* stream);

/* -------------------------------------------- K3: elementwise ring ops */
/* moduli: host array of L moduli (q_l < 2^62). Operand b is broadcast when
 * Bb == 1 (over ciphertexts) or Pb == 1 (over polys); else Bb == B, Pb == P. */
#define FHE_OP_ADD 0 /* ring.poly_add    (ring.py:219-223) */
#define FHE_OP_SUB 1 /* ring.poly_sub    (ring.py:226-230) */
#define FHE_OP_MUL 2 /* NttPlan.pointwise (ring.py:193-197) */
int fhe_poly_binary(int op, const uint64_t* moduli, int L, int B, int P, int n,
                    const uint64_t* a, const uint64_t* b, int Bb, int Pb,
                    uint64_t* out, void* stream);
/* bfv.pmult with a prepared plaintext (bfv.py:359-372): out = a ⊙ w mod q_l by
 * Shoup multiplication, w_shoup = fhe_shoup_companions(w) (floor(w 2^64 / q_l),
 * once per prepared plaintext). Same broadcast rules as fhe_poly_binary; the
 * result equals FHE_OP_MUL bit for bit. q_l < 2^63. */
int fhe_poly_mul_shoup(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* a,
                       const uint64_t* w, const uint64_t* w_shoup, int Bb, int Pb, uint64_t* out,
                       void* stream);
int fhe_shoup_companions(const uint64_t* moduli, int L, int B, int P, int n, const uint64_t* w,
                         uint64_t* w_shoup, void* stream);
/* ring.poly_neg (ring.py:233-235) */
int fhe_poly_neg(const uint64_t* moduli, int L, int B, int P, int n,
                 const uint64_t* a, uint64_t* out, void* stream);
/* ring.scalar_mul (ring.py:238-243): k_per_limb host array, k < q_l */
int fhe_poly_scalar_mul(const uint64_t* moduli, int L, int B, int P, int n,
                        const uint64_t* a, const uint64_t* k_per_limb, uint64_t* out,
                        void* stream);
/* ring.monomial_mul (ring.py:279-299): out = a * x^(-shift) (any shift) */
int fhe_poly_monomial(const uint64_t* moduli, int L, int B, int P, int n,
                      const uint64_t* a, int64_t shift, uint64_t* out, void* stream);
/* ResNet shortcut add in the conv output layout (inference chain; the DRot of
 * ring.monomial_mul, ring.py:279-299, then bfv.hadd, bfv.py:316-320):
 * out[j] = y[j] + a[j / c_n] * x^(-tile*(j mod c_n)) for j < count, both
 * polynomials; y, out: [count][2][n], a: [ceil(count/c_n)][2][n] (the packed
 * block input, c_n channel tiles of `tile` slots per ciphertext). out may be y. */
int fhe_residual_add(uint64_t q, int count, int c_n, int tile, int n, const uint64_t* y,
                     const uint64_t* a, uint64_t* out, void* stream);
/* ring.apply_galois (ring.py:316-334): out = a(x^gpow), gpow odd */
int fhe_poly_automorphism(const uint64_t* moduli, int L, int B, int P, int n,
                          const uint64_t* a, uint64_t gpow, uint64_t* out, void* stream);
/* bfv._delta_times (bfv.py:166-168) then + base:
 * out = (base + delta * (m mod p)) mod q ; base may be NULL (treated as 0).
 * m rows are int64 values (any sign). Used by plain_add / encrypt_online. */
int fhe_poly_add_delta(uint64_t q, uint64_t p, uint64_t delta, int R, int n,
                       const uint64_t* base, const int64_t* m, uint64_t* out,
                       void* stream);
/* bfv.encrypt_private combine step (bfv.py:181):
 * out = (delta * (m mod p) - as - e) mod q, m and e int64 (e small, signed;
 * m NULL: encryptions of zero),
 * as canonical [0,q) (= iNTT(NTT(a) * s_eval)). */
int fhe_encrypt_combine(uint64_t q, uint64_t p, uint64_t delta, int R, int n,
                        const int64_t* m, const uint64_t* as, const int64_t* e,
                        uint64_t* out, void* stream);
/* mod-switch a row set into another modulus: out = centered(v mod p) mod q
 * (bfv.prepare_plaintext lift, bfv.py:351-356) */
int fhe_poly_lift_centered(uint64_t p, uint64_t q, int R, int n, const int64_t* v,
                           uint64_t* out, void* stream);

/* ---------------------- ring.WidePoly lazy accumulator (ring.py:347-406) */
/* lo/hi: int64 [n] limb accumulators (30-bit limbs, reference layout).
 * accumulate:        lo += (f & (2^30-1)) * scalar ; hi += (f >> 30) * scalar
 * accumulate_split:  lo += flo * scalar ; hi += fhi * scalar
 * add_rotated:       (lo,hi) += (olo,ohi) * x^(-shift) (signed, lazy)
 * finalize:          out = ((hi << 30) + lo) mod q, canonical            */
int fhe_wide_accumulate(int n, const uint64_t* f, int64_t scalar, int64_t* lo, int64_t* hi,
                        void* stream);
int fhe_wide_accumulate_split(int n, const int64_t* flo, const int64_t* fhi, int64_t scalar,
                              int64_t* lo, int64_t* hi, void* stream);
int fhe_wide_add_rotated(int n, const int64_t* olo, const int64_t* ohi, int64_t shift,
                         int64_t* lo, int64_t* hi, void* stream);
int fhe_wide_finalize(int n, uint64_t q, const int64_t* lo, const int64_t* hi, uint64_t* out,
                      void* stream);

/* ------------------------------------ K6: decryption rounding + budget */
/* bfv.decrypt_with_budget (bfv.py:278-293) given the raw phase
 * u = [c1 s + c0]_q (canonical): m = ((u + delta/2) // delta) mod p and
 * maxw[r] = max |u - delta * round(u/delta)| over row r (host reads it). */
int fhe_decrypt_round(uint64_t q, uint64_t p, uint64_t delta, int R, int n,
                      const uint64_t* u, uint64_t* m_out, uint64_t* maxw_out,
                      void* stream);
/* fhe_decrypt_round with the per-row residual maxima folded into ONE device
 * word: *max_all = max(*max_all, max |residual| of every row) (atomicMax; the
 * caller zeroes it, fhe_zero, before the first round it covers). A layer's
 * whole share exchange then needs one 8-byte read for its noise-budget check
 * (the reference checks each decryption, bfv.py:278-293). */
int fhe_decrypt_round_max(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const uint64_t* u,
                          uint64_t* m_out, uint64_t* max_all, void* stream);
/* bfv.decrypt over a batch in one launch (bfv.py:278-293, K6 fused): cts = DEVICE
 * [k][2][n] ciphertexts mod q (eval = 0: COEFF domain, 1: EVAL domain), s_eval =
 * DEVICE [n] secret key in EVAL order; writes m_out [k][n] = round(Δ^-1 [c1 s + c0]_q)
 * mod p and folds every row's largest |residual| into *max_all (atomic max). The
 * same values as fhe_ntt_forward + fhe_binary(mul, add) + fhe_ntt_inverse +
 * fhe_decrypt_round_max, in one kernel (one CTA per ciphertext); n = 1024, 2048, 4096. */
int fhe_decrypt_fused(const fhe_plan* plan, int k, int eval, const uint64_t* cts, const uint64_t* s_eval,
                      uint64_t p, uint64_t delta, uint64_t* m_out, uint64_t* max_all, void* stream);
/* bfv.to_eval + pmult + plain_add of a ciphertext batch in one launch (the layer
 * exchange's server round 2): ct = DEVICE [k][2][n] in COEFF form, pt / add = DEVICE
 * [k][n] in EVAL order; out [k][2][n] = NTT(ct) ⊙ pt (+ add on c0). Identical to
 * fhe_ntt_forward + fhe_ct_pmult_add; n = 1024, 2048, 4096; add may be NULL. */
int fhe_ntt_pmult_add(const fhe_plan* plan, int k, const uint64_t* ct, const uint64_t* pt, const uint64_t* add,
                      uint64_t* out, void* stream);

/* ------------------------------------------ K1: Flash convolution core */
/* Lazy DRot x CMult accumulation with one reduction per coefficient
 * (conv._proposed_channel conv.py:326-352, _CtAccum conv.py:269-291,
 * WidePoly ring.py:347-406). For output o in [0,c_o), fragment f in [0,frags),
 * poly p in {0,1}, coefficient s in [0,n):
 *   out[o*frags+f][p][s] = ( Σ_k w[o][k] * (in[src_k + f*frag_stride][p] * x^(-step_k))[s]
 *                           + (p == 0 && bias ? bias_delta[o] * mask[f][s] : 0) ) mod q
 * step_k in (-n, n). weights int16 [c_o][K] (|w| < 2^15; the reference bounds |w| < 2^8); term_src/term_step int32 [K];
 * bias_delta [c_o] (Δ·(b mod p) mod q) and bias_mask uint8 [frags][n] may be
 * NULL. Caller enforces the lazy budget (fhe_conv_check_budget). */
int fhe_conv_flash(uint64_t q, int n, const uint64_t* in, int n_in,
                   const int16_t* weights, int c_o, int K, const int32_t* term_src,
                   const int32_t* term_step, int frags, int frag_stride,
                   const uint64_t* bias_delta, const uint8_t* bias_mask, uint64_t* out,
                   void* stream);
/* K1-TC: the same contraction on tcgen05.mma.kind::i8 (u8 digit planes x s8
 * weights -> s32, 8 planes recombined exactly mod q), canonical mod q, bias
 * fused, for a STACK of independent layers in one cooperative persistent
 * launch (one CTA per SM). Per layer: (1) relayout of the input into the
 * digit-plane operand X, uint8 [2][frags][ceil(c_i/32)][n + 2h][256 B] (UMMA
 * core-matrix order), by dedicated relayout warps of all CTAs from a shared
 * work counter, up to three layers ahead of the GEMM; (2) warp-specialised tcgen05 GEMM,
 * tile = 128 output channels x pos_tile (16 or 32) positions, 32 input
 * channels per pipeline stage, starting once its layer's X is complete.
 * One layer = conv.conv_proposed; several = conv.issue_k1 / the serving path. */
typedef struct fhe_conv_tc_layer {
  const uint64_t* in;     /* DEVICE [n_in][2][n] input ciphertexts */
  int n_in, c_i, frags, fstride;
  const int32_t* chan;    /* DEVICE int32 pairs [c_i][2] = (source ct, slot shift) of
                             channel j (the packing of conv.py:113-130); fragment f
                             reads source + f*fstride */
  int h;                  /* halo = max |tap step| */
  const int8_t* w;        /* DEVICE int8 [ceil(c_o/128)][ceil(c_i/32)][taps][16][256 B]
                             (8 output x 16 input channels per 128 B), |w| <= 127,
                             127*255*ceil32(c_i)*taps < 2^31 */
  int c_o, taps, pos_tile;
  const int32_t* tap_steps; /* HOST int32 [taps] DRot steps, each in [-h, h] */
  const uint64_t* bias_delta; /* DEVICE [c_o] or NULL (conv._bias_plaintext) */
  const uint8_t* bias_mask;   /* DEVICE [frags][n] slots that receive the bias */
  uint64_t* out;          /* DEVICE [c_o*frags][2][n] */
  int rep;                /* 1 (or 0), 2 or 4: position groups stacked in the 128 accumulator
                             rows for c_o <= 128/rep (pos_tile 32): a tile covers 32 rep
                             positions; w then holds taps*rep tap blocks, block r*taps + t
                             carrying tap t's weights in rows [r*128/rep, r*128/rep + c_o)
                             (zero elsewhere) — group r reads the window 32 r positions on */
  int tsplit;             /* 0 or 1: nothing. 2 (with rep == 2, c_o <= 64): the two position
                             groups INTERLEAVE — accumulator row 2 o + r computes channel o at
                             positions s0 + 2 u + r. taps / tap_steps are then the MERGED taps:
                             the distinct values of step_t + r (each in [-h, h + 1]), and w holds
                             one tap block per merged tap with W[o][j][t] in row 2 o + r of the
                             block of step_t + r (zero elsewhere): taps of the two groups that
                             read the same window offset share one full-height MMA. X is stored
                             de-interleaved per plane (even positions, then odd) by the relayout */
} fhe_conv_tc_layer;
/* layers: HOST array of nl (<= 24) layers sharing (q, n), 2^56 <= q < 2^62.
 * X: DEVICE scratch. x_stride > 0: 3 operand buffers x_stride bytes apart
 *   (x_stride >= the largest layer's X; one buffer when nl == 1), layer l uses
 *   buffer l % 3 (relayout runs up to three layers ahead of the GEMM).
 *   x_stride == 0: every layer owns a region, consecutive and 256-byte
 *   aligned (sum of ceil256(2*frags*ceil(c_i/32)*(n+2h)*256) bytes), and the
 *   relayout of later layers never waits for earlier GEMMs.
 * sync: DEVICE uint64[3 + 4*24], zeroed once before first use: the launch
 *   counter and, per layer, work / relayout-done / GEMM-done / tile counters
 *   (CTAs grab tiles dynamically, the last grab of a launch resets the
 *   layer's tile counter; FHE_TC_DYNAMIC=0 deals them statically). The other
 *   counters only grow (graph-replay safe; the GEMM-done counters advance only
 *   with x_stride > 0 and nl > 3, the one mode that waits on them); reuse one
 *   sync buffer only for stacks with the same number of layers and the same
 *   x_stride mode, and never for launches that may run concurrently. */
int fhe_conv_tc_stack(uint64_t q, int n, const fhe_conv_tc_layer* layers, int nl,
                      uint8_t* X, size_t x_stride, uint64_t* sync, void* stream);
/* conv.avg_pool (conv.py:604-623): every row (polynomial) of in [rows][n]
 * replaced by the sum of its k x k DRot taps (steps dy*w_p + dx, weight 1),
 * computed separably (k row taps, then k column taps of the row sums; exact
 * mod q, so identical to the k^2-tap contraction). (k-1)(w_p+1) < n, n <= 8192. */
int fhe_avg_pool(uint64_t q, int n, int rows, int k, int w_p, const uint64_t* in, uint64_t* out,
                 void* stream);
/* The serving path's per-job step in one call (conv.conv_proposed_stream):
 * host_in (PINNED, in_bytes) -> layer->in on stream `up`, event ev_up; `comp`
 * waits for it and runs the layer (fhe_conv_tc_stack, nl = 1), event ev_comp;
 * `down` waits for that and copies layer->out to host_out (PINNED, out_bytes).
 * Streams and events are cudaStream_t / cudaEvent_t; the two events may be
 * reused for every job (waits bind to the latest record). */
int fhe_conv_stream_job(uint64_t q, int n, const fhe_conv_tc_layer* layer, const void* host_in,
                        size_t in_bytes, void* host_out, size_t out_bytes, uint8_t* X, size_t x_stride,
                        uint64_t* sync, void* up, void* comp, void* down, void* ev_up, void* ev_comp);
/* Host-only budget guard (conv._check_budget conv.py:314-319, ring.py:366-372):
 * FHE_ERR_BUDGET if max_o Σ_k |w[o][k]| >= 2^32. weights: HOST int64 [c_o][K]. */
int fhe_conv_check_budget(const int64_t* weights_host, int c_o, int K);

/* -------------------------------------------- K4: hoisted key switching */
/* Keys to Montgomery form (one-time, at switching-key upload):
 * rows [B][L][P][n] -> x * 2^64 mod q_l. */
int fhe_to_montgomery(const uint64_t* moduli, int L, int B, int P, int n,
                      const uint64_t* a, uint64_t* out, void* stream);
/* bfv.hrot (bfv.py:467-500) after hoisting: ct rows [B][L][2][n] (EVAL),
 * digits rows [B][L][ndig][n] (fhe_ntt_forward_digits of iNTT(c1)),
 * keys_mont rows [L][ndig][2][n] (swk0_i, swk1_i in Montgomery form).
 * perm(x) = index_of_exp[(exp_at_index[x] * gpow) mod 2n] (ring.py:199-202):
 *   out[b][l][0][x] = ct[b][l][0][perm x] + Σ_i D_i[perm x] * swk0_i[x]   mod q_l
 *   out[b][l][1][x] =                       Σ_i D_i[perm x] * swk1_i[x]   mod q_l */
int fhe_keyswitch_apply(const uint64_t* moduli, int L, int B, int n, const uint64_t* ct,
                        const uint64_t* digits, const uint64_t* keys_mont, int ndig,
                        uint64_t gpow, uint64_t* out, void* stream);

/* A whole rotation sweep in one launch (bfv.hrot for S steps of the same
 * ciphertexts, bfv.py:467-500; the digit NTTs of bfv.py:485-497 do not depend
 * on the step and are computed once): for every step s, exactly
 * fhe_keyswitch_apply(..., keys_mont[s], gpows[s], outs[s]). keys_mont / outs:
 * HOST arrays of S DEVICE pointers ([L][ndig][2][n] keys, [B][L][2][n]
 * outputs); gpows: HOST [S] Galois elements. ndig <= 8. */
int fhe_keyswitch_multi(const uint64_t* moduli, int L, int B, int n, const uint64_t* ct, const uint64_t* digits,
                        int ndig, int S, const uint64_t* const* keys_mont, const uint64_t* gpows,
                        uint64_t* const* outs, void* stream);

/* Row plumbing (no arithmetic). fhe_gather_rows: srcs is a HOST array of k
 * DEVICE row pointers (n words each) -> dst DEVICE [k][n] (the stack form of a
 * list of polynomials). fhe_copy_2d: cudaMemcpy2DAsync device to device (e.g.
 * interleaving c0 / c1 row stacks into [k][2][n]). fhe_zero: cudaMemsetAsync. */
int fhe_gather_rows(const uint64_t* const* srcs, int k, int n, uint64_t* dst, void* stream);
int fhe_copy_2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
                void* stream);
/* count (<= 8) DEVICE-to-DEVICE copies of bytes[i] (multiples of 8, 8-byte aligned) in
 * one kernel launch (srcs / dsts / bytes: HOST arrays). */
int fhe_copy_many(int count, const void* const* srcs, void* const* dsts, const size_t* bytes, void* stream);
int fhe_zero(void* dst, size_t bytes, void* stream);

/* Fused PMult-accumulate of the conventional convolution (conv.py:457-564:
 * the pmult + hadd chain per output ciphertext), EVAL domain, one launch:
 *   out[o][p] = Σ_{k in [term_off[o], term_off[o+1])} R[terms[2k]][p] ⊙ PT[terms[2k+1]]  mod q
 * R: DEVICE [nR][2][n] rotated ciphertexts; pt_mont: DEVICE [nPT][n] prepared
 * plaintexts in Montgomery form (fhe_to_montgomery); term_off: DEVICE int32
 * [n_out+1]; terms: DEVICE int32 pairs (rotation row, plaintext row), indices
 * validated by the caller. out: DEVICE [n_out][2][n], canonical. */
int fhe_pmac(uint64_t q, int n, const uint64_t* R, const uint64_t* pt_mont, const int32_t* term_off,
             const int32_t* terms, int n_out, uint64_t* out, void* stream);

/* Fused conventional convolution (conv.py:457-564, north_star (b)): rotation,
 * encoded-weight multiply and accumulation in one pass, EVAL domain, modulus q.
 * For output o and slot x:
 *   out[o][p][x] = Σ_g Σ_{(o, pt) in terms(g)} PT[pt][x] · R_g[p][x]   mod q
 * with R_g = HRot(C[src_g], step_g) formed in registers from the hoisted digits
 * (bfv.hrot, bfv.py:467-500) — rotated ciphertexts are never written:
 *   R_g[0][x] = C[src][0][π(x)] + Σ_i D[src][i][π(x)] K[key_g][i][0][x]
 *   R_g[1][x] =                   Σ_i D[src][i][π(x)] K[key_g][i][1][x]
 * π(x) = index_of_exp[(exp_at_index[x] · gpow_g) mod 2n] (ring.py:199-202);
 * key_g = -1 means step 0 (R_g = C[src]).
 * C: DEVICE [nsrc][2][n]; D: DEVICE [nsrc][ndig][n] (fhe_ntt_forward_digits);
 * K_mont: DEVICE [nkeys][ndig][2][n] Montgomery keys; groups: DEVICE int32
 * [G][2] = (src, key); gpow: DEVICE uint64 [G]; outputs in tiles of 16:
 * tile_off: DEVICE int32 [ceil(n_out/16)][G+1] CSR offsets into terms, terms:
 * DEVICE int32 pairs (o mod 16, plaintext row); pt_mont: DEVICE [nPT][n]
 * Montgomery plaintexts. gchunks > 1 splits the groups over that many CTAs
 * per slot block (partial: DEVICE [gchunks][n_out][2][n] scratch). ndig <= 16,
 * ndig · q < 2^64. out: DEVICE [n_out][2][n], canonical. */
int fhe_rot_pmac(uint64_t q, int n, int ndig, const uint64_t* C, const uint64_t* D, const uint64_t* K_mont,
                 int G, const int32_t* groups, const uint64_t* gpow, int n_out, const int32_t* tile_off,
                 const int32_t* terms, const uint64_t* pt_mont, int gchunks, uint64_t* partial, uint64_t* out,
                 void* stream);

/* ------------------------------------ K5: x^2+x share arithmetic (act2pc) */
/* Client share pass, one vectorised pass
 * over decrypted slots w in [0,p): y = (w^2 + w * 2^f) mod p. */
int fhe_act_client_square(uint64_t p, int f, int64_t count, const uint64_t* w,
                          uint64_t* y, void* stream);
/* Server finalize constant: c = (r^2 - r*2^f + v) mod p,
 * from r, r_sq, v in [0,p). */
int fhe_act_server_const(uint64_t p, int f, int64_t count, const uint64_t* r,
                         const uint64_t* r_sq, const uint64_t* v, uint64_t* c,
                         void* stream);

/* ---- K5 over a whole layer (row stacks [R][2][n], all pointers DEVICE) ---- */
/* Client repack (conv.py:148-197: channel_positions of the conv output, stride
 * applied, composed with pack_vectors of the next layer's layout) and the
 * batch-slot placement of bfv.encode_batch (bfv.py:124-133) as one gather:
 *   out[i] = idx[i] >= 0 ? src[idx[i]] : 0,   i < count. */
int fhe_act_gather(int64_t count, const int32_t* idx, const uint64_t* src, uint64_t* out,
                   void* stream);
/* bfv.encrypt_online (bfv.py:248-263) over rows, optionally fused with the
 * client square:
 *   v = m[r][perm ? perm[s] : s] mod p;  if (square) v = v^2 + v*2^f mod p
 *   out[r][0][s] = zero[r][0][s] + Δ v mod q;   out[r][1][s] = zero[r][1][s]
 * zero: precomputed encryptions of 0 (single use); perm: int32 [n] or NULL
 * (bfv.decode_batch's slot gather, bfv.py:135-139). Also serves server_round1
 * (plain_add of the masks, zero = the conv output). out must not alias zero. */
int fhe_act_encrypt_rows(uint64_t q, uint64_t p, uint64_t delta, int f, int square, int R, int n,
                         const uint64_t* zero, const uint64_t* m, const int32_t* perm,
                         uint64_t* out, void* stream);
/* bfv.pmult then bfv.plain_add in the EVAL domain (bfv.py:330-372), one pass:
 *   out[r][0] = ct[r][0] ⊙ pt[r] + add[r],  out[r][1] = ct[r][1] ⊙ pt[r]   mod q
 * pt, add: [R][n] EVAL (prepared plaintext / NTT'd Δ·v); add may be NULL. */
int fhe_ct_pmult_add(uint64_t q, int R, int n, const uint64_t* ct, const uint64_t* pt,
                     const uint64_t* add, uint64_t* out, void* stream);
/* act2pc server_finalize: psub(a, b) then plain_add of the
 * constant c = r^2 - r*2^f + v (fhe_act_server_const), [R][n] mod p. */
int fhe_act_finalize(uint64_t q, uint64_t p, uint64_t delta, int R, int n, const uint64_t* a,
                     const uint64_t* b, const uint64_t* c, uint64_t* out, void* stream);
/* Fused form of the client's repack + encryption (same values, one launch):
 * fhe_act_encrypt_gather = fhe_act_gather(gidx) + fhe_act_encrypt_rows (the message of
 *   element i is m[gidx[i]], gidx DEVICE int32 [R][n]). */
int fhe_act_encrypt_gather(uint64_t q, uint64_t p, uint64_t delta, int f, int square, int R, int n,
                           const uint64_t* zero, const uint64_t* m, const int32_t* gidx, uint64_t* out,
                           void* stream);
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* FLASHHE_H */
