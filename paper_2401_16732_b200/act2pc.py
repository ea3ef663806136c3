"""Two-round x²+x share protocol on the B200.

The reference package specifies but does not ship this module; names follow
SPEC.md:304-331. Server and client steps compose the bfv primitives (all GPU
kernels) and the K5 share pass (`fhe_act_client_square`,
`fhe_act_server_const`): one vectorised mod-p pass per step.

Algebra (frac bits f; the paper's protocol is f = 0):
  server r1:  ⟦a + r⟧                     = plain_add(⟦a⟧, r)               (direct)
  client r1:  w = a + r;  ⟦w² + w·2^f⟧ (direct), ⟦w⟧ (batch)       via encrypt_online
  server r2:  ⟦2rw + v⟧ = ⟦2ar + 2r² + v⟧ = pmult(⟦w⟧, 2r) + v               (batch)
  client r2:  ⟦2ar + 2r² + v⟧ re-encrypted direct
  finalize:   ⟦w² + w·2^f⟧ − ⟦2ar + 2r² + v⟧ + (r² − r·2^f + v) = ⟦a² + a·2^f⟧
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native, bfv, device, ring
from .bfv import Ciphertext, Encoding
from .ring import Domain
from .errors import EncodingError, ProtocolError
from .params import RingParams


class Round(Enum):
    INIT = 0
    MASKED = 1
    CROSS_SENT = 2
    DONE = 3


@dataclass
class FixedPointCodec:
    frac_bits: int
    p: int


@dataclass
class ActivationSession:
    """Server-private masks of one protocol run (single use)."""

    r: np.ndarray
    v: np.ndarray
    r_sq: np.ndarray
    layer_id: int = 0
    round: Round = Round.INIT
    codec: FixedPointCodec | None = None
    ct1: Ciphertext | None = field(default=None, repr=False)


def offline_prepare(count: int, params: RingParams, rng, frac_bits: int = 0, layer_id: int = 0) -> list[ActivationSession]:
    """Server masks r, v and r² for `count` runs; no bytes are exchanged."""
    codec = FixedPointCodec(frac_bits, params.p)
    sessions = []
    for _ in range(count):
        r = rng.integers(0, params.p, params.n, dtype=np.int64)
        v = rng.integers(0, params.p, params.n, dtype=np.int64)
        sessions.append(ActivationSession(r, v, r * r % params.p, layer_id, Round.INIT, codec))
    return sessions


def _expect(session: ActivationSession, rnd: Round):
    if session.round != rnd:
        raise ProtocolError(f"session is in round {session.round.name}, expected {rnd.name}")


def server_round1(conv_out: Ciphertext, session: ActivationSession, params: RingParams) -> Ciphertext:
    """⟦a + r⟧ = plain_add(⟦a⟧, encode_direct(r))."""
    _expect(session, Round.INIT)
    if conv_out.encoding != Encoding.DIRECT:
        raise EncodingError("activation input must be direct-encoded")
    msg = bfv.plain_add(conv_out, bfv.encode_direct(session.r, params), params)
    session.round = Round.MASKED
    return msg


def client_square(w: torch.Tensor, p: int, frac_bits: int = 0) -> torch.Tensor:
    """K5 client pass: (w² + w·2^f) mod p over a device tensor of slots."""
    w = w.contiguous()
    y = torch.empty_like(w)
    _native.call("fhe_act_client_square", p, frac_bits, w.numel(), w.data_ptr(), y.data_ptr(), device.stream())
    return y


def server_const(r, r_sq, v, p: int, frac_bits: int = 0) -> torch.Tensor:
    """K5 server pass: (r² − r·2^f + v) mod p."""
    tr, ts, tv = (device.to_device(np.asarray(a, dtype=np.int64)) for a in (r, r_sq, v))
    c = torch.empty_like(tr)
    _native.call("fhe_act_server_const", p, frac_bits, tr.numel(), tr.data_ptr(), ts.data_ptr(), tv.data_ptr(),
                 c.data_ptr(), device.stream())
    return c


def _decrypt_checked(ct: Ciphertext, sk: bfv.SecretKey) -> torch.Tensor:
    m, maxw = bfv.decrypt_rows([ct], sk)
    if bfv._budget(sk.params, maxw[0]) <= 0:
        raise ProtocolError("noise budget exhausted: ciphertext no longer decrypts reliably")
    return m.reshape(-1)


def client_round1(msg: Ciphertext, sk: bfv.SecretKey, zero_pool: bfv.ZeroPool,
                  codec: FixedPointCodec | None = None) -> tuple[Ciphertext, Ciphertext]:
    """Decrypt w = a + r, return (⟦w² + w·2^f⟧ direct, ⟦w⟧ batch)."""
    params = sk.params
    f = codec.frac_bits if codec else 0
    w = _decrypt_checked(msg, sk)
    y = client_square(w, params.p, f)
    ct_sq = bfv.encrypt_online(bfv.Plaintext(bfv.ModPoly(y, params.p), Encoding.DIRECT), zero_pool.take(), params)
    ct_w = bfv.encrypt_online(bfv.encode_batch(w.cpu().numpy(), params), zero_pool.take(), params)
    return ct_sq, ct_w


def server_round2(msgs: tuple[Ciphertext, Ciphertext], session: ActivationSession, params: RingParams) -> Ciphertext:
    """⟦2r·w + v⟧ = pmult(to_eval(⟦w⟧), encode_batch(2r)) + v (batch, EVAL)."""
    _expect(session, Round.MASKED)
    ct_sq, ct_w = msgs
    if ct_w.encoding != Encoding.BATCH or ct_sq.encoding != Encoding.DIRECT:
        raise EncodingError("round-1 messages must be (direct, batch)")
    two_r = bfv.encode_batch(2 * session.r % params.p, params)
    prod = bfv.pmult(bfv.to_eval(ct_w, params), two_r, params)
    out = bfv.plain_add(prod, bfv.encode_batch(session.v, params), params)
    session.ct1 = ct_sq
    session.round = Round.CROSS_SENT
    return out


def client_round2(msg: Ciphertext, sk: bfv.SecretKey, zero_pool: bfv.ZeroPool) -> Ciphertext:
    """Decrypt the batch message, re-encrypt its slots with direct encoding."""
    params = sk.params
    m = _decrypt_checked(msg, sk)
    z = bfv.decode_batch(bfv.Plaintext(bfv.ModPoly(m, params.p), Encoding.BATCH), params)
    return bfv.encrypt_online(bfv.encode_direct(z, params), zero_pool.take(), params)


def server_finalize(ct1: Ciphertext, ct2: Ciphertext, session: ActivationSession, params: RingParams) -> Ciphertext:
    """⟦a² + a·2^f⟧ = ct1 − ct2 + (r² − r·2^f + v)."""
    _expect(session, Round.CROSS_SENT)
    f = session.codec.frac_bits if session.codec else 0
    c = server_const(session.r, session.r_sq, session.v, params.p, f)
    diff = bfv.psub(ct1, ct2)
    out = bfv.plain_add(diff, bfv.Plaintext(bfv.ModPoly(c, params.p), Encoding.DIRECT), params)
    session.round = Round.DONE
    session.ct1 = None
    return out


def run_activation(conv_out: Ciphertext, session: ActivationSession, sk: bfv.SecretKey, zero_pool: bfv.ZeroPool,
                   params: RingParams) -> Ciphertext:
    """Both parties in-process (tests / benches): the full two-round exchange."""
    m1 = server_round1(conv_out, session, params)
    sq, w = client_round1(m1, sk, zero_pool, session.codec)
    m2 = server_round2((sq, w), session, params)
    back = client_round2(m2, sk, zero_pool)
    return server_finalize(sq, back, session, params)


# ---------------------------------------------------------------------------
# One layer of activations at once: the same protocol over row stacks
# [k, 2, n], with the client's repack into the next conv's tile layout
# (conv.py:148-197) folded into its decrypt -> square -> encrypt step.
#
# Both parties derive the public slot map of a RepackPlan from the model
# geometry. The server draws r over the conv output's slots and v over the
# next layout's slots; r' = r gathered through the map is what the client's
# repacked w' = a' + r' carries, so every later step works slot-for-slot in
# the next layout and the finalize yields ⟦a'² + a'·2^f⟧ already packed for
# the next convolution (zero borders / halos included: a' = r' = 0 there).


def repack_index(src, channels: int, dst, n: int) -> np.ndarray:
    """[k_dst, n] flat source slot (ct·n + slot) of every next-layout slot, −1
    where the next layout holds a zero: channel_positions of the conv output
    (stride applied, conv.py:162-177) composed with pack_vectors (conv.py:180-197)."""
    from . import conv

    h, w = src.out_dims()
    flat = np.empty((channels, h * w), dtype=np.int64)
    for j in range(channels):
        ci, si = conv.channel_positions(src, j)
        flat[j] = ci * n + si + 1
    return np.stack(conv.pack_vectors(flat.reshape(channels, h, w), dst, 1 << 62)) - 1


class RepackPlan:
    """Slot map conv output (stride pending) -> next conv input layout."""

    def __init__(self, src, channels: int, dst, params: RingParams):
        h, w = src.out_dims()
        if (dst.height, dst.width) != (h, w) or dst.stride != 1:
            raise EncodingError("next layout does not match the activation geometry")
        if dst.ring != params.n or src.ring != params.n:
            raise EncodingError("activations repack between direct layouts")
        n = params.n
        self.src, self.dst, self.channels, self.n = src, dst, channels, n
        self.k_src, self.k_dst = src.ct_count(channels), dst.ct_count(channels)
        if self.k_src * n >= 1 << 31:
            raise ValueError("layer too large for 32-bit slot indices")
        idx = repack_index(src, channels, dst, n)
        slot = bfv._slot_index(params)  # batch slot s -> evaluation position
        inv = np.empty(n, dtype=np.int64)
        inv[slot] = np.arange(n)
        self.idx_host = idx
        self.idx = device.to_device_i32(idx)
        self.idx_eval = device.to_device_i32(idx[:, inv])
        self.slot = device.to_device_i32(slot)

    def gather_host(self, values: np.ndarray) -> np.ndarray:
        """Host restatement of the map (offline mask preparation, tests)."""
        flat = np.asarray(values, dtype=np.int64).reshape(-1)
        return np.where(self.idx_host >= 0, flat[np.maximum(self.idx_host, 0)], 0)


_repack_plans: dict = {}


def repack_plan(src, channels: int, dst, params: RingParams) -> RepackPlan:
    """RepackPlan cached per geometry (its device maps and the layer graph that
    replays its exchange are reused by every inference through that layer)."""
    key = (src, channels, dst, params.fingerprint())
    plan = _repack_plans.get(key)
    if plan is None:
        plan = _repack_plans[key] = RepackPlan(src, channels, dst, params)
    return plan


def _gather(idx: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    src_c = src.contiguous()
    out = torch.empty(idx.shape, dtype=torch.int64, device=idx.device)
    _native.call("fhe_act_gather", idx.numel(), idx.data_ptr(), src_c.data_ptr(), out.data_ptr(), device.stream())
    return out


def _encrypt_rows(zero: torch.Tensor, m: torch.Tensor, params: RingParams, square: bool = False, f: int = 0,
                  perm: torch.Tensor | None = None) -> torch.Tensor:
    k = zero.shape[0]
    z, mm = zero.contiguous(), m.contiguous()
    out = torch.empty((k, 2, params.n), dtype=torch.int64, device=z.device)
    _native.call("fhe_act_encrypt_rows", params.q, params.p, params.delta, f, int(square), k, params.n,
                 z.data_ptr(), mm.data_ptr(), device.ptr(perm), out.data_ptr(), device.stream())
    return out


def _batch_coeffs(evals_p: torch.Tensor, params: RingParams) -> torch.Tensor:
    """bfv.encode_batch after slot placement: iNTT mod p of eval-order rows."""
    return ring.ntt_rows(evals_p, params.n, [params.p], inverse=True)


@dataclass
class LayerSession:
    """Server-private masks of one layer's protocol run (single use)."""

    plan: RepackPlan
    r: torch.Tensor  # [k_src, n] mod p, over the conv output's slots
    two_r_eval: torch.Tensor  # [k_dst, n] prepare_plaintext(encode_batch(2 r'))
    v_eval: torch.Tensor  # [k_dst, n] NTT(Δ · encode_batch(v)): plain_add in EVAL
    const: torch.Tensor  # [k_dst, n] r'² − r'·2^f + v mod p
    r_dst: np.ndarray = field(default=None, repr=False)  # host r' (server-private)
    v: np.ndarray = field(default=None, repr=False)  # host v (server-private)
    layer_id: int = 0
    round: Round = Round.INIT
    codec: FixedPointCodec | None = None
    ct1: torch.Tensor | None = field(default=None, repr=False)


def offline_prepare_layer(plan: RepackPlan, params: RingParams, rng, frac_bits: int = 0,
                          layer_id: int = 0) -> LayerSession:
    """Masks for one layer: r uniform over every conv
    output slot, v over every slot of the next layout; the batch plaintexts
    2r' and v are encoded, lifted and NTT'd here, offline."""
    n, p, q = params.n, params.p, params.q
    r = rng.integers(0, p, (plan.k_src, n), dtype=np.int64)
    v = rng.integers(0, p, (plan.k_dst, n), dtype=np.int64)
    r_dst = plan.gather_host(r)
    inv_perm = np.empty(n, dtype=np.int64)
    inv_perm[bfv._slot_index(params)] = np.arange(n)
    two_r = _batch_coeffs(device.to_device(np.ascontiguousarray((2 * r_dst % p)[:, inv_perm])), params)
    lifted = torch.empty_like(two_r)
    _native.call("fhe_poly_lift_centered", p, q, plan.k_dst, n, two_r.data_ptr(), lifted.data_ptr(), device.stream())
    two_r_eval = ring.ntt_rows(lifted, n, [q])
    v_coeffs = _batch_coeffs(device.to_device(np.ascontiguousarray(v[:, inv_perm])), params)
    v_delta = bfv._add_delta(None, v_coeffs, params, plan.k_dst)
    v_eval = ring.ntt_rows(v_delta, n, [q])
    rd, vd = device.to_device(r_dst), device.to_device(v)
    rsq = device.to_device(r_dst * r_dst % p)
    const = torch.empty_like(rd)
    _native.call("fhe_act_server_const", p, frac_bits, rd.numel(), rd.data_ptr(), rsq.data_ptr(), vd.data_ptr(),
                 const.data_ptr(), device.stream())
    return LayerSession(plan, device.to_device(r), two_r_eval, v_eval, const, r_dst, v, layer_id, Round.INIT,
                        FixedPointCodec(frac_bits, p))


def _stack_rows(x) -> torch.Tensor:
    return bfv.cts_rows(x.cts if hasattr(x, "cts") else x)


def server_round1_layer(conv_out, session: LayerSession, params: RingParams) -> torch.Tensor:
    """⟦a + r⟧ for every ciphertext of the layer (plain_add of the masks)."""
    _expect(session, Round.INIT)
    cts = conv_out.cts if hasattr(conv_out, "cts") else conv_out
    if len(cts) != session.plan.k_src:
        raise EncodingError("conv output does not match the session's layout")
    if cts[0].encoding != Encoding.DIRECT:
        raise EncodingError("activation input must be direct-encoded")
    msg = _encrypt_rows(bfv.cts_rows(cts), session.r, params)
    session.round = Round.MASKED
    return msg


def _check_budget_rows(params: RingParams, acc: "bfv.MaxAcc"):
    """The client's noise-budget check over every decryption `acc` covers
    (one 8-byte device read)."""
    if bfv._budget(params, acc.value()) <= 0:
        raise ProtocolError("noise budget exhausted: ciphertext no longer decrypts reliably")


def _decrypt_rows_checked(rows: torch.Tensor, domain, sk: bfv.SecretKey, pending: "bfv.MaxAcc | None" = None
                          ) -> torch.Tensor:
    """Decrypt a layer's messages; the noise-budget check runs now (one host
    sync) or, with `pending` (a device max accumulator), is left for the
    caller to run once at the end of the exchange (run_layer_activation: no
    sync between the rounds)."""
    params = sk.params
    cts = bfv.cts_from_rows(rows, params.q, Encoding.DIRECT, domain)
    acc = pending if pending is not None else bfv.MaxAcc(rows.device)
    m = bfv.decrypt_rows_max(cts, sk, acc)
    if pending is None:
        _check_budget_rows(params, acc)
    return m


def client_round1_layer(msg: torch.Tensor, plan: RepackPlan, sk: bfv.SecretKey, zeros: bfv.ZeroRowPool,
                        codec: FixedPointCodec | None = None, pending: "bfv.MaxAcc | None" = None
                        ) -> tuple[torch.Tensor, torch.Tensor]:
    """Decrypt w = a + r, repack into the next layout (w'), return
    (⟦w'² + w'·2^f⟧ direct, ⟦w'⟧ batch) — one pass per step for the layer."""
    params = sk.params
    f = codec.frac_bits if codec else 0
    w = _decrypt_rows_checked(msg, Domain.COEFF, sk, pending)
    z = zeros.take_rows(2 * plan.k_dst)
    ct_sq = _encrypt_rows(z[: plan.k_dst], _gather(plan.idx, w), params, square=True, f=f)
    coeffs = _batch_coeffs(_gather(plan.idx_eval, w), params)
    ct_w = _encrypt_rows(z[plan.k_dst :], coeffs, params)
    return ct_sq, ct_w


def server_round2_layer(msgs: tuple[torch.Tensor, torch.Tensor], session: LayerSession,
                        params: RingParams) -> torch.Tensor:
    """⟦2r'·w' + v⟧ = pmult(to_eval(⟦w'⟧), 2r') + v (batch, EVAL), one pass."""
    _expect(session, Round.MASKED)
    ct_sq, ct_w = msgs
    k = session.plan.k_dst
    if ct_w.shape[0] != k or ct_sq.shape[0] != k:
        raise EncodingError("round-1 messages do not match the session's layout")
    w_eval = ring.ntt_rows(ct_w.reshape(-1, params.n), params.n, [params.q])
    out = torch.empty_like(ct_w)
    _native.call("fhe_ct_pmult_add", params.q, k, params.n, w_eval.data_ptr(), session.two_r_eval.data_ptr(),
                 session.v_eval.data_ptr(), out.data_ptr(), device.stream())
    session.ct1 = ct_sq
    session.round = Round.CROSS_SENT
    return out


def client_round2_layer(msg: torch.Tensor, plan: RepackPlan, sk: bfv.SecretKey,
                        zeros: bfv.ZeroRowPool, pending: "bfv.MaxAcc | None" = None) -> torch.Tensor:
    """Decrypt the batch messages, re-encrypt their slots direct (decode_batch
    as NTT mod p + slot gather fused into the encryption pass)."""
    params = sk.params
    m = _decrypt_rows_checked(msg, Domain.EVAL, sk, pending)
    evals = ring.ntt_rows(m, params.n, [params.p])
    return _encrypt_rows(zeros.take_rows(plan.k_dst), evals, params, perm=plan.slot)


def server_finalize_layer(ct1: torch.Tensor, ct2: torch.Tensor, session: LayerSession, params: RingParams,
                          scale: int = 0):
    """⟦a'² + a'·2^f⟧ = ct1 − ct2 + (r'² − r'·2^f + v), packed for the next conv."""
    from . import conv

    _expect(session, Round.CROSS_SENT)
    plan = session.plan
    out = torch.empty_like(ct1)
    _native.call("fhe_act_finalize", params.q, params.p, params.delta, plan.k_dst, params.n, ct1.data_ptr(),
                 ct2.contiguous().data_ptr(), session.const.data_ptr(), out.data_ptr(), device.stream())
    session.round = Round.DONE
    session.ct1 = None
    cts = bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF)
    return conv.PackedTensor(cts, plan.dst, plan.channels, scale)


class _StaticKey:
    """Stands in for a SecretKey inside a captured exchange: s_eval from a
    static device buffer (refilled per replay), so one graph serves any key."""

    def __init__(self, params: RingParams, s_eval: torch.Tensor):
        self.params, self._s = params, s_eval

    def s_eval_dev(self) -> torch.Tensor:
        return self._s


class _LayerGraph:
    """One layer's whole exchange (both parties, ~20 kernels) captured once per
    (RepackPlan, fraction bits) into a CUDA graph over static operand buffers:
    a replay costs one launch instead of ~20 Python/ctypes launches. The
    kernels and data are the eager path's, so the ciphertexts are identical."""

    def __init__(self, plan: RepackPlan, params: RingParams, f: int):
        n, ks, kd = params.n, plan.k_src, plan.k_dst
        dev = device.require_cuda()
        z = lambda *shape: device.zeros_i64(shape)  # noqa: E731
        self.inp, self.zeros = z(ks, 2, n), z(3 * kd, 2, n)
        self.r, self.two_r, self.v_eval, self.const = z(ks, n), z(kd, n), z(kd, n), z(kd, n)
        self.s_eval = z(n)
        self.acc = bfv.MaxAcc(dev)  # the exchange's largest decryption residual (zeroed by every replay)
        key = _StaticKey(params, self.s_eval)

        def body():
            pending = self.acc
            _native.call("fhe_zero", pending.t.data_ptr(), 8, device.stream())
            m1 = _encrypt_rows(self.inp, self.r, params)
            w = _decrypt_rows_checked(m1, Domain.COEFF, key, pending)
            # the repack gather fused into the encryption of the squares (fhe_act_encrypt_gather)
            ct_sq = torch.empty((kd, 2, n), dtype=torch.int64, device=dev)
            _native.call("fhe_act_encrypt_gather", params.q, params.p, params.delta, f, 1, kd, n,
                         self.zeros.data_ptr(), w.contiguous().data_ptr(), plan.idx.data_ptr(), ct_sq.data_ptr(),
                         device.stream())
            ct_w = _encrypt_rows(self.zeros[kd : 2 * kd], _batch_coeffs(_gather(plan.idx_eval, w), params), params)
            # server: to_eval + pmult(2r') + plain_add(v) in one launch (fhe_ntt_pmult_add)
            m2 = torch.empty_like(ct_w)
            _native.call("fhe_ntt_pmult_add", device.native_plan(n, params.q), kd, ct_w.data_ptr(),
                         self.two_r.data_ptr(), self.v_eval.data_ptr(), m2.data_ptr(), device.stream())
            mm = _decrypt_rows_checked(m2, Domain.EVAL, key, pending)
            evals = ring.ntt_rows(mm, n, [params.p])
            # the client's round-2 message is materialised (it crosses to the server)
            back = _encrypt_rows(self.zeros[2 * kd :], evals, params, perm=plan.slot)
            out = torch.empty_like(ct_sq)
            _native.call("fhe_act_finalize", params.q, params.p, params.delta, kd, n, ct_sq.data_ptr(),
                         back.data_ptr(), self.const.data_ptr(), out.data_ptr(), device.stream())
            return out

        body()  # plans, tables and kernels initialised outside the capture
        torch.cuda.synchronize()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(side), torch.cuda.graph(self.graph, stream=side):
            self.out = body()
        torch.cuda.current_stream().wait_stream(side)

    def run(self, conv_rows: torch.Tensor, session: "LayerSession", sk: bfv.SecretKey, zero_rows: torch.Tensor):
        # the replay's operands into the static buffers: seven copies, one launch (fhe_copy_many)
        pairs = ((conv_rows, self.inp), (zero_rows, self.zeros), (session.r, self.r),
                 (session.two_r_eval, self.two_r), (session.v_eval, self.v_eval), (session.const, self.const),
                 (sk.s_eval_dev(), self.s_eval))
        srcs = (ctypes.c_void_p * 7)()
        dsts = (ctypes.c_void_p * 7)()
        nbytes = (ctypes.c_size_t * 7)()
        keep = []
        for i, (src, dst) in enumerate(pairs):
            src = src.contiguous()
            keep.append(src)
            if src.numel() != dst.numel():
                raise EncodingError("exchange operand does not match the layer graph")
            srcs[i], dsts[i], nbytes[i] = src.data_ptr(), dst.data_ptr(), dst.numel() * 8
        _native.call("fhe_copy_many", 7, srcs, dsts, nbytes, device.stream())
        self.graph.replay()
        return self.out.clone(), self.acc


_layer_graphs: dict = {}


def _graph_for(plan: RepackPlan, params: RingParams, f: int) -> _LayerGraph:
    key = (id(plan), params.fingerprint(), f)
    hit = _layer_graphs.get(key)
    if hit is None or hit[0] is not plan:
        hit = _layer_graphs[key] = (plan, _LayerGraph(plan, params, f))
    return hit[1]


def _defer_budget(acc: "bfv.MaxAcc", into) -> None:
    """Keep the round's largest decryption residual for a later check: an
    8-byte device copy into slot `into = (tensor, index)` (no host read now)."""
    buf, i = into
    buf[i : i + 1].copy_(acc.t)


def run_layer_activation(conv_out, session: LayerSession, sk: bfv.SecretKey, zeros: bfv.ZeroRowPool,
                         params: RingParams, graph: bool | None = None, budget_into=None):
    """Both parties in-process: one layer's full two-round exchange. With
    `graph` (default: FLASHHE_ACT_GRAPH != 0) the exchange replays a CUDA graph
    captured per RepackPlan (identical ciphertexts, one launch).
    `budget_into = (device int64 tensor, index)` (addition): the client's
    noise-budget check is deferred — the round's largest residual is stored
    there for one check after a whole chain (check_deferred_budgets) instead
    of one host read per layer."""
    import os

    if graph is None:
        graph = os.environ.get("FLASHHE_ACT_GRAPH", "1") != "0"
    if graph:
        from . import conv

        plan = session.plan
        _expect(session, Round.INIT)
        cts = conv_out.cts if hasattr(conv_out, "cts") else conv_out
        if len(cts) != plan.k_src:
            raise EncodingError("conv output does not match the session's layout")
        if cts[0].encoding != Encoding.DIRECT:
            raise EncodingError("activation input must be direct-encoded")
        zero_rows = zeros.take_rows(3 * plan.k_dst)  # rounds 1 (2 k) and 2 (k), in the eager order
        f = session.codec.frac_bits if session.codec else 0
        out, maxw = _graph_for(plan, params, f).run(bfv.cts_rows(cts), session, sk, zero_rows)
        session.round = Round.DONE
        if budget_into is not None:
            _defer_budget(maxw, budget_into)
        else:
            _check_budget_rows(params, maxw)
        res = bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF)
        return conv.PackedTensor(res, plan.dst, plan.channels, getattr(conv_out, "scale", 0))
    plan = session.plan
    pending = bfv.MaxAcc()  # the client's noise-budget checks, run once after the exchange (one host sync)
    m1 = server_round1_layer(conv_out, session, params)
    sq, w = client_round1_layer(m1, plan, sk, zeros, session.codec, pending)
    m2 = server_round2_layer((sq, w), session, params)
    back = client_round2_layer(m2, plan, sk, zeros, pending)
    out = server_finalize_layer(sq, back, session, params, getattr(conv_out, "scale", 0))
    if budget_into is not None:
        _defer_budget(pending, budget_into)
    else:
        _check_budget_rows(params, pending)
    return out


# ---------------------------------------------------------------------------
# A masked repack round: the layout change without the activation, for a
# pending stride that a server-side linear layer leaves before the next conv
# (config 5's 2x2 average pool after the stem). An addition beyond the paper,
# in the manner of SPEC's rescale_round: the server masks
# ⟦a⟧ with r, the client decrypts a + r, repacks it and re-encrypts it
# (direct), the server removes the repacked mask r'. One round trip, two
# messages, the client sees only a + r.


def check_deferred_budgets(params: RingParams, residuals) -> None:
    """The client's noise-budget checks of a chain run with `budget_into`: one
    host read of every stored residual; raises like the per-round check."""
    vmax = int(residuals.cpu().numpy().max()) if residuals.numel() else 0  # one D2H copy, no reduction kernel
    if bfv._budget(params, vmax) <= 0:
        raise ProtocolError("noise budget exhausted: ciphertext no longer decrypts reliably")


@dataclass
class RepackSession:
    plan: RepackPlan
    r: torch.Tensor  # [k_src, n] masks mod p over the source slots (server-private)
    neg_r_dst: torch.Tensor  # [k_dst, n] (−r') mod p in the next layout
    round: Round = Round.INIT


def offline_prepare_repack(plan: RepackPlan, params: RingParams, rng) -> RepackSession:
    r = rng.integers(0, params.p, (plan.k_src, params.n), dtype=np.int64)
    neg = (-plan.gather_host(r)) % params.p
    return RepackSession(plan, device.to_device(r), device.to_device(neg))


def run_repack_round(x, session: RepackSession, sk: bfv.SecretKey, zeros: bfv.ZeroRowPool,
                     params: RingParams, budget_into=None):
    """⟦a⟧ (any direct layout, stride pending) -> ⟦a'⟧ packed for the next conv
    (`budget_into`: as run_layer_activation's)."""
    from . import conv

    _expect(session, Round.INIT)
    plan = session.plan
    cts = x.cts if hasattr(x, "cts") else x
    if len(cts) != plan.k_src:
        raise EncodingError("tensor does not match the repack session's layout")
    masked = _encrypt_rows(bfv.cts_rows(cts), session.r, params)  # server: ⟦a + r⟧
    session.round = Round.MASKED
    pending = bfv.MaxAcc()
    w = _decrypt_rows_checked(masked, Domain.COEFF, sk, pending)  # client: a + r, repacked, re-encrypted
    back = _encrypt_rows(zeros.take_rows(plan.k_dst), _gather(plan.idx, w), params)
    out = _encrypt_rows(back, session.neg_r_dst, params)  # server: ⟦a' + r'⟧ − r' (plain_add of −r')
    session.round = Round.DONE
    if budget_into is not None:
        _defer_budget(pending, budget_into)
    else:
        _check_budget_rows(params, pending)
    cts_out = bfv.cts_from_rows(out, params.q, Encoding.DIRECT, Domain.COEFF)
    return conv.PackedTensor(cts_out, plan.dst, plan.channels, getattr(x, "scale", 0))
