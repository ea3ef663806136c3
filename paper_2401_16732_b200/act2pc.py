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

from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native, bfv, device
from .bfv import Ciphertext, Encoding
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
