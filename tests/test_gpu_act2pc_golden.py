"""x²+x share protocol pinned to REFERENCE transcripts.

tests/golden/act2pc.json holds, per case, the sha256 of every protocol
message produced by composing privinfer's own primitives (plain_add,
encode_direct/encode_batch, encrypt_online, to_eval, pmult, psub, decrypt,
decode_*, conv.channel_positions / pack_vectors) per SPEC.md:304-331 —
tests/golden/make_act2pc_golden.py. The GPU protocol (act2pc.*_layer, the
CUDA-graph replay run_layer_activation, and the single-ciphertext API
run_activation) must reproduce every message bit for bit from the same seed.
"""

import json
from dataclasses import replace

import numpy as np
import pytest
import torch

from conftest import GOLDEN, sha

pytestmark = pytest.mark.gpu

GOLD = json.loads((GOLDEN / "act2pc.json").read_text())
SINGLE = GOLD.pop("single_ct")
CASES = GOLD


def _setup(g):
    from paper_2401_16732_b200 import act2pc, bfv, conv, params

    P = params.default_params()
    rng = np.random.default_rng(g["seed"])
    sk = bfv.keygen(P, rng)
    H, c = g["H"], g["channels"]
    src0 = replace(conv.layout_direct(P, H, H, 3), c_n=1)
    a = rng.integers(-60, 60, (c, H, H), dtype=np.int64)
    cts = [bfv.encrypt_private(bfv.encode_direct(v, P), sk, rng) for v in conv.pack_vectors(a, src0, P.p)]
    rows = bfv.cts_rows(cts).reshape(-1, 2, P.n)
    assert sha(rows.cpu().numpy()) == g["h:conv_out"]
    src = replace(src0, stride=g["stride"])
    ho = H // g["stride"]
    dst = conv.layout_direct(P, ho, ho, g["f_next"])
    plan = act2pc.RepackPlan(src, c, dst, P)
    assert (plan.k_src, plan.k_dst) == (g["k_src"], g["k_dst"])
    zeros = bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst)
    sess = act2pc.offline_prepare_layer(plan, P, rng, frac_bits=g["frac_bits"])
    x = conv.PackedTensor(bfv.cts_from_rows(rows.clone(), P.q, bfv.Encoding.DIRECT, bfv.Domain.COEFF), src, c)
    return P, sk, plan, zeros, sess, x


def _h(t):
    return sha(t.reshape(-1, 2, t.shape[-1]).cpu().numpy())


@pytest.mark.parametrize("name", sorted(CASES))
def test_layer_protocol_matches_reference_transcript(name):
    from paper_2401_16732_b200 import act2pc, bfv

    g = CASES[name]
    P, sk, plan, zeros, sess, x = _setup(g)
    m1 = act2pc.server_round1_layer(x, sess, P)
    assert _h(m1) == g["h:m1"]
    sq, ctw = act2pc.client_round1_layer(m1, plan, sk, zeros, sess.codec)
    assert _h(sq) == g["h:sq"]
    assert _h(ctw) == g["h:ct_w"]
    m2 = act2pc.server_round2_layer((sq, ctw), sess, P)
    assert _h(m2) == g["h:m2"]
    back = act2pc.client_round2_layer(m2, plan, sk, zeros)
    assert _h(back) == g["h:back"]
    out = act2pc.server_finalize_layer(sq, back, sess, P)
    assert _h(bfv.cts_rows(out.cts)) == g["h:out"]
    # the same exchange as one CUDA-graph replay, from the same seed
    P, sk, plan, zeros, sess, x = _setup(g)
    out_g = act2pc.run_layer_activation(x, sess, sk, zeros, P, graph=True)
    assert _h(bfv.cts_rows(out_g.cts)) == g["h:out"]


def test_single_ciphertext_api_matches_reference_transcript():
    """run_activation and its round functions on one ciphertext (the SPEC's
    per-ciphertext calls, no layout change), f = 3."""
    from paper_2401_16732_b200 import act2pc, bfv, params

    g = SINGLE
    P = params.default_params()

    def setup():
        rng = np.random.default_rng(g["seed"])
        sk = bfv.keygen(P, rng)
        a = rng.integers(-300, 300, P.n, dtype=np.int64)
        ct = bfv.encrypt_private(bfv.encode_direct(a, P), sk, rng)
        pool = bfv.precompute_zero(sk, rng, 3)
        (sess,) = act2pc.offline_prepare(1, P, rng, frac_bits=g["frac_bits"])
        return sk, ct, pool, sess

    rows = lambda c: bfv.cts_rows([c]).cpu().numpy()  # noqa: E731
    sk, ct, pool, sess = setup()
    assert sha(rows(ct)) == g["h:ct"]
    m1 = act2pc.server_round1(ct, sess, P)
    assert sha(rows(m1)) == g["h:m1"]
    sq, w = act2pc.client_round1(m1, sk, pool, sess.codec)
    assert sha(rows(sq)) == g["h:sq"] and sha(rows(w)) == g["h:ct_w"]
    m2 = act2pc.server_round2((sq, w), sess, P)
    assert sha(rows(m2)) == g["h:m2"]
    back = act2pc.client_round2(m2, sk, pool)
    assert sha(rows(back)) == g["h:back"]
    out = act2pc.server_finalize(sq, back, sess, P)
    assert sha(rows(out)) == g["h:out"]
    sk, ct, pool, sess = setup()
    assert sha(rows(act2pc.run_activation(ct, sess, sk, pool, P))) == g["h:out"]
