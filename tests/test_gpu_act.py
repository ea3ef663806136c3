"""One layer of x²+x activations on the device (SPEC.md:304-331 over row
stacks) with the client repack into the next conv's layout (conv.py:148-197):
bit-exact against the oracle composition, and decrypting to pack(a² + a·2^f)."""

from dataclasses import replace

import numpy as np
import pytest

from oracle import flash_oracle as O

pytestmark = pytest.mark.gpu


def _conv_output(P, rng, sk, H, c, f_w, stride):
    """A real conv_proposed output (small weights) to activate."""
    from paper_2401_16732_b200 import bfv, conv

    x = rng.integers(-3, 4, (c, H, H), dtype=np.int64)
    w = rng.integers(-2, 3, (c, c, f_w, f_w), dtype=np.int64)
    layer = conv.ConvLayerSpec(H, H, f_w, c, c, w)
    xin = conv.pack_input(x, P, f_w, lambda pt: bfv.encrypt_private(pt, sk, rng))
    y = conv.conv_proposed(xin, layer, P)
    if stride > 1:
        y = conv.PackedTensor(y.cts, replace(y.layout, stride=stride), y.channels, y.scale)
    return y


def _oracle_decrypt(cts, s, P):
    rows = np.stack([np.stack([ct.c0.coeffs, ct.c1.coeffs]) for ct in cts])
    return np.stack([O.decrypt_round(O.decrypt_phase(r[0], r[1], s, P.q), P.q, P.p)[0] for r in rows])


def _pack_channels(slots, src_layout, channels, dst_layout, p):
    """Oracle repack: read each channel at its readable slots, pack_vectors."""
    from paper_2401_16732_b200 import conv

    h, w = src_layout.out_dims()
    vals = np.stack([slots[conv.channel_positions(src_layout, j)] for j in range(channels)])
    return np.stack(conv.pack_vectors(vals.reshape(channels, h, w), dst_layout, p))


@pytest.mark.parametrize(
    "H,c,f_src,stride,f_dst,frac",
    [
        (32, 2, 3, 1, 3, 0),  # one tile per ct (c_n 1)
        (16, 8, 3, 1, 3, 0),  # c_n 6 in and out (packed)
        (16, 8, 3, 2, 1, 0),  # stride-2 subsample into a 1x1 layout (projection input)
        (64, 2, 3, 1, 3, 0),  # fragmented in and out (3 fragments, halos)
        (64, 2, 3, 2, 3, 2),  # fragmented -> stride 2 -> c_n 1, fixed-point f = 2
    ],
)
def test_layer_activation_bit_exact(H, c, f_src, stride, f_dst, frac):
    from paper_2401_16732_b200 import act2pc, bfv, conv, params

    P = params.default_params()
    p, q = P.p, P.q
    rng = np.random.default_rng(1000 + H + c + stride + f_dst)
    sk = bfv.keygen(P, rng)
    y = _conv_output(P, rng, sk, H, c, f_src, stride)
    dst = conv.layout_direct(P, H // stride, H // stride, f_dst)
    plan = act2pc.RepackPlan(y.layout, c, dst, P)
    assert plan.k_src == len(y.cts) and plan.k_dst == dst.ct_count(c)
    sess = act2pc.offline_prepare_layer(plan, P, rng, frac_bits=frac)
    zeros = bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst)
    z = zeros.rows.cpu().numpy().copy()
    out = act2pc.run_layer_activation(y, sess, sk, zeros, P)
    assert sess.round == act2pc.Round.DONE and len(zeros) == 0
    assert out.layout == dst and out.channels == c

    # oracle composition from the conv output, the masks and the zero pool
    s = np.asarray(sk.s.coeffs)
    a_src = _oracle_decrypt(y.cts, s, P)
    r_src = sess.r.cpu().numpy()
    w_dst = _pack_channels((a_src + r_src) % p, y.layout, c, dst, p)
    r_dst = _pack_channels(r_src, y.layout, c, dst, p)
    assert np.array_equal(r_dst, sess.r_dst)
    k = plan.k_dst
    yv = O.x2x_client(w_dst, p, frac)
    zv = (2 * r_dst.astype(object) * w_dst + sess.v) % p
    cv = O.x2x_server_const(r_dst, r_dst * r_dst % p, sess.v, p, frac)
    sq0 = O.add_delta(z[:k, 0], yv, q, p)
    back0 = O.add_delta(z[2 * k :, 0], zv.astype(np.int64), q, p)
    exp0 = O.add_delta(((sq0.astype(object) - back0) % q).astype(np.int64), cv, q, p)
    exp1 = ((z[:k, 1].astype(object) - z[2 * k :, 1]) % q).astype(np.int64)
    got = bfv.cts_rows(out.cts).cpu().numpy()
    assert np.array_equal(got[:, 0], exp0)
    assert np.array_equal(got[:, 1], exp1)

    # and it decrypts to a² + a·2^f, packed for the next convolution
    a = conv.unpack(y, sk, signed=False)
    fa = (a.astype(object) ** 2 + a.astype(object) * (1 << frac)) % p
    expect = np.stack(conv.pack_vectors(fa.astype(np.int64), dst, p))
    m, _ = bfv.decrypt_rows(out.cts, sk)
    assert np.array_equal(m.cpu().numpy(), expect)


def test_layer_activation_feeds_next_conv():
    """conv -> x²+x (repacked) -> conv: the second conv decrypts to the
    integer conv of (conv(x))² + conv(x)."""
    from paper_2401_16732_b200 import act2pc, bfv, conv, params

    P = params.default_params()
    rng = np.random.default_rng(77)
    sk = bfv.keygen(P, rng)
    H, c = 16, 4
    x = rng.integers(-2, 3, (c, H, H), dtype=np.int64)
    w1 = rng.integers(-1, 2, (c, c, 3, 3), dtype=np.int64)
    w2 = rng.integers(-1, 2, (c, c, 3, 3), dtype=np.int64)
    l1 = conv.ConvLayerSpec(H, H, 3, c, c, w1)
    l2 = conv.ConvLayerSpec(H, H, 3, c, c, w2)
    xin = conv.pack_input(x, P, 3, lambda pt: bfv.encrypt_private(pt, sk, rng))
    y1 = conv.conv_proposed(xin, l1, P)
    plan = act2pc.RepackPlan(y1.layout, c, conv.layout_direct(P, H, H, 3), P)
    act = act2pc.run_layer_activation(y1, act2pc.offline_prepare_layer(plan, P, rng), sk,
                                      bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst), P)
    y2 = conv.conv_proposed(act, l2, P)

    def plain_conv(v, wt):
        pad = np.pad(v, ((0, 0), (1, 1), (1, 1)))
        out = np.zeros_like(v)
        for dy in range(3):
            for dx in range(3):
                out += np.einsum("oi,ihw->ohw", wt[:, :, dy, dx], pad[:, dy : dy + H, dx : dx + H])
        return out

    a1 = plain_conv(x, w1)
    want = bfv.centered(plain_conv(a1 * a1 + a1, w2), P.p)
    assert np.array_equal(conv.unpack(y2, sk), want)


def test_zero_rows_match_single_precompute():
    from paper_2401_16732_b200 import bfv, params

    P = params.default_params()
    sk = bfv.keygen(P, np.random.default_rng(5))
    rows = bfv.precompute_zero_rows(sk, np.random.default_rng(9), 3).rows.cpu().numpy()
    pool = bfv.precompute_zero(sk, np.random.default_rng(9), 3)
    for i, zc in enumerate(pool.entries):
        assert np.array_equal(rows[i, 0], zc.ct.c0.coeffs)
        assert np.array_equal(rows[i, 1], zc.ct.c1.coeffs)


def test_layer_protocol_errors():
    from paper_2401_16732_b200 import act2pc, bfv, conv, params
    from paper_2401_16732_b200.errors import EncodingError, ProtocolError

    P = params.default_params()
    rng = np.random.default_rng(3)
    sk = bfv.keygen(P, rng)
    y = _conv_output(P, rng, sk, 16, 2, 3, 1)
    dst = conv.layout_direct(P, 16, 16, 3)
    plan = act2pc.RepackPlan(y.layout, 2, dst, P)
    with pytest.raises(EncodingError):
        act2pc.RepackPlan(y.layout, 2, conv.layout_direct(P, 8, 8, 3), P)  # wrong geometry
    sess = act2pc.offline_prepare_layer(plan, P, rng)
    zeros = bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst - 1)  # one short
    m1 = act2pc.server_round1_layer(y, sess, P)
    with pytest.raises(ProtocolError):
        act2pc.server_round1_layer(y, sess, P)  # masks are single use
    sq, w = act2pc.client_round1_layer(m1, plan, sk, zeros)
    m2 = act2pc.server_round2_layer((sq, w), sess, P)
    with pytest.raises(ProtocolError):
        act2pc.client_round2_layer(m2, plan, sk, zeros)  # pool exhausted: never reuse a zero


def test_layer_graph_matches_eager():
    """The CUDA-graph replay of the layer exchange gives the eager path's
    ciphertexts bit for bit (same masks, same zero rows)."""
    from paper_2401_16732_b200 import act2pc, bfv, conv, params

    P = params.default_params()
    rng = np.random.default_rng(99)
    sk = bfv.keygen(P, rng)
    y = _conv_output(P, rng, sk, 16, 8, 3, 2)
    plan = act2pc.repack_plan(y.layout, 8, conv.layout_direct(P, 8, 8, 3), P)
    outs = []
    for graph in (False, True, True):
        r2 = np.random.default_rng(5)
        sess = act2pc.offline_prepare_layer(plan, P, r2)
        zeros = bfv.precompute_zero_rows(sk, r2, 3 * plan.k_dst)
        outs.append(bfv.cts_rows(act2pc.run_layer_activation(y, sess, sk, zeros, P, graph=graph).cts).cpu().numpy())
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
