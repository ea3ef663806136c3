"""ResNet shortcut addition (conv.residual_add / fhe_residual_add) vs the
reference-pinned ring ops it composes: bfv.drot (the DRot that moves channel
j's tile of a packed block input to slot 0) and bfv.hadd, ciphertext by
ciphertext; then the decrypted slots of an encrypted block input added to a
real conv output."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _P():
    from paper_2401_16732_b200 import params

    return params.default_params()


@pytest.mark.parametrize("hw,channels", [(8, 20), (8, 37), (16, 5), (32, 3), (56, 4)])
def test_residual_add_equals_drot_hadd(hw, channels):
    from paper_2401_16732_b200 import bfv, conv, device
    from paper_2401_16732_b200.bfv import Encoding
    from paper_2401_16732_b200.ring import Domain

    P = _P()
    rng = np.random.default_rng(hw * 100 + channels)
    lay = conv.layout_direct(P, hw, hw, 3)
    out_lay = conv._out_layout(lay)
    k_in, k_out = lay.ct_count(channels), out_lay.ct_count(channels)
    a_rows = device.to_device(rng.integers(0, P.q, (k_in, 2, P.n), dtype=np.uint64).astype(np.int64))
    y_rows = device.to_device(rng.integers(0, P.q, (k_out, 2, P.n), dtype=np.uint64).astype(np.int64))
    mk = lambda r: bfv.cts_from_rows(r, P.q, Encoding.DIRECT, Domain.COEFF)  # noqa: E731
    a = conv.PackedTensor(mk(a_rows), lay, channels)
    y = conv.PackedTensor(mk(y_rows.clone()), out_lay, channels)
    got = conv.residual_add(y, a, P, inplace=False)
    got_rows = bfv.cts_rows(got.cts).cpu().numpy()
    c_n, tile = (1, 0) if lay.fragmented else (lay.c_n, lay.tile)
    for j in range(k_out):
        want = bfv.hadd(mk(y_rows)[j], bfv.drot(mk(a_rows)[j // c_n], tile * (j % c_n)))
        assert np.array_equal(got_rows[j], np.stack([want.c0.coeffs, want.c1.coeffs])), j
    # in place: y's own rows
    inpl = conv.residual_add(y, a, P)
    assert torch.equal(bfv.cts_rows(inpl.cts), torch.as_tensor(got_rows, device=y_rows.device))


@pytest.mark.parametrize("hw,channels", [(8, 24), (56, 3)])
def test_residual_add_decrypts_to_the_sum(hw, channels):
    """A real conv output plus the encrypted block input: the readable slots
    of every channel decrypt to conv + input (mod p)."""
    from paper_2401_16732_b200 import bfv, conv

    P = _P()
    rng = np.random.default_rng(5 + hw)
    sk = bfv.keygen(P, rng)
    x = rng.integers(0, 16, (channels, hw, hw), dtype=np.int64)
    w = rng.integers(-127, 128, (channels, channels, 3, 3), dtype=np.int64)
    xin = conv.pack_input_private(x, P, 3, sk, rng)
    y = conv.conv_proposed(xin, conv.ConvLayerSpec(hw, hw, 3, channels, channels, w), P)
    z = conv.residual_add(y, xin, P)
    from paper_2401_16732_b200 import inference

    want = (inference._conv_same(x, w) + x) % P.p
    rows = bfv.decrypt_rows(z.cts, sk)[0].cpu().numpy()
    for j in range(channels):
        ci, si = conv.channel_positions(z.layout, j)
        got = rows[ci, si] % P.p
        assert np.array_equal(got, want[j].reshape(-1)), j
