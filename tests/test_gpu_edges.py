"""Edge cases through the device path: empty batches, zero weights, a single
channel, maximum-weight budgets, and the reference's error behaviour."""

import numpy as np
import pytest
import torch

from oracle import flash_oracle as O

pytestmark = pytest.mark.gpu

Q = 1152921486375014401


def _P():
    from paper_2401_16732_b200 import params

    return params.default_params()


def test_empty_batches_are_no_ops():
    from paper_2401_16732_b200 import conv, ring

    P = _P()
    t = torch.empty((0, P.n), dtype=torch.int64, device="cuda")
    assert ring.ntt_rows(t, P.n, [P.q]).shape == (0, P.n)
    assert conv.conv_proposed_stream([], P) == []


def test_all_zero_weights_give_zero_or_bias_only():
    from paper_2401_16732_b200 import bfv, conv

    P = _P()
    rng = np.random.default_rng(5)
    lay = conv.layout_direct(P, 16, 16, 3)
    arr = rng.integers(0, Q, (lay.ct_count(4), 2, P.n), dtype=np.int64)
    x = conv.PackedTensor(bfv.cts_from_rows(torch.from_numpy(arr).cuda(), Q, bfv.Encoding.DIRECT, bfv.Domain.COEFF),
                          lay, 4)
    zero = conv.ConvLayerSpec(16, 16, 3, 4, 3, np.zeros((3, 4, 3, 3), dtype=np.int64))
    y = bfv.cts_rows(conv.conv_proposed(x, zero, P).cts).cpu().numpy()
    assert not y.any()
    biased = conv.ConvLayerSpec(16, 16, 3, 4, 3, np.zeros((3, 4, 3, 3), dtype=np.int64), bias=np.array([1, 0, -2]))
    yb = bfv.cts_rows(conv.conv_proposed(x, biased, P).cts).cpu().numpy()
    assert not yb[:, 1].any() and not yb[1, 0].any()
    mask = conv._bias_mask(conv.replace(lay, c_n=1), 0).astype(bool)
    assert np.all(yb[0, 0][mask] == P.delta) and not yb[0, 0][~mask].any()
    assert np.all(yb[2, 0][mask] == P.delta * (P.p - 2) % Q)


def test_single_channel_and_max_weight_budget():
    """c_i = c_o = 1 with |w| = 255 (the reference's 8-bit bound: integer-pipe
    K1) and a tensor-core layer at the largest exact contraction of config 4."""
    from paper_2401_16732_b200 import bfv, conv

    P = _P()
    rng = np.random.default_rng(6)
    lay = conv.layout_direct(P, 32, 32, 3)
    arr = rng.integers(0, Q, (1, 2, P.n), dtype=np.int64)
    w = np.full((1, 1, 3, 3), 255, dtype=np.int64)
    x = conv.PackedTensor(bfv.cts_from_rows(torch.from_numpy(arr).cuda(), Q, bfv.Encoding.DIRECT, bfv.Domain.COEFF),
                          lay, 1)
    y = bfv.cts_rows(conv.conv_proposed(x, conv.ConvLayerSpec(32, 32, 3, 1, 1, w), P).cts).cpu().numpy()
    ld = {"n": P.n, "w_p": lay.w_p, "pad": lay.pad, "tile": lay.tile, "c_n": lay.c_n, "frags": lay.frags}
    want = O.conv_proposed(arr, w.reshape(1, 1, 9), ld, Q)
    assert np.array_equal(y, want)
    with pytest.raises(conv.ParameterError):
        conv.ConvLayerSpec(32, 32, 3, 1, 1, np.full((1, 1, 3, 3), 256))


def test_act2pc_layer_single_channel():
    from paper_2401_16732_b200 import act2pc, bfv, conv

    P = _P()
    rng = np.random.default_rng(8)
    sk = bfv.keygen(P, rng)
    a = rng.integers(-20, 20, (1, 8, 8), dtype=np.int64)
    x = conv.pack_input(a, P, 3, lambda pt: bfv.encrypt_private(pt, sk, rng))
    plan = act2pc.RepackPlan(conv.replace(x.layout, c_n=1), 1, conv.layout_direct(P, 8, 8, 3), P)
    assert plan.k_src == 1 and plan.k_dst == 1
    out = act2pc.run_layer_activation(x, act2pc.offline_prepare_layer(plan, P, rng), sk,
                                      bfv.precompute_zero_rows(sk, rng, 3), P)
    assert np.array_equal(conv.unpack(out, sk), bfv.centered(a * a + a, P.p))


def test_copy_many_kernel():
    """fhe_copy_many: several device copies of different sizes in one launch."""
    import ctypes

    import numpy as np
    import torch

    from paper_2401_16732_b200 import _native, device

    rng = np.random.default_rng(3)
    sizes = [1, 7, 4096, 0, 33, 100000]
    srcs = [torch.from_numpy(rng.integers(-2**62, 2**62, max(s, 1), dtype=np.int64)).cuda() for s in sizes]
    dsts = [torch.zeros(max(s, 1), dtype=torch.int64, device="cuda") for s in sizes]
    a = (ctypes.c_void_p * 6)(*[t.data_ptr() for t in srcs])
    b = (ctypes.c_void_p * 6)(*[t.data_ptr() for t in dsts])
    c = (ctypes.c_size_t * 6)(*[8 * s for s in sizes])
    _native.call("fhe_copy_many", 6, a, b, c, device.stream())
    for s, x, y in zip(sizes, srcs, dsts):
        assert torch.equal(x[:s], y[:s])
        if s == 0:
            assert int(y[0]) == 0
