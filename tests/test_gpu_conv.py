"""K1 (Flash conv / pool / FC) parity on the device vs reference goldens + oracle."""

import numpy as np
import pytest
import torch

from conftest import load_npz, sha
from oracle import flash_oracle as O

pytestmark = pytest.mark.gpu

Q = 1152921486375014401
P_ = 270337
N = 2048


def _P():
    from paper_2401_16732_b200 import params

    return params.default_params()


def _cts(arr, q=Q):
    from paper_2401_16732_b200 import bfv

    t = torch.from_numpy(np.ascontiguousarray(arr)).cuda()
    return bfv.cts_from_rows(t, q, bfv.Encoding.DIRECT, bfv.Domain.COEFF)


def _out(cts):
    from paper_2401_16732_b200 import bfv

    return bfv.cts_rows(cts).cpu().numpy()


def _case(golden, name):
    g = golden["conv"][name]
    r = np.random.default_rng(g["seed"])
    arr = r.integers(0, Q, (g["n_in"], 2, N), dtype=np.int64)
    w = r.integers(-127, 128, (g["c_o"], g["c_i"], g["f_w"], g["f_w"]), dtype=np.int64)
    b = r.integers(-1000, 1000, g["c_o"], dtype=np.int64) if g["bias"] else None
    return g, arr, w, b


@pytest.mark.parametrize("path", ["auto", "int"])
@pytest.mark.parametrize("name", ["cfg1", "r20_stem", "r20_s2", "r20_s3", "proj1x1", "frag64", "frag64_bias",
                                  "packed16_bias", "r18_8x8_512", "vgg4x4", "stem7x7_224"])
def test_conv_proposed_matches_reference(golden, name, path, monkeypatch):
    from paper_2401_16732_b200 import conv

    monkeypatch.setenv("FLASHHE_CONV_PATH", path)
    g, arr, w, b = _case(golden, name)
    P = _P()
    lay = conv.layout_direct(P, g["H"], g["W"], g["f_w"])
    spec = conv.ConvLayerSpec(g["H"], g["W"], g["f_w"], g["c_i"], g["c_o"], w, bias=b)
    y = conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, g["c_i"]), spec, P)
    assert len(y.cts) == g["n_out"]
    assert sha(_out(y.cts)) == g["h:out"]
    assert y.layout.c_n == 1 and y.channels == g["c_o"]


TC_CASES = [
    # H, W, f_w, c_i, c_o, bias
    (64, 64, 3, 32, 8, True),     # fragmented (3 frags, halo 67) + bias
    (16, 16, 3, 16, 136, True),   # c_n = 6, two output-channel tiles, bias
    (8, 8, 3, 48, 20, False),     # c_n = 20, partial channel block
    (32, 32, 1, 40, 130, False),  # 1x1 projection, c_n = 2
    (4, 4, 3, 33, 5, False),      # c_n = 56
]


@pytest.mark.parametrize("case", TC_CASES)
def test_conv_tc_vs_oracle(case, monkeypatch):
    """K1-TC against the pinned oracle (and against K1 on the integer pipes)."""
    from oracle.flash_oracle import add_bias
    from paper_2401_16732_b200 import conv

    H, W, f_w, c_i, c_o, bias = case
    P = _P()
    rng = np.random.default_rng(H * 1000 + c_i)
    lay = conv.layout_direct(P, H, W, f_w)
    arr = rng.integers(0, Q, (lay.ct_count(c_i), 2, N), dtype=np.int64)
    arr[:, :, ::17] = 0
    arr[:, :, 5::17] = Q - 1
    w = rng.integers(-127, 128, (c_o, c_i, f_w, f_w), dtype=np.int64)
    b = rng.integers(-5000, 5000, c_o, dtype=np.int64) if bias else None
    spec = conv.ConvLayerSpec(H, W, f_w, c_i, c_o, w, bias=b)
    plan = conv.conv_plan(spec, lay, P)
    assert plan.tc is not None, "case should take the tensor-core path"
    monkeypatch.setenv("FLASHHE_CONV_PATH", "tc")
    y_tc = _out(conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, c_i), spec, P).cts)
    monkeypatch.setenv("FLASHHE_CONV_PATH", "int")
    y_int = _out(conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, c_i), spec, P).cts)
    assert np.array_equal(y_tc, y_int)
    layd = {"n": N, "w_p": lay.w_p, "pad": lay.pad, "tile": lay.tile, "c_n": lay.c_n, "frags": lay.frags}
    chans = sorted({0, c_o // 2, c_o - 1})
    ref = O.conv_proposed(arr, w.reshape(c_o, c_i, -1), layd, Q, channels=chans)
    if b is not None:
        out_lay = {"n": N, "height": H, "width": W, "pad": lay.pad, "w_p": lay.w_p, "frags": lay.frags,
                   "frag_len": lay.frag_len, "halo": lay.halo}
        ref = add_bias(ref, b[chans], O.bias_masks(out_lay), P.delta, P.p, Q)
    sel = np.concatenate([np.arange(c * lay.frags, (c + 1) * lay.frags) for c in chans])
    assert np.array_equal(y_tc[sel], ref)


def test_conv_proposed_stream_matches_single_calls():
    """The overlapped serving API gives exactly conv_proposed's ciphertexts,
    for host-resident (pinned and pageable) and device-resident inputs."""
    from paper_2401_16732_b200 import bfv, conv

    P = _P()
    rng = np.random.default_rng(77)
    jobs, refs = [], []
    for k, (H, f_w, c_i, c_o) in enumerate([(16, 3, 32, 40), (8, 3, 64, 130), (32, 1, 24, 16), (16, 3, 3, 8)]):
        lay = conv.layout_direct(P, H, H, f_w)
        arr = rng.integers(0, Q, (lay.ct_count(c_i), 2, N), dtype=np.int64)
        spec = conv.ConvLayerSpec(H, H, f_w, c_i, c_o, rng.integers(-127, 128, (c_o, c_i, f_w, f_w)))
        refs.append(_out(conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, c_i), spec, P).cts))
        cts = _cts(arr) if k == 2 else bfv.cts_from_host(arr, Q, pin=(k != 1))
        jobs.append((conv.PackedTensor(cts, lay, c_i), spec))
    outs = conv.conv_proposed_stream(jobs, P)
    for y, ref in zip(outs, refs):
        assert np.array_equal(y.cts.host_stack(), ref)
        assert np.array_equal(_out(y.cts), ref)


def test_conv_proposed_stream_large_pinned_after_pageable():
    """Large pinned host jobs after a pageable tensor-core job (which takes
    the issue_k1 path) in one call, with the digit-plane scratch first grown
    to its final size inside the call: every job still equals conv_proposed
    (the fast path once kept a scratch pointer across a growth),
    repeated so the allocator recycles the inputs and outputs."""
    from paper_2401_16732_b200 import bfv, conv, device

    P = _P()
    rng = np.random.default_rng(78)
    geoms = [(16, 3, 32, 40, False), (64, 3, 64, 64, True), (56, 3, 64, 64, True), (8, 3, 64, 130, True)]
    specs = []
    for H, f_w, c_i, c_o, pin in geoms:
        lay = conv.layout_direct(P, H, H, f_w)
        spec = conv.ConvLayerSpec(H, H, f_w, c_i, c_o, rng.integers(-127, 128, (c_o, c_i, f_w, f_w)))
        specs.append((lay, spec, c_i, pin))
    for rep in range(2):
        jobs, refs = [], []
        for lay, spec, c_i, pin in specs:
            arr = rng.integers(0, Q, (lay.ct_count(c_i), 2, N), dtype=np.int64)
            refs.append(_out(conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, c_i), spec, P).cts))
            jobs.append((conv.PackedTensor(bfv.cts_from_host(arr, Q, pin=pin), lay, c_i), spec))
        torch.cuda.synchronize()
        device._scratch.pop((torch.cuda.current_device(), "conv_tc_x"), None)  # the call sizes it afresh
        outs = conv.conv_proposed_stream(jobs, P)
        for k, (y, ref) in enumerate(zip(outs, refs)):
            assert np.array_equal(y.cts.host_stack(), ref), f"rep {rep} job {k}"


def test_conv_cfg1_full_arrays():
    from paper_2401_16732_b200 import conv

    d = load_npz("conv_cfg1.npz")
    P = _P()
    lay = conv.layout_direct(P, 32, 32, 3)
    spec = conv.ConvLayerSpec(32, 32, 3, 16, 16, d["weights"])
    y = conv.conv_proposed(conv.PackedTensor(_cts(d["cts"]), lay, 16), spec, P)
    assert np.array_equal(_out(y.cts), d["out"])


def test_config1_end_to_end_decrypt():
    """Real encryptions: bit-exact ciphertexts and identical decrypted outputs."""
    from paper_2401_16732_b200 import bfv, conv
    from paper_2401_16732_b200.ring import ModPoly

    d = load_npz("config1_e2e.npz")
    P = _P()
    sk = bfv.SecretKey(ModPoly(d["s"], P.q), P)
    lay = conv.layout_direct(P, 32, 32, 3)
    x = conv.PackedTensor(_cts(d["cts"]), lay, 16)
    y = conv.conv_proposed(x, conv.ConvLayerSpec(32, 32, 3, 16, 16, d["w"]), P)
    assert np.array_equal(_out(y.cts), d["out"])
    assert np.array_equal(conv.unpack(y, sk), d["dec"])
    # and the decrypted result equals the plaintext integer convolution
    xp = np.pad(d["x"], ((0, 0), (1, 1), (1, 1)))
    ref = np.zeros((16, 32, 32), dtype=np.int64)
    for dy in range(3):
        for dx in range(3):
            ref += np.einsum("oi,ihw->ohw", d["w"][:, :, dy, dx], xp[:, dy : dy + 32, dx : dx + 32])
    assert np.array_equal(d["dec"], ref)


def test_config1_pack_encrypt_bit_exact(golden):
    """The same seed through our pack_input/encrypt_private gives the reference's ciphertexts."""
    from paper_2401_16732_b200 import bfv, conv

    d = load_npz("config1_e2e.npz")
    P = _P()
    r = np.random.default_rng(golden["config1_e2e"]["seed"])
    sk = bfv.keygen(P, r)
    assert np.array_equal(sk.s.coeffs, d["s"])
    xin = r.integers(0, 8, (16, 32, 32), dtype=np.int64)
    assert np.array_equal(xin, d["x"])
    w = r.integers(-127, 128, (16, 16, 3, 3), dtype=np.int64)
    assert np.array_equal(w, d["w"])
    x = conv.pack_input(xin, P, 3, lambda pt: bfv.encrypt_private(pt, sk, r))
    assert np.array_equal(_out(x.cts), d["cts"])
    y = conv.conv_proposed(x, conv.ConvLayerSpec(32, 32, 3, 16, 16, w), P)
    assert [bfv.noise_budget(c, sk) for c in y.cts[:2]] == golden["config1_e2e"]["budget_out"]


def test_pool_fc_match_reference(golden):
    from paper_2401_16732_b200 import conv

    g = golden["pool_fc"]
    P = _P()
    r = np.random.default_rng(g["seed"])
    arr = r.integers(0, Q, (8, 2, N), dtype=np.int64)
    lay8 = conv.replace(conv.layout_direct(P, 8, 8, 3), c_n=1)
    pooled = conv.avg_pool(conv.PackedTensor(_cts(arr), lay8, 8), 8, P)
    assert sha(_out(pooled.cts)) == g["h:pool"]
    assert pooled.layout.stride == 8
    fcw = r.integers(-127, 128, (10, 8), dtype=np.int64)
    fcb = r.integers(-100, 100, 10, dtype=np.int64)
    fco = conv.fully_connected(pooled, fcw, P, bias=fcb)
    assert sha(_out(fco)) == g["h:fc"]


def test_conv_small_ring(golden):
    from paper_2401_16732_b200 import conv, params

    g = golden["conv_n256"]
    P = params.RingParams(**g["params"])
    r = np.random.default_rng(g["seed"])
    lay = conv.layout_direct(P, 4, 4, 3)
    arr = r.integers(0, P.q, (lay.ct_count(9), 2, 256), dtype=np.int64)
    wts = r.integers(-127, 128, (5, 9, 3, 3), dtype=np.int64)
    y = conv.conv_proposed(conv.PackedTensor(_cts(arr, P.q), lay, 9), conv.ConvLayerSpec(4, 4, 3, 9, 5, wts), P)
    assert sha(_out(y.cts)) == g["h:out"]


def test_conv_edge_cases():
    from paper_2401_16732_b200 import conv
    from paper_2401_16732_b200.errors import AccumulatorBudgetError, EncodingError, ParameterError

    P = _P()
    rng = np.random.default_rng(4)
    lay = conv.layout_direct(P, 8, 8, 3)
    arr = rng.integers(0, Q, (1, 2, N), dtype=np.int64)
    x = conv.PackedTensor(_cts(arr), lay, 3)
    # identity kernel -> input
    w = np.zeros((1, 1, 3, 3), dtype=np.int64)
    w[0, 0, 1, 1] = 1
    y = conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, 1), conv.ConvLayerSpec(8, 8, 3, 1, 1, w), P)
    assert np.array_equal(_out(y.cts)[0], arr[0])
    # all-zero weights -> zero ciphertext
    y = conv.conv_proposed(x, conv.ConvLayerSpec(8, 8, 3, 3, 2, np.zeros((2, 3, 3, 3))), P)
    assert not _out(y.cts).any()
    # extreme weights ±255 (MAX_WEIGHT_BITS bound) vs oracle
    w = rng.choice([-255, 255, -1, 0, 1], size=(4, 3, 3, 3))
    y = conv.conv_proposed(x, conv.ConvLayerSpec(8, 8, 3, 3, 4, w), P)
    layd = {"n": N, "w_p": lay.w_p, "pad": 1, "tile": lay.tile, "c_n": lay.c_n, "frags": 1}
    assert np.array_equal(_out(y.cts), O.conv_proposed(arr, w.reshape(4, 3, 9), layd, Q))
    # extreme coefficients: all q-1 / zeros
    arr2 = np.full((1, 2, N), Q - 1, dtype=np.int64)
    arr2[0, 1, ::3] = 0
    w = np.full((2, 3, 3, 3), -255)
    y = conv.conv_proposed(conv.PackedTensor(_cts(arr2), lay, 3), conv.ConvLayerSpec(8, 8, 3, 3, 2, w), P)
    assert np.array_equal(_out(y.cts), O.conv_proposed(arr2, w.reshape(2, 3, 9), layd, Q))
    # errors, raised before launch like the reference
    with pytest.raises(ParameterError):
        conv.conv_proposed(x, conv.ConvLayerSpec(16, 16, 3, 3, 2, np.zeros((2, 3, 3, 3))), P)
    with pytest.raises(ParameterError):
        conv.conv_proposed(conv.PackedTensor(x.cts, conv.replace(lay, stride=2), 3),
                           conv.ConvLayerSpec(8, 8, 3, 3, 2, np.zeros((2, 3, 3, 3))), P)
    bx = conv.PackedTensor([conv.bfv.Ciphertext(c.c0, c.c1, conv.Encoding.BATCH, c.domain) for c in x.cts], lay, 3)
    with pytest.raises(EncodingError):
        conv.conv_proposed(bx, conv.ConvLayerSpec(8, 8, 3, 3, 2, np.zeros((2, 3, 3, 3))), P)
    with pytest.raises(AccumulatorBudgetError):
        conv._check_budget(np.full((1, 1 << 25), 200))  # Σ|w| = 6.7e9 ≥ 2^32


def test_full_size_r18_layer_properties():
    """(8², 512→512): linearity over inputs, and sampled channels vs the oracle."""
    from paper_2401_16732_b200 import conv

    P = _P()
    rng = np.random.default_rng(12)
    lay = conv.layout_direct(P, 8, 8, 3)
    n_in = lay.ct_count(512)
    a = rng.integers(0, Q, (n_in, 2, N), dtype=np.int64)
    b = rng.integers(0, Q, (n_in, 2, N), dtype=np.int64)
    w = rng.integers(-127, 128, (512, 512, 3, 3), dtype=np.int64)
    spec = conv.ConvLayerSpec(8, 8, 3, 512, 512, w)
    run = lambda arr: _out(conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, 512), spec, P).cts)
    ya, yb, yab = run(a), run(b), run(((a.astype(object) + b) % Q).astype(np.int64))
    assert np.array_equal(yab, ((ya.astype(object) + yb) % Q).astype(np.int64))
    layd = {"n": N, "w_p": lay.w_p, "pad": 1, "tile": lay.tile, "c_n": lay.c_n, "frags": 1}
    chans = [0, 255, 511]
    ref = O.conv_proposed(a, w.reshape(512, 512, 9), layd, Q, channels=chans)
    assert np.array_equal(ya[chans], ref)


def test_conv_conventional_matches_reference(golden):
    from paper_2401_16732_b200 import bfv, conv

    g = golden["conv_conventional"]
    P = _P()
    r = np.random.default_rng(g["seed"])
    sk = bfv.keygen(P, r)
    xc = r.integers(0, 8, (4, 16, 16), dtype=np.int64)
    wc = r.integers(-127, 128, (4, 4, 3, 3), dtype=np.int64)
    spec = conv.ConvLayerSpec(16, 16, 3, 4, 4, wc)
    swk = bfv.gen_switching_keys(sk, conv.conventional_steps(spec, P), r, decomp_log=conv.CONV_DECOMP_LOG)
    xb = conv.pack_input(xc, P, 3, lambda pt: bfv.encrypt_private(pt, sk, r), batch=True)
    assert sha(_out(xb.cts)) == g["h:in"]
    y = conv.conv_conventional(xb, spec, swk, P)
    assert sha(_out(y.cts)) == g["h:out"]
    assert conv.unpack(y, sk).tolist() == g["dec"]


def test_conv_conventional_fragmented_matches_reference(golden):
    """Fragmented batch layout (32x32 tile > n/2 slots) with bias, vs the
    reference run with the harness-side _galois_element shim."""
    from paper_2401_16732_b200 import bfv, conv

    g = golden["conv_conventional_frag"]
    P = _P()
    r = np.random.default_rng(g["seed"])
    sk = bfv.keygen(P, r)
    xf = r.integers(0, 8, (2, 32, 32), dtype=np.int64)
    wf = r.integers(-127, 128, (3, 2, 3, 3), dtype=np.int64)
    spec = conv.ConvLayerSpec(32, 32, 3, 2, 3, wf, bias=np.array([5, 0, -7], dtype=np.int64))
    assert conv.conventional_steps(spec, P) == g["steps"]
    swk = bfv.gen_switching_keys(sk, conv.conventional_steps(spec, P), r, decomp_log=conv.CONV_DECOMP_LOG)
    xb = conv.pack_input(xf, P, 3, lambda pt: bfv.encrypt_private(pt, sk, r), batch=True)
    assert sha(_out(xb.cts)) == g["h:in"]
    y = conv.conv_conventional(xb, spec, swk, P)
    assert sha(_out(y.cts)) == g["h:out"]
    assert conv.unpack(y, sk).tolist() == g["dec"]


def test_fully_connected_tensor_core_matches_int_and_oracle(monkeypatch):
    """Config-4 FC shape (512 -> 200, one value per pooled ciphertext, bias):
    the tensor-core path (one tap, per-input DRot slot as channel offset)
    gives exactly the integer-pipe ciphertexts and the oracle's rows."""
    from paper_2401_16732_b200 import conv

    P = _P()
    r = np.random.default_rng(512)
    c, v_out = 512, 200
    lay = conv.replace(conv.replace(conv.layout_direct(P, 8, 8, 3), c_n=1), stride=8)
    arr = r.integers(0, Q, (c, 2, N), dtype=np.int64)
    x = conv.PackedTensor(_cts(arr), lay, c)
    w = r.integers(-127, 128, (v_out, c), dtype=np.int64)
    b = r.integers(-100, 100, v_out, dtype=np.int64)
    tc = _out(conv.fully_connected(x, w, P, bias=b))
    monkeypatch.setenv("FLASHHE_CONV_PATH", "int")
    ref = _out(conv.fully_connected(x, w, P, bias=b))
    assert np.array_equal(tc, ref)
    pos = [conv.channel_positions(lay, j) for j in range(c)]
    ct_idx = np.concatenate([p[0] for p in pos])
    slots = np.concatenate([p[1] for p in pos])
    rows = [0, 77, 199]
    want = O.fully_connected(arr, w[rows], ct_idx, slots, Q)
    delta = P.delta
    for i, o in enumerate(rows):  # bias: Δ·b[o] on slot 0 of c0 (conv.py:626-668)
        want[i, 0, 0] = (int(want[i, 0, 0]) + delta * (int(b[o]) % P.p)) % Q
    assert np.array_equal(tc[rows], want)


@pytest.mark.parametrize("h,k,c", [(32, 2, 3), (64, 2, 2), (8, 8, 4), (16, 4, 8)])
def test_avg_pool_separable_matches_oracle(h, k, c):
    """The separable pool kernel equals the k²-tap DRot sum (conv.py:604-623)
    on packed, fragmented and global-pool geometries."""
    from paper_2401_16732_b200 import conv

    P = _P()
    r = np.random.default_rng(h * 10 + k)
    lay = conv.layout_direct(P, h, h, 3)
    arr = r.integers(0, Q, (lay.ct_count(c), 2, N), dtype=np.int64)
    pooled = conv.avg_pool(conv.PackedTensor(_cts(arr), lay, c), k, P)
    assert pooled.layout.stride == k
    assert np.array_equal(_out(pooled.cts), O.avg_pool(arr, k, lay.w_p, Q))


@pytest.mark.parametrize("H,c_i,c_o", [(16, 8, 20), (32, 3, 17), (8, 24, 24)])
def test_conv_conventional_fused_matches_materialized(monkeypatch, H, c_i, c_o):
    """The fused rotate-multiply-accumulate pass (fhe_rot_pmac, rotations never
    written) gives exactly the two-kernel ciphertexts (batched K4 rotations +
    fhe_pmac) — packed layouts with column swaps, fragmented layouts, more
    than one 16-output tile — and decrypts to the plain convolution."""
    from paper_2401_16732_b200 import bfv, conv

    P = _P()
    r = np.random.default_rng(H * 100 + c_o)
    sk = bfv.keygen(P, r)
    x = r.integers(0, 4, (c_i, H, H), dtype=np.int64)
    w = r.integers(-3, 4, (c_o, c_i, 3, 3), dtype=np.int64)
    spec = conv.ConvLayerSpec(H, H, 3, c_i, c_o, w)
    swk = bfv.gen_switching_keys(sk, conv.conventional_steps(spec, P), r, decomp_log=conv.CONV_DECOMP_LOG)
    xb = conv.pack_input(x, P, 3, lambda pt: bfv.encrypt_private(pt, sk, r), batch=True)
    fused = _out(conv.conv_conventional(xb, spec, swk, P).cts)
    monkeypatch.setenv("FLASHHE_CONVENTIONAL", "materialized")
    mat = conv.conv_conventional(xb, spec, swk, P)
    assert np.array_equal(fused, _out(mat.cts))
    pad = np.pad(x, ((0, 0), (1, 1), (1, 1)))
    want = np.zeros((c_o, H, H), dtype=np.int64)
    for dy in range(3):
        for dx in range(3):
            want += np.einsum("oi,ihw->ohw", w[:, :, dy, dx], pad[:, dy : dy + H, dx : dx + H])
    assert np.array_equal(conv.unpack(mat, sk), bfv.centered(want, P.p))


# K1-TC epilogue variants (csrc/conv_tc.cu): q = 2^60 - delta with delta < 2^35
# takes the pseudo-Mersenne reduction (finish_pm / finish_pm_pair, the
# reference's default q), any other 2^56 <= q < 2^62 the Shoup reduction; the
# 32-bit plane pairs apply to short contractions (127·255·257·c_i·taps < 2^31:
# 1x1 projections, the tap-folded 7x7 stem). Each case is checked against the
# integer-pipe kernel (an independent implementation) and the oracle. (The
# moduli are primes = 1 mod 2n, as RingParams requires.)
_EPI_MODULI = {
    "pm_default": 1152921486375014401,  # delta = 0x43eb3afff
    "pm_edge": 1152921470247149569,  # delta = 0x7ffff5fff, just below 2^35
    "shoup_60": 1152921467550908417,  # delta = 0x8a0b4bfff >= 2^35
    "shoup_61": 2305843003754438657,  # a 61-bit q
    "shoup_57": 72057595874308097,  # a 57-bit q (2^56 <= q)
}


ILV_CASES = [
    # H, W, f_w, c_i, c_o, bias — layers that take the interleaved position groups (c_o <= 64)
    (56, 56, 3, 64, 64, True),    # a config-5 s1 layer: fragmented, 2 channel blocks, 12 merged taps, bias
    (224, 224, 7, 3, 64, True),   # the config-5 stem: row-folded, 8 merged taps, pair epilogue, bias
    (16, 16, 3, 40, 37, True),    # c_n = 6, c_o not a multiple of 16 (partly active warp), bias
    (8, 8, 3, 70, 24, False),     # c_n = 20, 3 channel blocks (the last partial), c_o <= 32: two quadrants active
    (32, 32, 3, 64, 64, False),   # c_n = 1, rep-1 layer before (long contraction)
]


@pytest.mark.parametrize("case", ILV_CASES)
def test_conv_tc_interleaved_groups(case, monkeypatch):
    """Layers with c_o <= 64 run two interleaved position groups (LayerDesc.ilv:
    merged taps, window read at stride 2, lane-pair exchange in the epilogue):
    equal to the integer-pipe kernel on every coefficient, to the stacked-group
    launch (FLASHHE_TC_ILV=0) and to the oracle on sampled channels."""
    from oracle.flash_oracle import add_bias
    from paper_2401_16732_b200 import conv

    H, W, f_w, c_i, c_o, bias = case
    P = _P()
    rng = np.random.default_rng(H * 77 + c_i)
    lay = conv.layout_direct(P, H, W, f_w)
    arr = rng.integers(0, Q, (lay.ct_count(c_i), 2, N), dtype=np.int64)
    arr[:, :, ::19] = Q - 1
    w = rng.integers(-127, 128, (c_o, c_i, f_w, f_w), dtype=np.int64)
    b = rng.integers(-5000, 5000, c_o, dtype=np.int64) if bias else None

    def run(path, ilv):
        monkeypatch.setenv("FLASHHE_CONV_PATH", path)
        monkeypatch.setenv("FLASHHE_TC_ILV", ilv)
        spec = conv.ConvLayerSpec(H, W, f_w, c_i, c_o, w, bias=b)  # a fresh plan cache per mode
        plan = conv.conv_plan(spec, lay, P)
        assert plan.tc is not None
        if path == "tc":
            assert (plan.tc.tsplit == 2) == (ilv == "auto"), "interleaving should follow FLASHHE_TC_ILV"
        return _out(conv.conv_proposed(conv.PackedTensor(_cts(arr), lay, c_i), spec, P).cts)

    y_ilv = run("tc", "auto")
    assert np.array_equal(y_ilv, run("int", "auto"))
    assert np.array_equal(y_ilv, run("tc", "0"))
    layd = {"n": N, "w_p": lay.w_p, "pad": lay.pad, "tile": lay.tile, "c_n": lay.c_n, "frags": lay.frags}
    chans = sorted({0, c_o // 2, c_o - 1})
    ref = O.conv_proposed(arr, w.reshape(c_o, c_i, -1), layd, Q, channels=chans)
    if b is not None:
        out_lay = {"n": N, "height": H, "width": W, "pad": lay.pad, "w_p": lay.w_p, "frags": lay.frags,
                   "frag_len": lay.frag_len, "halo": lay.halo}
        ref = add_bias(ref, b[chans], O.bias_masks(out_lay), P.delta, P.p, Q)
    sel = np.concatenate([np.arange(c * lay.frags, (c + 1) * lay.frags) for c in chans])
    assert np.array_equal(y_ilv[sel], ref)


@pytest.mark.parametrize("qname", sorted(_EPI_MODULI))
@pytest.mark.parametrize("geom", [(8, 3, 64, 130), (16, 1, 64, 96), (32, 7, 3, 16)])
def test_tc_epilogue_moduli(qname, geom, monkeypatch):
    from paper_2401_16732_b200 import conv, params

    q = _EPI_MODULI[qname]
    H, f_w, c_i, c_o = geom
    P = params.RingParams(n=N, q=q, p=P_, sigma=3.2, decomp_log=16)
    rng = np.random.default_rng(H + 7 * c_o)
    lay = conv.layout_direct(P, H, H, f_w)
    arr = rng.integers(0, q, (lay.ct_count(c_i), 2, N), dtype=np.int64)
    arr[:, :, ::13] = q - 1  # extreme coefficients: the largest plane sums
    w = rng.choice([-127, 127, -1, 0, 1, 5], size=(c_o, c_i, f_w, f_w))
    w[: c_o // 2] = 127  # a channel block of maximal positive sums
    spec = conv.ConvLayerSpec(H, H, f_w, c_i, c_o, w)
    assert conv.conv_plan(spec, lay, P).tc is not None
    monkeypatch.setenv("FLASHHE_CONV_PATH", "tc")
    y_tc = _out(conv.conv_proposed(conv.PackedTensor(_cts(arr, q), lay, c_i), spec, P).cts)
    monkeypatch.setenv("FLASHHE_CONV_PATH", "int")
    y_int = _out(conv.conv_proposed(conv.PackedTensor(_cts(arr, q), lay, c_i), spec, P).cts)
    assert np.array_equal(y_tc, y_int)
    layd = {"n": N, "w_p": lay.w_p, "pad": lay.pad, "tile": lay.tile, "c_n": lay.c_n, "frags": lay.frags}
    chans = sorted({0, c_o // 2, c_o - 1})
    ref = O.conv_proposed(arr, w.reshape(c_o, c_i, -1), layd, q, channels=chans)
    got = y_tc.reshape(c_o, lay.frags, 2, N)[chans].reshape(-1, 2, N)
    assert np.array_equal(got, ref.reshape(-1, 2, N))


def test_conv_proposed_many_matches_single_calls():
    """conv_proposed_many (one stacked launch for several inputs of one layer,
    incl. more than the 24 jobs of one launch) equals conv_proposed per input."""
    from paper_2401_16732_b200 import conv

    P = _P()
    rng = np.random.default_rng(99)
    for H, f_w, c_i, c_o, count in [(16, 3, 32, 48, 3), (8, 3, 64, 130, 26)]:
        lay = conv.layout_direct(P, H, H, f_w)
        spec = conv.ConvLayerSpec(H, H, f_w, c_i, c_o, rng.integers(-127, 128, (c_o, c_i, f_w, f_w)))
        xs = [conv.PackedTensor(_cts(rng.integers(0, Q, (lay.ct_count(c_i), 2, N), dtype=np.int64)), lay, c_i)
              for _ in range(count)]
        ys = conv.conv_proposed_many(xs, spec, P)
        for x, y in zip(xs, ys):
            ref = conv.conv_proposed(x, spec, P)
            assert np.array_equal(_out(y.cts), _out(ref.cts))
            assert y.layout == ref.layout and y.channels == ref.channels and y.scale == ref.scale


def test_conv_proposed_many_edges():
    """No inputs -> no launch, empty result; a geometry mismatch raises like conv_proposed."""
    from paper_2401_16732_b200 import conv
    from paper_2401_16732_b200.errors import ParameterError

    P = _P()
    rng = np.random.default_rng(5)
    spec = conv.ConvLayerSpec(8, 8, 3, 4, 4, rng.integers(-127, 128, (4, 4, 3, 3)))
    assert conv.conv_proposed_many([], spec, P) == []
    lay = conv.layout_direct(P, 16, 16, 3)
    x = conv.PackedTensor(_cts(rng.integers(0, Q, (lay.ct_count(4), 2, N), dtype=np.int64)), lay, 4)
    with pytest.raises(ParameterError):
        conv.conv_proposed_many([x], spec, P)
