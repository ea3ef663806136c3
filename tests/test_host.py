"""Host-side logic and the C ABI surface — CPU only, no kernel launches."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT
from oracle import flash_oracle as O

Q = 1152921486375014401


def _declared_symbols():
    text = (ROOT / "include" / "flashhe.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fhe_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2401_16732_b200 import _native

    lib = ctypes.CDLL(str(_native.LIB_PATH))
    syms = _declared_symbols()
    assert len(syms) >= 25
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes binding covers exactly the declared surface
    assert sorted(_native.SIGNATURES) == syms


def test_host_root_and_tables_match_oracle():
    from paper_2401_16732_b200 import _native

    lib = _native.lib()
    for n, q in [(16, 65537), (2048, Q), (4096, 1152921467550908417), (256, 7681)]:
        psi = ctypes.c_uint64()
        _native.check(lib.fhe_find_root(n, q, ctypes.byref(psi)))
        assert psi.value == O.find_root(n, q)
        pb = np.zeros(n, dtype=np.uint64)
        ib = np.zeros(n, dtype=np.uint64)
        ni = ctypes.c_uint64()
        _native.check(lib.fhe_plan_tables_host(n, q, pb.ctypes.data, ib.ctypes.data, ctypes.byref(ni)))
        ref_p, ref_i, ref_n = O.ntt_tables(n, q)
        assert pb.astype(object).tolist() == ref_p
        assert ib.astype(object).tolist() == ref_i
        assert ni.value == ref_n


def test_c_abi_errors_map_to_reference_exceptions():
    from paper_2401_16732_b200 import _native
    from paper_2401_16732_b200.errors import AccumulatorBudgetError, ParameterError

    lib = _native.lib()
    psi = ctypes.c_uint64()
    with pytest.raises(ParameterError):
        _native.check(lib.fhe_find_root(16, 65539, ctypes.byref(psi)))  # 65539 != 1 mod 32
    with pytest.raises(ParameterError):
        _native.check(lib.fhe_find_root(12, 65537, ctypes.byref(psi)))
    w = np.full((2, 3), 1 << 31, dtype=np.int64)
    with pytest.raises(AccumulatorBudgetError):
        _native.check(lib.fhe_conv_check_budget(w.ctypes.data, 2, 3))
    w[:] = 5
    _native.check(lib.fhe_conv_check_budget(w.ctypes.data, 2, 3))


def test_ntt_plan_host_attributes():
    from paper_2401_16732_b200 import ring

    plan = ring.NttPlan(2048, Q)
    g = np.load(ROOT / "tests" / "golden" / "ntt_default.npz")
    assert np.array_equal(plan.psi_brv, g["psi_brv"])
    assert np.array_equal(plan.ipsi_brv, g["ipsi_brv"])
    assert np.array_equal(plan.eval_perm(3), O.eval_perm(2048, 3))
    with pytest.raises(ring.ParameterError):
        ring.NttPlan(16, 65539)


def test_layouts_match_reference(golden):
    from paper_2401_16732_b200 import conv, params

    P = params.default_params()
    for name, g in golden["conv"].items():
        lay = conv.layout_direct(P, g["H"], g["W"], g["f_w"])
        for k, v in g["layout"].items():
            assert getattr(lay, k) == v, (name, k)
        assert lay.ct_count(g["c_i"]) == g["n_in"]
    pl = golden["pool_fc"]["pool_layout"]
    lay8 = conv.replace(conv.layout_direct(P, 8, 8, 3), c_n=1, stride=8)
    assert all(getattr(lay8, k) == v for k, v in pl.items())


def test_layout_edge_cases():
    from paper_2401_16732_b200 import conv, params
    from paper_2401_16732_b200.errors import ParameterError

    P = params.default_params()
    lay = conv.layout_direct(P, 224, 224, 7)
    assert (lay.frags, lay.halo) == (80, 693)
    assert conv.layout_direct(P, 64, 64, 3).frags == 3
    assert conv.layout_direct(P, 16, 16, 3).c_n == 6
    assert conv.layout_direct(P, 8, 8, 3).c_n == 20
    assert conv.layout_direct(P, 4, 4, 3).c_n == 56
    with pytest.raises(ParameterError):
        conv.ConvLayerSpec(4, 4, 2, 1, 1, np.zeros((1, 1, 2, 2)))
    with pytest.raises(ParameterError):
        conv.ConvLayerSpec(4, 4, 3, 1, 1, np.full((1, 1, 3, 3), 256))


def test_pack_unpack_positions_roundtrip():
    """pack_vectors then channel_positions reads each channel back (host)."""
    from paper_2401_16732_b200 import conv, params

    P = params.default_params()
    rng = np.random.default_rng(0)
    for (c, h, w, f) in [(5, 16, 16, 3), (2, 64, 64, 3), (3, 8, 8, 1), (1, 224, 224, 7)]:
        x = rng.integers(-100, 100, (c, h, w))
        lay = conv.layout_direct(P, h, w, f)
        vecs = conv.pack_vectors(x, lay, P.p)
        for j in range(c):
            ci, si = conv.channel_positions(lay, j)
            got = np.array([vecs[a][b] for a, b in zip(ci, si)])
            assert np.array_equal(got, (x[j] % P.p).ravel())
        if h == 224:  # 7x7 halo (693) does not fit a 1024-slot batch orbit — reference raises too
            with pytest.raises(conv.ParameterError):
                conv.layout_batch(P, h, w, f)
            continue
        blay = conv.layout_batch(P, h, w, f)
        bvecs = conv.pack_vectors(x, blay, P.p)
        for j in range(c):
            ci, si = conv.channel_positions(blay, j)
            assert np.array_equal(np.array([bvecs[a][b] for a, b in zip(ci, si)]), (x[j] % P.p).ravel())


def test_repack_index_matches_unpack_then_pack():
    """The client's one-gather repack (act2pc.repack_index) equals reading
    every channel at its readable slots and packing into the next layout —
    strided, fragmented and multi-tile layouts (conv.py:162-197)."""
    from dataclasses import replace

    from paper_2401_16732_b200 import act2pc, conv, params

    P = params.default_params()
    rng = np.random.default_rng(2)
    cases = [(3, 32, 3, 1, 3), (8, 16, 3, 2, 1), (2, 64, 3, 1, 3), (2, 64, 3, 2, 3), (20, 8, 3, 1, 3), (1, 224, 7, 2, 3)]
    for c, h, f_src, stride, f_dst in cases:
        src = replace(replace(conv.layout_direct(P, h, h, f_src), c_n=1), stride=stride)
        dst = conv.layout_direct(P, h // stride, h // stride, f_dst)
        slots = rng.integers(0, P.p, (src.ct_count(c), P.n))
        idx = act2pc.repack_index(src, c, dst, P.n)
        assert idx.shape == (dst.ct_count(c), P.n) and idx.max() < slots.size
        got = np.where(idx >= 0, slots.reshape(-1)[np.maximum(idx, 0)], 0)
        vals = np.stack([slots[conv.channel_positions(src, j)] for j in range(c)])
        want = np.stack(conv.pack_vectors(vals.reshape(c, h // stride, h // stride), dst, P.p))
        assert np.array_equal(got, want)


def test_conventional_steps_and_storage():
    from paper_2401_16732_b200 import conv, params

    P = params.default_params()
    spec = conv.ConvLayerSpec(16, 16, 3, 4, 4, np.ones((4, 4, 3, 3)))
    import json

    g = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())
    assert conv.conventional_steps(spec, P) == g["conv_conventional"]["steps"]
    # VGG-16 switching keys at T=16: 11.67 MB (paper "12 MB")
    steps = conv.vgg16_step_set(P)
    mb = len(steps) * P.decomp_count * 2 * P.n * 8 / 1e6
    assert abs(mb - 11.67) < 0.05


def test_wire_format_frames():
    """bfv.py:525-561 wire frames: header <BBB> (encoding, domain, seeded), c0
    as little-endian u64, then the 32-byte c1 seed or c1; batched stacks are
    consecutive unseeded frames."""
    import struct

    from paper_2401_16732_b200 import bfv, params
    from paper_2401_16732_b200.ring import Domain, ModPoly

    P = params.default_params()
    rng = np.random.default_rng(12)
    seed = bytes(range(32))
    c0 = rng.integers(0, P.q, P.n, dtype=np.int64)
    c1 = bfv.expand_seed(seed, P)
    fresh = bfv.Ciphertext(ModPoly(c0, P.q), ModPoly(c1, P.q), bfv.Encoding.DIRECT, Domain.COEFF, fresh=True, seed=seed)
    wire = bfv.ct_to_bytes(fresh)
    assert wire == struct.pack("<BBB", 1, 0, 1) + c0.astype("<u8").tobytes() + seed
    assert len(wire) == bfv.ct_wire_size(P, True)
    back = bfv.ct_from_bytes(wire, P)
    assert np.array_equal(back.c0.coeffs, c0) and np.array_equal(back.c1.coeffs, c1) and back.seed == seed
    full = bfv.ct_to_bytes(fresh, seed_compress=False)
    assert full == struct.pack("<BBB", 1, 0, 0) + c0.astype("<u8").tobytes() + c1.astype("<u8").tobytes()
    assert len(full) == bfv.ct_wire_size(P, False)
    ev = bfv.Ciphertext(ModPoly(c1, P.q, Domain.EVAL), ModPoly(c0, P.q, Domain.EVAL), bfv.Encoding.BATCH, Domain.EVAL)
    assert bfv.ct_to_bytes(ev)[:3] == struct.pack("<BBB", 0, 1, 0)  # EVAL never seed-compressed
    cts = [bfv.Ciphertext(ModPoly(rng.integers(0, P.q, P.n, dtype=np.int64), P.q),
                          ModPoly(rng.integers(0, P.q, P.n, dtype=np.int64), P.q), bfv.Encoding.DIRECT, Domain.COEFF)
           for _ in range(3)]
    blob = bfv.cts_to_bytes(cts, bfv.Encoding.DIRECT, Domain.COEFF)
    assert blob == b"".join(bfv.ct_to_bytes(c, seed_compress=False) for c in cts)
    stack = bfv.cts_from_bytes(blob, 3, P, pin=False)
    got = stack.host_stack()
    for i, c in enumerate(cts):
        assert np.array_equal(got[i, 0], c.c0.coeffs) and np.array_equal(got[i, 1], c.c1.coeffs)


def test_wire_frames_match_reference_frames():
    """Frames of privinfer's own bfv.ct_to_bytes (tests/golden/make_wire_golden.py):
    a fresh seeded encryption (seed-compressed and full), an EVAL batch
    ciphertext and a non-fresh sum, and a batch of unseeded frames; the
    package's writer reproduces each byte string and its parser reads them."""
    import hashlib
    import json

    from conftest import GOLDEN
    from paper_2401_16732_b200 import bfv, params
    from paper_2401_16732_b200.ring import Domain, ModPoly

    P = params.default_params()
    meta = json.loads((GOLDEN / "wire.json").read_text())
    arr = np.load(GOLDEN / "wire.npz")
    cts = {}
    for name in meta["batch"]["order"]:
        g = meta[name]
        dom = Domain.EVAL if g["domain"] else Domain.COEFF
        seed = arr[f"{name}_seed"].tobytes() or None
        ct = bfv.Ciphertext(ModPoly(arr[f"{name}_c0"], P.q, dom), ModPoly(arr[f"{name}_c1"], P.q, dom),
                            bfv.Encoding(g["encoding"]), dom, fresh=g["fresh"], seed=seed)
        cts[name] = ct
        seeded, full = bfv.ct_to_bytes(ct), bfv.ct_to_bytes(ct, seed_compress=False)
        assert hashlib.sha256(seeded).hexdigest() == g["h:seeded"] and len(seeded) == g["len:seeded"]
        assert hashlib.sha256(full).hexdigest() == g["h:full"] and len(full) == g["len:full"]
        assert list(seeded[:3]) == g["head"]
        back = bfv.ct_from_bytes(seeded, P)
        assert np.array_equal(back.c0.coeffs, arr[f"{name}_c0"]) and np.array_equal(back.c1.coeffs, arr[f"{name}_c1"])
        assert back.domain == dom and back.encoding == ct.encoding
    assert bfv.ct_wire_size(P, True) == meta["wire_size"]["seeded"]
    assert bfv.ct_wire_size(P, False) == meta["wire_size"]["full"]
    blob = b"".join(bfv.ct_to_bytes(cts[k], seed_compress=False) for k in meta["batch"]["order"])
    assert hashlib.sha256(blob).hexdigest() == meta["batch"]["h"]
    # a batch of unseeded frames from mixed headers is refused by the stack parser
    with pytest.raises(bfv.EncodingError):
        bfv.cts_from_bytes(blob, 3, P, pin=False)
    same = b"".join(bfv.ct_to_bytes(c, seed_compress=False) for c in (cts["summed"], cts["fresh"]))
    stack = bfv.cts_from_bytes(same, 2, P, pin=False).host_stack()
    assert np.array_equal(stack[1, 0], arr["fresh_c0"]) and np.array_equal(stack[0, 1], arr["summed_c1"])


def test_stack_schedule_is_johnson_optimal():
    """conv._stack_schedule orders a stacked launch's independent jobs by
    Johnson's rule for the two-stage (relayout -> GEMM) flow shop: on random
    small instances its makespan equals the brute-force optimum."""
    import itertools
    from types import SimpleNamespace

    from paper_2401_16732_b200 import conv

    def makespan(order, times):
        t1 = t2 = 0.0
        for k in order:
            r, g = times[k]
            t1 += r
            t2 = max(t2, t1) + g
        return t2

    rng = np.random.default_rng(3)
    for _ in range(40):
        m = int(rng.integers(2, 7))
        times = [(float(rng.uniform(0.1, 5)), float(rng.uniform(0.1, 5))) for _ in range(m)]
        stub = {}
        items = []
        for k, (r, g) in enumerate(times):
            plan = SimpleNamespace(tag=k)
            stub[k] = (r, g)
            items.append((plan, None, None, None))
        orig = conv._stage_times
        conv._stage_times = lambda plan: stub[plan.tag]  # the rule under test, on chosen stage times
        try:
            order = [it[0].tag for it in conv._stack_schedule(items)]
        finally:
            conv._stage_times = orig
        assert sorted(order) == list(range(m))
        best = min(makespan(p, times) for p in itertools.permutations(range(m)))
        assert abs(makespan(order, times) - best) < 1e-9


def test_stream_order_smallest_upload_then_largest_download():
    """conv._stream_order: the job with the smallest upload first, the largest
    download second, the rest in the call's order; every job exactly once."""
    from types import SimpleNamespace as NS

    from paper_2401_16732_b200 import conv, params

    P = params.default_params()

    def job(k_in, k_out):
        return (NS(cts=[None] * k_in), None, NS(n_out=k_out))

    meta = [job(240, 5120), job(128, 128), job(16, 32), job(64, 512), job(16, 64)]
    order = conv._stream_order(meta, P)
    assert sorted(order) == list(range(len(meta)))
    assert order[:2] == [2, 0] and order[2:] == [1, 3, 4]
    assert conv._stream_order(meta[:2], P) == [0, 1]


def test_residual_add_rejects_mismatched_layouts():
    """conv.residual_add checks the operand layouts before touching the device."""
    from dataclasses import replace

    from paper_2401_16732_b200 import conv, params
    from paper_2401_16732_b200.errors import EncodingError

    P = params.default_params()
    lay = conv.layout_direct(P, 8, 8, 3)
    y = conv.PackedTensor([], conv._out_layout(lay), 16)
    for bad in (conv.PackedTensor([], conv.layout_direct(P, 16, 16, 3), 16),  # other resolution
                conv.PackedTensor([], lay, 8),  # other channel count
                conv.PackedTensor([], replace(lay, stride=2), 16)):  # stride pending
        with pytest.raises(EncodingError):
            conv.residual_add(y, bad, P)


def test_blocks_and_residual_integer_model():
    """The basic-block map of the stacks and the residual integer model: an
    identity block adds its input, a projection block its strided 1x1 map."""
    from paper_2401_16732_b200 import inference, stacks

    blk = inference.blocks(stacks.config4())
    assert blk["s1b1c2"] == ("s1b1c1", None)
    assert blk["s2b1c2"][1].name == "s2b1proj" and len(blk) == 8
    p = 65537
    L = stacks.Layer
    layers = [L("stem", "conv", 4, 4, 3, 1, 2), L("s1b1c1", "conv", 4, 4, 3, 2, 2), L("s1b1c2", "conv", 4, 4, 3, 2, 2),
              L("avgpool", "pool", 4, 4, 4, 2, 2), L("fc", "fc", 1, 1, 1, 2, 1)]
    rng = np.random.default_rng(3)
    w = inference.random_weights(layers, rng, bound=3)
    x = rng.integers(0, 4, (1, 4, 4))
    sq = lambda a: (a * a + a) % p  # noqa: E731
    a0 = sq(inference._conv_same(x, w["stem"]) % p)
    a1 = sq(inference._conv_same(a0, w["s1b1c1"]) % p)
    a2 = sq((inference._conv_same(a1, w["s1b1c2"]) + a0) % p)
    want = (w["fc"] @ a2.reshape(2, -1).sum(axis=1)) % p
    assert np.array_equal(inference.plain_forward(layers, x, w, p), want)
