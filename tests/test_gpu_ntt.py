"""K2 (batched NTT) and K3 (elementwise) parity on the device vs oracle/goldens."""

import numpy as np
import pytest
import torch

from conftest import load_npz, sha
from oracle import flash_oracle as O

pytestmark = pytest.mark.gpu

Q = 1152921486375014401


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


def test_ntt_default_golden():
    from paper_2401_16732_b200 import ring

    g = load_npz("ntt_default.npz")
    plan = ring.get_plan(2048, Q)
    assert np.array_equal(plan.fwd(g["x"]), g["fwd"])
    assert np.array_equal(plan.inv(g["x"]), g["inv"])
    assert np.array_equal(plan.inv(plan.fwd(g["x"])), g["x"])


@pytest.mark.parametrize("n,q", [(2, 5), (4, 17), (8, 17), (16, 65537), (32, 12289), (64, 12289), (256, 7681),
                                 (1024, 12289), (2048, 270337)])
def test_ntt_small_and_odd_sizes(n, q):
    from paper_2401_16732_b200 import ring

    rng = np.random.default_rng(n)
    x = rng.integers(0, q, (3, n), dtype=np.int64)
    plan = ring.get_plan(n, q)
    f = plan.fwd(x)
    i = plan.inv(x)
    for r in range(3):
        assert np.array_equal(f[r], O.ntt_fwd(x[r], q)), (n, q)
        assert np.array_equal(i[r], O.ntt_inv(x[r], q)), (n, q)


def test_spec_ntt_kats():
    from paper_2401_16732_b200 import ring
    from paper_2401_16732_b200.ring import Domain, ModPoly

    d = np.zeros(16, dtype=np.int64)
    d[0] = 1
    assert ring.ntt_forward(ModPoly(d, 65537)).coeffs.tolist() == [1] * 16
    assert ring.ntt_forward(ModPoly(np.zeros(16), 65537)).coeffs.tolist() == [0] * 16
    f = ModPoly(np.array([1, 1, 0, 0]), 17)
    assert ring.negacyclic_mul(f, f).coeffs.tolist() == [1, 2, 1, 0]
    x3 = ModPoly(np.array([0, 0, 0, 1]), 17)
    x1 = ModPoly(np.array([0, 1, 0, 0]), 17)
    assert ring.negacyclic_mul(x3, x1).coeffs.tolist() == [16, 0, 0, 0]
    with pytest.raises(ring.ParameterError):
        ring.ntt_inverse(ModPoly(d, 65537, Domain.COEFF))


def test_negacyclic_mul_vs_schoolbook():
    from paper_2401_16732_b200 import ring
    from paper_2401_16732_b200.ring import ModPoly

    rng = np.random.default_rng(11)
    for _ in range(20):
        f = rng.integers(0, Q, 32)
        g = rng.integers(0, 1 << 40, 32)
        # q must be ≡ 1 mod 64 for n = 32: the default q is ≡ 1 mod 4096
        out = ring.negacyclic_mul(ModPoly(f, Q), ModPoly(g, Q)).coeffs
        assert np.array_equal(out, O.negacyclic_schoolbook(f, g, Q))


@pytest.mark.parametrize("N", [4096, 8192, 16384])
def test_config2_batched_limbs(golden, N):
    """[B=3][L=4][P=2][N] in one launch; each row checked against the
    reference's per-limb transform (golden hashes for the limb inputs)."""
    from paper_2401_16732_b200 import ring

    ent = golden["ntt"]["sweep"][str(N)]
    limbs = ent["limbs"]
    B, L, P = 3, len(limbs), 2
    x = np.zeros((B, L, P, N), dtype=np.int64)
    rng = np.random.default_rng(N)
    for l, q in enumerate(limbs):
        x[:, l] = rng.integers(0, q, (B, P, N), dtype=np.int64)
    golden_rows = []
    for l, (q, e) in enumerate(zip(limbs, ent["limb"])):
        r = np.random.default_rng(e["seed"])
        a = r.integers(0, q, N, dtype=np.int64)
        x[1, l, 0] = a
        golden_rows.append(e)
    t = _dev(x)
    f = ring.ntt_rows(t, N, limbs, P=P).cpu().numpy()
    i = ring.ntt_rows(t, N, limbs, inverse=True, P=P).cpu().numpy()
    for l, e in enumerate(golden_rows):
        assert sha(f[1, l, 0]) == e["h:fwd"]
        assert sha(i[1, l, 0]) == e["h:inv"]
    # round trip everywhere, and a random row vs the oracle
    back = ring.ntt_rows(_dev(f), N, limbs, inverse=True, P=P).cpu().numpy()
    assert np.array_equal(back, x)
    assert np.array_equal(f[2, 3, 1], O.ntt_fwd(x[2, 3, 1], limbs[3]))


@pytest.mark.parametrize("N", [4096, 8192, 16384])
def test_config2_full_batch_properties(golden, N):
    """Config 2 at the size bench.py times ([B=64][L=4][P=2][N], one launch;
    the split two-kernel transform at N >= 8192): size-independent properties
    over every row — inverse(forward(x)) == x, forward is Z_q-linear, forward of
    a negacyclic shift x·X is the forward of x times the forward of X — plus
    sampled rows against the oracle (ring.py:129-162)."""
    from paper_2401_16732_b200 import ring

    limbs = golden["ntt"]["sweep"][str(N)]["limbs"]
    B, L, P = 64, len(limbs), 2
    rng = np.random.default_rng(N + 1)
    x = np.zeros((B, L, P, N), dtype=np.int64)
    y = np.zeros_like(x)
    for l, q in enumerate(limbs):
        x[:, l] = rng.integers(0, q, (B, P, N), dtype=np.int64)
        y[:, l] = rng.integers(0, q, (B, P, N), dtype=np.int64)
    qv = _dev(np.array(limbs, dtype=np.int64)).view(1, L, 1, 1)
    tx, ty = _dev(x), _dev(y)
    fx = ring.ntt_rows(tx, N, limbs, P=P)
    fy = ring.ntt_rows(ty, N, limbs, P=P)
    assert int(fx.min()) >= 0 and bool((fx < qv).all())
    assert torch.equal(ring.ntt_rows(fx, N, limbs, inverse=True, P=P), tx)
    assert torch.equal(ring.ntt_rows((tx + ty) % qv, N, limbs, P=P), (fx + fy) % qv)
    # x·X: coefficients move up one slot, the top one wraps around negated
    sh = torch.roll(tx, 1, dims=-1)
    sh[..., 0] = (qv - sh[..., 0:1]).squeeze(-1) % qv.squeeze(-1)
    mono = np.zeros((1, L, 1, N), dtype=np.int64)
    mono[..., 1] = 1
    fm = ring.ntt_rows(_dev(mono), N, limbs, P=1)  # [1][L][1][N]
    fsh = ring.ntt_rows(sh, N, limbs, P=P).cpu().numpy()
    fxh, fmh = fx.cpu().numpy(), fm.cpu().numpy()
    for l, q in enumerate(limbs):
        want = (fxh[::16, l].astype(object) * fmh[0, l, 0].astype(object)) % q  # every 16th ciphertext (big ints)
        assert np.array_equal(fsh[::16, l].astype(object), want), f"limb {l}: shift theorem"
    for b, l, p in ((0, 0, 0), (63, L - 1, 1), (17, 1, 0)):
        assert np.array_equal(fxh[b, l, p], O.ntt_fwd(x[b, l, p], limbs[l]))


@pytest.mark.parametrize("N", [4096, 16384])
def test_config2_pmult_add(golden, N):
    from paper_2401_16732_b200 import _native, ring

    ent = golden["ntt"]["sweep"][str(N)]
    limbs = ent["limbs"]
    a = np.zeros((len(limbs), N), dtype=np.int64)
    b = np.zeros_like(a)
    for l, (q, e) in enumerate(zip(limbs, ent["limb"])):
        r = np.random.default_rng(e["seed"])
        a[l] = r.integers(0, q, N, dtype=np.int64)
        b[l] = r.integers(0, q, N, dtype=np.int64)
    mul = ring.binary_rows(_native.OP_MUL, _dev(a), _dev(b), N, limbs).cpu().numpy()
    add = ring.binary_rows(_native.OP_ADD, _dev(a), _dev(b), N, limbs).cpu().numpy()
    for l, e in enumerate(ent["limb"]):
        assert sha(mul[l]) == e["h:pmul"]
        assert sha(add[l]) == e["h:add"]
    # the Shoup form bfv.pmult uses gives the same words (golden), also broadcast
    # over a batch of 3 ciphertexts x 2 polys
    import torch

    from paper_2401_16732_b200 import device

    L = len(limbs)
    mods = _native.u64_array(limbs)
    bd = _dev(b)
    bp = torch.empty_like(bd)
    _native.call("fhe_shoup_companions", mods, L, 1, 1, N, bd.data_ptr(), bp.data_ptr(), device.stream())
    ad = _dev(a)
    out = torch.empty_like(ad)
    _native.call("fhe_poly_mul_shoup", mods, L, 1, 1, N, ad.data_ptr(), bd.data_ptr(), bp.data_ptr(), 1, 1,
                 out.data_ptr(), device.stream())
    got = out.cpu().numpy()
    for l, e in enumerate(ent["limb"]):
        assert sha(got[l]) == e["h:pmul"]
    rng = np.random.default_rng(N)
    xs = np.stack([rng.integers(0, q, (3, 2, N), dtype=np.int64) for q in limbs], axis=1)  # [3][L][2][N]
    xd = _dev(xs)
    o2 = torch.empty_like(xd)
    _native.call("fhe_poly_mul_shoup", mods, L, 3, 2, N, xd.data_ptr(), bd.data_ptr(), bp.data_ptr(), 1, 1,
                 o2.data_ptr(), device.stream())
    ref = ring.binary_rows(_native.OP_MUL, xd, bd, N, limbs, P=2, Bb=1, Pb=1).cpu().numpy()
    assert np.array_equal(o2.cpu().numpy(), ref)


@pytest.mark.parametrize("B,Pb", [(2, 1), (9, 2), (64, 1)])
def test_pmult_shoup_batch_broadcast(B, Pb):
    """Shoup pmult with one plaintext broadcast over the batch (the chunked
    kernel: full and partial 4-ciphertext chunks, per-poly or shared plaintext)
    equals the generic Barrett multiply word for word."""
    import torch

    from paper_2401_16732_b200 import _native, device, params, ring

    N, L = 4096, 3
    limbs = params.limb_primes(N, params.find_plaintext_modulus(N), L)
    mods = _native.u64_array(limbs)
    rng = np.random.default_rng(B * 10 + Pb)
    x = np.stack([rng.integers(0, q, (B, 2, N), dtype=np.int64) for q in limbs], axis=1)  # [B][L][2][N]
    w = np.stack([rng.integers(0, q, (Pb, N), dtype=np.int64) for q in limbs])[None]  # [1][L][Pb][N]
    xd, wd = _dev(x), _dev(w)
    wp = torch.empty_like(wd)
    _native.call("fhe_shoup_companions", mods, L, 1, Pb, N, wd.data_ptr(), wp.data_ptr(), device.stream())
    out = torch.empty_like(xd)
    _native.call("fhe_poly_mul_shoup", mods, L, B, 2, N, xd.data_ptr(), wd.data_ptr(), wp.data_ptr(), 1, Pb,
                 out.data_ptr(), device.stream())
    ref = ring.binary_rows(_native.OP_MUL, xd, wd, N, limbs, P=2, Bb=1, Pb=Pb).cpu().numpy()
    assert np.array_equal(out.cpu().numpy(), ref)


def test_digit_ntt_vs_oracle():
    from paper_2401_16732_b200 import _native, device

    rng = np.random.default_rng(5)
    n, T, l = 2048, 16, 4
    src = rng.integers(0, Q, (2, n), dtype=np.int64)
    out = torch.empty((2, l, n), dtype=torch.int64, device="cuda")
    _native.call("fhe_ntt_forward_digits", device.plan_array(n, [Q]), 1, 2, _dev(src).data_ptr(), out.data_ptr(),
                 T, l, device.stream())
    out = out.cpu().numpy()
    for b in range(2):
        for i in range(l):
            assert np.array_equal(out[b, i], O.ntt_fwd((src[b] >> (T * i)) & ((1 << T) - 1), Q))


def test_elementwise_vs_oracle():
    from paper_2401_16732_b200 import ring
    from paper_2401_16732_b200.ring import Domain, ModPoly

    rng = np.random.default_rng(8)
    n = 2048
    a = rng.integers(0, Q, n, dtype=np.int64)
    b = rng.integers(0, Q, n, dtype=np.int64)
    a[:5] = 0
    fa, fb = ModPoly(a, Q), ModPoly(b, Q)
    assert np.array_equal(ring.poly_add(fa, fb).coeffs, (a.astype(object) + b) % Q)
    assert np.array_equal(ring.poly_sub(fa, fb).coeffs, (a.astype(object) - b) % Q)
    assert np.array_equal(ring.poly_neg(fa).coeffs, np.where(a == 0, 0, Q - a))
    for k in (0, 1, -1, 127, -270336, 1 << 61, -(1 << 62)):
        assert np.array_equal(ring.scalar_mul(fa, k).coeffs, (a.astype(object) * (k % Q)) % Q), k
    for s in (0, 1, 5, -5, 2047, 2048, 2049, -2048, 4095, 10000, -10001):
        assert np.array_equal(ring.monomial_mul(fa, s).coeffs, O.monomial_mul(a, s, Q)), s
        # inverse pair
        assert ring.monomial_mul(ring.monomial_mul(fa, s), -s) == fa
    for step in (1, 2, 7, 100):
        g = pow(3, step, 2 * n)
        assert np.array_equal(ring.automorphism(fa, step).coeffs, O.apply_galois(a, g, Q))
    assert np.array_equal(ring.apply_galois(fa, 2 * n - 1).coeffs, O.apply_galois(a, 2 * n - 1, Q))
    with pytest.raises(ring.ParameterError):
        ring.apply_galois(ModPoly(a, Q, Domain.EVAL), 3)
    with pytest.raises(ring.ParameterError):
        ring.poly_add(fa, ModPoly(b, Q, Domain.EVAL))


def test_monomial_no_modmul():
    from paper_2401_16732_b200 import ring
    from paper_2401_16732_b200.ring import ModPoly

    with ring.track_ops() as ops:
        ring.monomial_mul(ModPoly(np.arange(2048), Q), 3)
    assert ops["modmul"] == 0


def test_widepoly_vs_eager():
    """finalize(lazy) == per-step reduced sum, incl. rotations."""
    from paper_2401_16732_b200 import ring
    from paper_2401_16732_b200.ring import ModPoly

    rng = np.random.default_rng(1)
    n = 2048
    acc = ring.WidePoly(n, Q)
    other = ring.WidePoly(n, Q)
    expect = np.zeros(n, dtype=object)
    oth = np.zeros(n, dtype=object)
    for _ in range(100):
        f = rng.integers(0, Q, n, dtype=np.int64)
        w = int(rng.integers(-255, 256))
        acc.accumulate(ModPoly(f, Q), w)
        expect = (expect + f.astype(object) * w) % Q
        g = rng.integers(0, Q, n, dtype=np.int64)
        other.accumulate_split(g & ring.LIMB_MASK, g >> ring.LIMB_BITS, 3)
        oth = (oth + g.astype(object) * 3) % Q
    acc.add_rotated(other, 77)
    expect = (expect + O.monomial_mul(oth.astype(np.int64), 77, Q).astype(object)) % Q
    assert np.array_equal(acc.finalize().coeffs, expect.astype(np.int64))
    big = ring.WidePoly(n, Q)
    with pytest.raises(ring.AccumulatorBudgetError):
        for _ in range(3):
            big.accumulate(ModPoly(np.zeros(n), Q), 1 << 31)


@pytest.mark.parametrize("n", [1024, 2048, 4096])
@pytest.mark.parametrize("with_add", [True, False])
def test_ntt_pmult_add_fused(n, with_add):
    """fhe_ntt_pmult_add (forward transform + pmult + plain_add in one launch)
    equals fhe_ntt_forward followed by fhe_ct_pmult_add."""
    import torch

    from paper_2401_16732_b200 import _native, device, params, ring

    P = params.make_params(n)
    q = P.q
    rng = np.random.default_rng(n + int(with_add))
    k = 37
    ct = torch.from_numpy(rng.integers(0, q, (k, 2, n), dtype=np.int64)).cuda()
    pt = torch.from_numpy(rng.integers(0, q, (k, n), dtype=np.int64)).cuda()
    add = torch.from_numpy(rng.integers(0, q, (k, n), dtype=np.int64)).cuda() if with_add else None
    ev = ring.ntt_rows(ct.reshape(-1, n), n, [q]).reshape(k, 2, n)
    want = torch.empty_like(ct)
    _native.call("fhe_ct_pmult_add", q, k, n, ev.data_ptr(), pt.data_ptr(), device.ptr(add), want.data_ptr(),
                 device.stream())
    got = torch.empty_like(ct)
    _native.call("fhe_ntt_pmult_add", device.native_plan(n, q), k, ct.data_ptr(), pt.data_ptr(), device.ptr(add),
                 got.data_ptr(), device.stream())
    assert torch.equal(got, want)
