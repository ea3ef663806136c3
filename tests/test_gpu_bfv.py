"""BFV ops (K3/K4/K6) and the x²+x protocol (K5) on the device vs reference goldens."""

import numpy as np
import pytest
import torch

from conftest import sha
from oracle import flash_oracle as O

pytestmark = pytest.mark.gpu

Q = 1152921486375014401


def _P():
    from paper_2401_16732_b200 import params

    return params.default_params()


def _ct(ct):
    return np.stack([ct.c0.coeffs, ct.c1.coeffs])[None]


@pytest.fixture(scope="module")
def ops_state(golden):
    """Replay make_golden.py's BFV section with our implementation (same seed)."""
    from paper_2401_16732_b200 import bfv

    P = _P()
    rng = np.random.default_rng(golden["ops"]["seed"])
    sk = bfv.keygen(P, rng)
    msg = rng.integers(0, P.p, P.n, dtype=np.int64)
    ct_d = bfv.encrypt_private(bfv.encode_direct(msg, P), sk, rng)
    ct_b = bfv.to_eval(bfv.encrypt_private(bfv.encode_batch(msg, P), sk, rng), P)
    swk = bfv.gen_switching_keys(sk, [1, 7, bfv.COLUMN_ROTATION], rng)
    hr = {s: bfv.hrot(ct_b, s, swk) for s in (1, 7, bfv.COLUMN_ROTATION)}
    pool = bfv.precompute_zero(sk, rng, 2)
    onl = bfv.encrypt_online(bfv.encode_direct(msg, P), pool.take(), P)
    k = int(rng.integers(-1000, 1000))
    return dict(P=P, sk=sk, msg=msg, ct_d=ct_d, ct_b=ct_b, swk=swk, hr=hr, onl=onl, k=k, pool=pool)


def test_keys_and_encryptions_bit_exact(golden, ops_state):
    e, s = golden["ops"], ops_state
    assert sha(s["sk"].s.coeffs) == e["h:s"]
    assert sha(s["sk"].s_eval) == e["h:s_eval"]
    assert sha(_ct(s["ct_d"])) == e["h:ct_d"]
    assert sha(_ct(s["ct_b"])) == e["h:ct_b"]
    assert sha(_ct(s["onl"])) == e["h:online"]
    for st, kk in s["swk"].keys.items():
        assert sha(np.stack([np.stack(k) for k in kk])) == e["h:keys"][str(st)]
    assert s["k"] == e["cmult_k"]


def test_homomorphic_ops_bit_exact(golden, ops_state):
    from paper_2401_16732_b200 import bfv, ring

    e, s = golden["ops"], ops_state
    P, ct_d, ct_b, msg = s["P"], s["ct_d"], s["ct_b"], s["msg"]
    assert sha(_ct(bfv.drot(ct_d, 37))) == e["h:drot37"]
    assert sha(_ct(bfv.drot(ct_d, -5))) == e["h:drot_neg5"]
    assert sha(_ct(bfv.cmult(ct_d, s["k"], P))) == e["h:cmult"]
    assert sha(_ct(bfv.hadd(ct_d, s["onl"]))) == e["h:hadd"]
    assert sha(_ct(bfv.psub(ct_d, s["onl"]))) == e["h:psub"]
    rev = msg[::-1].copy()
    assert sha(_ct(bfv.plain_add(ct_d, bfv.encode_direct(rev, P), P))) == e["h:plain_add_d"]
    assert sha(_ct(bfv.plain_add(ct_b, bfv.encode_batch(rev, P), P))) == e["h:plain_add_b"]
    assert sha(_ct(bfv.pmult(ct_b, bfv.encode_batch(rev, P), P))) == e["h:pmult"]
    assert sha(bfv.encode_batch(msg, P).poly.coeffs) == e["h:encode_batch"]
    assert sha(ring.automorphism(s["sk"].s, 3).coeffs) == e["h:automorphism3"]
    for st, c in s["hr"].items():
        assert sha(_ct(c)) == e["h:hrot"][str(st)]


def test_decrypt_and_budgets(golden, ops_state):
    from paper_2401_16732_b200 import bfv

    e, s = golden["ops"], ops_state
    P, sk, ct_d, ct_b = s["P"], s["sk"], s["ct_d"], s["ct_b"]
    assert sha(bfv.decrypt(ct_d, sk).poly.coeffs) == e["h:decrypt_d"]
    assert sha(bfv.decode_batch(bfv.decrypt(ct_b, sk), P)) == e["h:decode_b"]
    assert np.array_equal(bfv.decrypt(ct_d, sk).poly.coeffs, s["msg"])
    assert bfv.noise_budget(ct_d, sk) == e["budget_fresh"] == 37
    assert bfv.noise_budget(bfv.drot(ct_d, 37), sk) == e["budget_drot"]
    assert bfv.noise_budget(bfv.cmult(ct_d, 127, P), sk) == e["budget_cmult127"]
    assert bfv.noise_budget(s["hr"][1], sk) == e["budget_hrot1"]
    for st, c in s["hr"].items():
        assert sha(bfv.decode_batch(bfv.decrypt(c, sk), P)) == e["hrot_dec"][str(st)]


def test_op_instrumentation(ops_state):
    from paper_2401_16732_b200 import bfv, ring

    s = ops_state
    with ring.track_ops() as ops:
        bfv.drot(s["ct_d"], 9)
    assert ops["modmul"] == 0
    pool = bfv.precompute_zero(s["sk"], np.random.default_rng(0), 1)
    with ring.track_ops() as ops:
        bfv.encrypt_online(bfv.encode_direct(s["msg"], s["P"]), pool.take(), s["P"])
    assert ops["rng_draws"] == 0
    with pytest.raises(bfv.ProtocolError):
        bfv.encrypt_online(bfv.encode_direct(s["msg"], s["P"]), pool.entries[0], s["P"])
    with pytest.raises(bfv.ProtocolError):
        pool.take()


def test_encoding_errors(ops_state):
    from paper_2401_16732_b200 import bfv

    s = ops_state
    with pytest.raises(bfv.EncodingError):
        bfv.drot(s["ct_b"], 1)
    with pytest.raises(bfv.EncodingError):
        bfv.pmult(s["ct_d"], bfv.encode_batch(s["msg"], s["P"]), s["P"])
    with pytest.raises(bfv.EncodingError):
        bfv.hadd(s["ct_d"], s["ct_b"])
    with pytest.raises(bfv.EncodingError):
        bfv.hrot(s["ct_d"], 1, s["swk"])
    with pytest.raises(KeyError):
        bfv.hrot(s["ct_b"], 3, s["swk"])
    with pytest.raises(bfv.EncodingError):
        bfv.cmult(s["ct_d"], s["P"].p, s["P"])


@pytest.mark.parametrize("N", [4096, 8192, 16384])
def test_config2_hrot_sweep(golden, N):
    """Per-limb HRot at config-2 sizes with reference-generated keys (by seed)."""
    from paper_2401_16732_b200 import bfv, params, ring

    ent = golden["ntt"]["sweep"][str(N)]
    for li, e in enumerate(ent["limb"]):
        if "hrot" not in e:
            continue
        hr = e["hrot"]
        q = ent["limbs"][li]
        prm = params.RingParams(N, q, ent["p"])
        krng = np.random.default_rng(hr["key_seed"])
        sk = bfv.keygen(prm, krng)
        assert sha(sk.s.coeffs) == hr["h:s"]
        swk = bfv.gen_switching_keys(sk, hr["steps"], krng)
        c0 = krng.integers(0, q, N, dtype=np.int64)
        c1 = krng.integers(0, q, N, dtype=np.int64)
        ct = bfv.Ciphertext(ring.ModPoly(c0, q, ring.Domain.EVAL), ring.ModPoly(c1, q, ring.Domain.EVAL),
                            bfv.Encoding.BATCH, ring.Domain.EVAL)
        outs = bfv.hrot_many(ct, hr["steps"], swk)
        for st, o in zip(hr["steps"], outs):
            assert sha(np.stack([np.stack(k) for k in swk.keys[st]])) == hr["h:keys"][str(st)]
            assert sha(np.stack([o.c0.coeffs, o.c1.coeffs])) == hr["h:out"][str(st)]


@pytest.mark.parametrize("T,B", [(16, 5), (16, 1), (8, 3), (4, 2)])
def test_hrot_batch_kernel_vs_oracle(T, B):
    """K4 over a batch of ciphertexts sharing one key (the hoisted form). T=16
    (4 digits) and T=8 (8 digits, the most the column-split Acc60 MACs take)
    run the 60-bit path, T=4 (15 digits) the 128-bit MAC path; odd batches
    leave a partial 2-ciphertext chunk."""
    from paper_2401_16732_b200 import bfv

    P = _P()
    rng = np.random.default_rng(21 + T)
    sk = bfv.keygen(P, rng)
    swk = bfv.gen_switching_keys(sk, [3], rng, decomp_log=T)
    ndig = -(-Q.bit_length() // T)
    cts = rng.integers(0, Q, (B, 2, P.n), dtype=np.int64)
    t = torch.from_numpy(cts).cuda()
    dig = bfv.key_digits_rows(t[:, 1].contiguous(), P, T, ndig)
    out = bfv.keyswitch_rows(t, dig, 3, swk).cpu().numpy()
    g = O.galois_element(3, P.n)
    for b in range(B):
        o0, o1 = O.hrot(cts[b, 0], cts[b, 1], g, swk.keys[3], T, Q)
        assert np.array_equal(out[b, 0], o0) and np.array_equal(out[b, 1], o1)


def test_act2pc_end_to_end():
    """x²+x on shares: decrypt(finalize) == a² + a mod p and every message is
    bit-exact with the oracle composition."""
    from paper_2401_16732_b200 import act2pc, bfv

    P = _P()
    rng = np.random.default_rng(31)
    sk = bfv.keygen(P, rng)
    a = rng.integers(-300, 300, P.n, dtype=np.int64)
    ct_a = bfv.encrypt_private(bfv.encode_direct(a, P), sk, rng)
    pool = bfv.precompute_zero(sk, rng, 3)
    zeros = [(np.array(z.ct.c0.coeffs), np.array(z.ct.c1.coeffs)) for z in pool.entries]
    sess = act2pc.offline_prepare(1, P, rng)[0]
    assert np.array_equal(sess.r_sq, sess.r * sess.r % P.p)
    out = act2pc.run_activation(ct_a, sess, sk, pool, P)
    got = bfv.centered(bfv.decode_direct(bfv.decrypt(out, sk)), P.p)
    assert np.array_equal(got, bfv.centered(a * a + a, P.p))
    assert sess.round == act2pc.Round.DONE
    # oracle composition of the finalize ciphertext from the same zero pool:
    # ct_sq = ⟦y⟧ on zero 0, the client's round-2 reply = ⟦z⟧ on zero 2
    w = (a + sess.r) % P.p
    y = O.x2x_client(w, P.p)
    z = (2 * sess.r * w + sess.v) % P.p
    c = O.x2x_server_const(sess.r, sess.r_sq, sess.v, P.p)
    sq0 = O.add_delta(zeros[0][0], y, Q, P.p)
    back0 = O.add_delta(zeros[2][0], z, Q, P.p)
    diff0 = ((sq0.astype(object) - back0) % Q).astype(np.int64)
    exp0 = O.add_delta(diff0, c, Q, P.p)
    exp1 = ((zeros[0][1].astype(object) - zeros[2][1]) % Q).astype(np.int64)
    assert np.array_equal(out.c0.coeffs, exp0)
    assert np.array_equal(out.c1.coeffs, exp1)
    with pytest.raises(bfv.ProtocolError):
        act2pc.server_finalize(out, out, sess, P)  # session already DONE


@pytest.mark.parametrize("N,L,B,ndig,S", [(4096, 4, 5, 4, 40), (16384, 2, 3, 4, 13), (2048, 1, 2, 8, 11),
                                          (8192, 3, 1, 3, 7)])
def test_keyswitch_multi_equals_per_step(N, L, B, ndig, S):
    """fhe_keyswitch_multi (one launch for a whole rotation sweep, the digit
    rows read once) equals S separate fhe_keyswitch_apply launches bit for
    bit: several limbs, partial 2-ciphertext chunks, 3..8 digits (both MAC
    widths: 60-bit limbs take the column-split path), and S > 32 steps
    (split into launches of 32)."""
    from paper_2401_16732_b200 import _native, device, params

    p = params.find_plaintext_modulus(N)
    limbs = params.limb_primes(N, p, L)
    rng = np.random.default_rng(N + S)
    cts = torch.from_numpy(np.stack([rng.integers(0, q, (B, 2, N), dtype=np.int64) for q in limbs], 1)).cuda()
    dig = torch.from_numpy(np.stack([rng.integers(0, q, (B, ndig, N), dtype=np.int64) for q in limbs], 1)).cuda()
    keys = [torch.from_numpy(np.stack([rng.integers(0, q, (ndig, 2, N), dtype=np.int64) for q in limbs])).cuda()
            for _ in range(S)]
    gp = [int(g) for g in (2 * rng.integers(0, N, S) + 1)]
    mods = _native.u64_array(limbs)
    st = device.stream()
    want = []
    for s in range(S):
        o = torch.empty_like(cts)
        _native.call("fhe_keyswitch_apply", mods, L, B, N, cts.data_ptr(), dig.data_ptr(), keys[s].data_ptr(), ndig,
                     gp[s], o.data_ptr(), st)
        want.append(o)
    got = [torch.full_like(cts, -1) for _ in range(S)]
    import ctypes

    _native.call("fhe_keyswitch_multi", mods, L, B, N, cts.data_ptr(), dig.data_ptr(), ndig, S,
                 (ctypes.c_void_p * S)(*[k.data_ptr() for k in keys]), (ctypes.c_uint64 * S)(*gp),
                 (ctypes.c_void_p * S)(*[o.data_ptr() for o in got]), st)
    torch.cuda.synchronize()
    for s in range(S):
        assert torch.equal(got[s], want[s]), f"step {s} (gpow {gp[s]}) differs"


@pytest.mark.parametrize("n", [1024, 2048, 4096])
@pytest.mark.parametrize("domain", ["coeff", "eval"])
def test_decrypt_fused_matches_chain(n, domain, monkeypatch):
    """fhe_decrypt_fused (one launch: NTT, ·s, iNTT, + c0, round) equals the
    launch chain it replaces — messages and the folded residual maximum — on
    fresh encryptions and on arbitrary (over-noisy) rows."""
    import torch

    from paper_2401_16732_b200 import bfv, params
    from paper_2401_16732_b200.ring import Domain

    P = params.make_params(n)
    rng = np.random.default_rng(n + len(domain))
    sk = bfv.keygen(P, rng)
    fresh = bfv.precompute_zero_rows(sk, rng, 5).rows.reshape(-1, 2, n)  # encryptions of zero (COEFF)
    noise = torch.from_numpy(rng.integers(0, P.q, (7, 2, n), dtype=np.int64)).cuda()
    rows = torch.cat([fresh, noise])
    dom = Domain.EVAL if domain == "eval" else Domain.COEFF
    cts = bfv.cts_from_rows(rows.contiguous(), P.q, bfv.Encoding.DIRECT, dom)
    res = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("FLASHHE_DECRYPT_FUSED", fused)
        acc = bfv.MaxAcc()
        m = bfv.decrypt_rows_max(cts, sk, acc)
        res[fused] = (m.cpu().numpy(), acc.value())
    assert np.array_equal(res["1"][0], res["0"][0])
    assert res["1"][1] == res["0"][1]
