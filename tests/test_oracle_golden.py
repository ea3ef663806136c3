"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py). CPU only — no GPU needed."""

import numpy as np
import pytest

from conftest import load_npz, sha
from oracle import flash_oracle as O

Q = 1152921486375014401
P = 270337
N = 2048


def test_params_pinned(golden):
    from paper_2401_16732_b200 import params

    assert golden["make_params_2048"] == golden["params"]
    assert params.default_params().to_dict() == golden["params"]
    assert params.make_params(2048).to_dict() == golden["params"]


def test_ntt_default_tables_and_transforms(golden):
    g = load_npz("ntt_default.npz")
    assert O.find_root(N, Q) == golden["psi_default"]
    psi_brv, ipsi_brv, _ = O.ntt_tables(N, Q)
    assert np.array_equal(np.array(psi_brv, dtype=np.int64), g["psi_brv"])
    assert np.array_equal(np.array(ipsi_brv, dtype=np.int64), g["ipsi_brv"])
    assert np.array_equal(O.ntt_fwd(g["x"], Q), g["fwd"])
    assert np.array_equal(O.ntt_inv(g["x"], Q), g["inv"])


def test_ntt_small_kat(golden):
    e = golden["ntt"]["n16_q65537"]
    x = np.random.default_rng(e["seed"]).integers(0, 65537, 16, dtype=np.int64)
    assert O.ntt_fwd(x, 65537).tolist() == e["fwd"]
    assert O.ntt_inv(x, 65537).tolist() == e["inv"]
    # delta -> all ones; round trip
    d = np.zeros(16, dtype=np.int64)
    d[0] = 1
    assert O.ntt_fwd(d, 65537).tolist() == [1] * 16
    assert np.array_equal(O.ntt_inv(O.ntt_fwd(x, 65537), 65537), x)


@pytest.mark.parametrize("N_", ["4096", "8192"])
def test_ntt_sweep_limbs(golden, N_):
    ent = golden["ntt"]["sweep"][N_]
    n = int(N_)
    for q, e in zip(ent["limbs"], ent["limb"]):
        r = np.random.default_rng(e["seed"])
        a = r.integers(0, q, n, dtype=np.int64)
        b = r.integers(0, q, n, dtype=np.int64)
        assert O.find_root(n, q) == e["psi"]
        assert sha(O.ntt_fwd(a, q)) == e["h:fwd"]
        assert sha(O.ntt_inv(a, q)) == e["h:inv"]
        assert sha(O.pointwise(a, b, q)) == e["h:pmul"]


def test_limb_primes_match_survey(golden):
    from paper_2401_16732_b200 import params

    for N_, ent in golden["ntt"]["sweep"].items():
        assert params.limb_primes(int(N_), ent["p"], 4) == ent["limbs"]
        assert params.find_plaintext_modulus(int(N_)) == ent["p"]


def test_spec_ring_kats():
    # SPEC.md:61-63, 70-72, 78-81 (n=4, q=17; n=8)
    assert O.negacyclic_schoolbook([1, 1, 0, 0], [1, 1, 0, 0], 17).tolist() == [1, 2, 1, 0]
    assert O.negacyclic_schoolbook([0, 0, 0, 1], [0, 1, 0, 0], 17).tolist() == [16, 0, 0, 0]
    assert O.monomial_mul(np.array([1, 2, 3, 4]), 1, 17).tolist() == [2, 3, 4, 16]
    x = np.zeros(8, dtype=np.int64)
    x[1] = 1
    assert O.apply_galois(x, 3, 17).tolist() == [0, 0, 0, 1, 0, 0, 0, 0]


def test_oracle_ntt_product_vs_schoolbook():
    rng = np.random.default_rng(3)
    q = 12289  # ≡ 1 mod 64
    for _ in range(5):
        f = rng.integers(0, q, 32)
        g = rng.integers(0, q, 32)
        via = O.ntt_inv(O.pointwise(O.ntt_fwd(f, q), O.ntt_fwd(g, q), q), q)
        assert np.array_equal(via, O.negacyclic_schoolbook(f, g, q))


def _conv_case(golden, name):
    g = golden["conv"][name]
    r = np.random.default_rng(g["seed"])
    arr = r.integers(0, Q, (g["n_in"], 2, N), dtype=np.int64)
    w = r.integers(-127, 128, (g["c_o"], g["c_i"], g["f_w"], g["f_w"]), dtype=np.int64)
    b = r.integers(-1000, 1000, g["c_o"], dtype=np.int64) if g["bias"] else None
    return g, arr, w, b


def _bias_masks(lay):
    """Slots of conv._bias_plaintext (conv.py:414-424), per fragment."""
    ys = lay["pad"] + np.arange(lay["height"])
    xs = lay["pad"] + np.arange(lay["width"])
    tp = (ys[:, None] * lay["w_p"] + xs[None, :]).ravel()
    masks = np.zeros((lay["frags"], lay["n"]), dtype=np.uint8)
    for f in range(lay["frags"]):
        if lay["frags"] > 1:
            sel = tp[tp // lay["frag_len"] == f]
            masks[f, lay["halo"] + sel - f * lay["frag_len"]] = 1
        else:
            masks[f, tp] = 1
    return masks


@pytest.mark.parametrize(
    "name",
    ["cfg1", "r20_stem", "r20_s2", "proj1x1", "frag64", "frag64_bias", "packed16_bias", "vgg4x4", "r18_8x8_512"],
)
def test_oracle_conv_vs_reference(golden, name):
    g, arr, w, b = _conv_case(golden, name)
    assert sha(arr) == g["h:in"] and sha(w) == g["h:w"]
    out = O.conv_proposed(arr, w.reshape(g["c_o"], g["c_i"], -1), g["layout"], Q)
    if b is not None:
        out = O.add_bias(out, b, _bias_masks(g["out_layout"]), Q // P, P, Q)
    assert sha(out) == g["h:out"]


def test_oracle_conv_cfg1_full():
    d = load_npz("conv_cfg1.npz")
    lay = {"n": N, "w_p": 34, "pad": 1, "tile": 34 * 34, "c_n": 1, "frags": 1}
    out = O.conv_proposed(d["cts"], d["weights"].reshape(16, 16, 9), lay, Q)
    assert np.array_equal(out, d["out"])


def test_oracle_pool_fc(golden):
    g = golden["pool_fc"]
    r = np.random.default_rng(g["seed"])
    arr = r.integers(0, Q, (8, 2, N), dtype=np.int64)
    assert sha(arr) == g["h:in"]
    pooled = O.avg_pool(arr, 8, 10, Q)
    assert sha(pooled) == g["h:pool"]
    fcw = r.integers(-127, 128, (10, 8), dtype=np.int64)
    fcb = r.integers(-100, 100, 10, dtype=np.int64)
    # after the k=8 pool with stride marker, channel j's only readable slot is tile pos (1,1)
    slots = np.full(8, 1 * 10 + 1)
    out = O.fully_connected(pooled, fcw, np.arange(8), slots, Q)
    mask = np.zeros((1, N), dtype=np.uint8)
    mask[0, 0] = 1
    out = O.add_bias(out, fcb, mask, Q // P, P, Q)
    assert sha(out) == g["h:fc"]


def test_oracle_keys_and_hrot_default(golden):
    e = golden["ops"]
    rng = np.random.default_rng(e["seed"])
    s = O.keygen(N, Q, rng)
    assert sha(s) == e["h:s"]
    msg = rng.integers(0, P, N, dtype=np.int64)
    O.encrypt_private(msg, s, N, Q, P, 20, rng)          # ct_d (advances rng as the reference)
    O.encrypt_private(np.zeros(N), s, N, Q, P, 20, rng)  # ct_b draws (payload irrelevant here)
    keys = O.gen_switching_keys(s, [1, 7, -1], N, Q, 20, 16, rng)
    for st, kk in keys.items():
        assert sha(np.stack([np.stack(k) for k in kk])) == e["h:keys"][str(st)]


def test_oracle_hrot_sweep(golden):
    ent = golden["ntt"]["sweep"]["4096"]
    n, q = 4096, ent["limbs"][0]
    hr = ent["limb"][0]["hrot"]
    krng = np.random.default_rng(hr["key_seed"])
    s = O.keygen(n, q, krng)
    assert sha(s) == hr["h:s"]
    keys = O.gen_switching_keys(s, hr["steps"], n, q, 20, 16, krng)
    c0 = krng.integers(0, q, n, dtype=np.int64)
    c1 = krng.integers(0, q, n, dtype=np.int64)
    for st in hr["steps"]:
        assert sha(np.stack([np.stack(k) for k in keys[st]])) == hr["h:keys"][str(st)]
        o0, o1 = O.hrot(c0, c1, O.galois_element(st, n), keys[st], 16, q)
        assert sha(np.stack([o0, o1])) == hr["h:out"][str(st)]


def test_oracle_config1_decrypt():
    d = load_npz("config1_e2e.npz")
    out = d["out"]
    dec = []
    for u in range(2):
        ph = O.decrypt_phase(out[u, 0], out[u, 1], d["s"], Q)
        m, _ = O.decrypt_round(ph, Q, P)
        dec.append(m)
    # readable slots of channel j: tile rows 1..32, cols 1..32 of W_p = 34
    ys = 1 + np.arange(32)
    tp = (ys[:, None] * 34 + ys[None, :]).ravel()
    for u in range(2):
        v = dec[u][tp] % P
        v = v - (v > P // 2) * P
        assert np.array_equal(v.reshape(32, 32), d["dec"][u])


def test_x2x_algebra():
    rng = np.random.default_rng(0)
    a = rng.integers(0, P, 4096)
    r = rng.integers(0, P, 4096)
    v = rng.integers(0, P, 4096)
    w = (a + r) % P
    ct1 = O.x2x_client(w, P)
    ct2 = (2 * a * r + 2 * r * r + v) % P
    c = O.x2x_server_const(r, r * r % P, v, P)
    assert np.array_equal((ct1 - ct2 + c) % P, (a * a + a) % P)


@pytest.mark.parametrize("name", ["cfg1", "r20_stem", "r20_s2", "r20_s3", "proj1x1", "frag64", "r18_8x8_512",
                                  "vgg4x4", "stem7x7_224"])
def test_c_oracle_matches_reference_conv(golden, name):
    """oracle/conv_oracle.c (the CPU baseline and the --impl reference arm)
    reproduces the reference's conv_proposed outputs (golden sha256)."""
    from oracle import c_oracle

    g = golden["conv"][name]
    r = np.random.default_rng(g["seed"])
    arr = r.integers(0, Q, (g["n_in"], 2, N), dtype=np.int64)
    w = r.integers(-127, 128, (g["c_o"], g["c_i"], g["f_w"], g["f_w"]), dtype=np.int64)
    src, step, fstride = c_oracle.conv_terms(g["layout"], g["c_i"], g["f_w"])
    out = c_oracle.conv(Q, N, arr, w.reshape(g["c_o"], -1), src, step, g["layout"]["frags"], fstride, threads=4)
    assert out.shape[0] == g["n_out"]
    assert sha(out) == g["h:out"]
    # a strided unit selection lands each unit in its own row
    sel = np.arange(g["n_out"])[::-3][:5]
    assert np.array_equal(c_oracle.conv(Q, N, arr, w.reshape(g["c_o"], -1), src, step, g["layout"]["frags"],
                                        fstride, threads=2, units=sel), out[sel])
