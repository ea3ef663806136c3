"""Generate golden vectors by running the REFERENCE implementation itself.

Run in the build container only (needs /root/reference, read-only):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz + golden.json (committed). The reference is
imported read-only from /root/reference/pkg/src; the one known defect
(numpy-int step in bfv._galois_element under numpy 2.x) is
shimmed here, never edited in place.

Array-valued goldens are stored in full where small; large outputs are
stored as sha256 of the little-endian int64 bytes ("h:" keys).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)

from privinfer import bfv, conv, params as rparams, ring  # noqa: E402

_orig_ge = bfv._galois_element
bfv._galois_element = lambda s, n: _orig_ge(int(s), n)  # SURVEY §0.7 shim


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).astype("<i8").tobytes()).hexdigest()


def cts_array(cts) -> np.ndarray:
    return np.stack([np.stack([ct.c0.coeffs, ct.c1.coeffs]) for ct in cts]).astype(np.int64)


def make_cts(arr, domain=ring.Domain.COEFF, encoding=bfv.Encoding.DIRECT, q=None):
    return [
        bfv.Ciphertext(ring.ModPoly(a[0].copy(), q, domain), ring.ModPoly(a[1].copy(), q, domain), encoding, domain)
        for a in arr
    ]


def layout_dict(lay) -> dict:
    return {
        "n": lay.n, "height": lay.height, "width": lay.width, "pad": lay.pad, "ring": lay.ring,
        "units": lay.units, "c_n": lay.c_n, "frags": lay.frags, "frag_len": lay.frag_len,
        "halo": lay.halo, "stride": lay.stride, "w_p": lay.w_p, "tile": lay.tile,
    }


meta: dict = {"reference": REF, "generated_unix": int(time.time())}
P = rparams.default_params()
meta["params"] = P.to_dict()
meta["make_params_2048"] = rparams.make_params(2048).to_dict()

# ------------------------------------------------------------------ NTT
ntt = {}
plan = ring.get_plan(P.n, P.q)
meta["psi_default"] = plan.psi
rng = np.random.default_rng(101)
x = rng.integers(0, P.q, P.n, dtype=np.int64)
np.savez_compressed(OUT / "ntt_default.npz", x=x, fwd=plan.fwd(x), inv=plan.inv(x),
                    psi_brv=plan.psi_brv.astype(np.int64), ipsi_brv=plan.ipsi_brv.astype(np.int64))
small = ring.get_plan(16, 65537)
xs = np.random.default_rng(7).integers(0, 65537, 16, dtype=np.int64)
ntt["n16_q65537"] = {"seed": 7, "fwd": small.fwd(xs).tolist(), "inv": small.inv(xs).tolist(), "psi": small.psi}

# config-2 limb sweep: per-limb RingParams(n, q_i, p) instances
sweep = {}
for N in (4096, 8192, 16384):
    p = rparams.find_plaintext_modulus(N)
    limbs = []
    step = 2 * N * p
    qc = ((1 << 60) - 1) // step * step + 1
    while len(limbs) < 4:
        if rparams.is_prime(qc):
            limbs.append(qc)
        qc -= step
    ent = {"p": p, "limbs": limbs, "limb": []}
    for li, q in enumerate(limbs):
        pl = ring.get_plan(N, q)
        r = np.random.default_rng(1000 + 10 * N + li)
        a = r.integers(0, q, N, dtype=np.int64)
        b = r.integers(0, q, N, dtype=np.int64)
        fa = pl.fwd(a)
        e = {"seed": 1000 + 10 * N + li, "psi": pl.psi, "h:fwd": h(fa), "h:inv": h(pl.inv(a)),
             "h:pmul": h(pl.pointwise(a, b)),
             "h:add": h(ring.poly_add(ring.ModPoly(a, q), ring.ModPoly(b, q)).coeffs)}
        if li < 2:
            # hrot (T=16) on one limb ring; keys from the reference keygen
            prm = rparams.RingParams(N, q, p)
            krng = np.random.default_rng(2000 + N + li)
            sk = bfv.keygen(prm, krng)
            steps = [1, N // 4, bfv.COLUMN_ROTATION] if li == 0 else [2]
            swk = bfv.gen_switching_keys(sk, steps, krng)
            c0 = krng.integers(0, q, N, dtype=np.int64)
            c1 = krng.integers(0, q, N, dtype=np.int64)
            ct = bfv.Ciphertext(ring.ModPoly(c0, q, ring.Domain.EVAL), ring.ModPoly(c1, q, ring.Domain.EVAL),
                                bfv.Encoding.BATCH, ring.Domain.EVAL)
            e["hrot"] = {"key_seed": 2000 + N + li, "steps": steps,
                         "h:s": h(sk.s.coeffs),
                         "h:keys": {str(s): h(np.stack([np.stack(kk) for kk in swk.keys[s]])) for s in steps},
                         "h:out": {str(s): h(np.stack([(r_ := bfv.hrot(ct, s, swk)).c0.coeffs, r_.c1.coeffs]))
                                   for s in steps}}
        ent["limb"].append(e)
    sweep[str(N)] = ent
    print("sweep", N, "done", flush=True)
ntt["sweep"] = sweep
meta["ntt"] = ntt

# ------------------------------------------------------ BFV ops, n=2048
rng = np.random.default_rng(5)
sk = bfv.keygen(P, rng)
msg = rng.integers(0, P.p, P.n, dtype=np.int64)
ct_d = bfv.encrypt_private(bfv.encode_direct(msg, P), sk, rng)
ct_b = bfv.to_eval(bfv.encrypt_private(bfv.encode_batch(msg, P), sk, rng), P)
swk = bfv.gen_switching_keys(sk, [1, 7, bfv.COLUMN_ROTATION], rng)
hr = {s: bfv.hrot(ct_b, s, swk) for s in (1, 7, bfv.COLUMN_ROTATION)}
pool = bfv.precompute_zero(sk, rng, 2)
onl = bfv.encrypt_online(bfv.encode_direct(msg, P), pool.take(), P)
k = int(rng.integers(-1000, 1000))
ops = {
    "seed": 5, "cmult_k": k,
    "h:s": h(sk.s.coeffs), "h:s_eval": h(sk.s_eval),
    "h:ct_d": h(cts_array([ct_d])), "h:ct_b": h(cts_array([ct_b])),
    "h:keys": {str(s): h(np.stack([np.stack(kk) for kk in swk.keys[s]])) for s in swk.keys},
    "h:hrot": {str(s): h(cts_array([c])) for s, c in hr.items()},
    "budget_fresh": bfv.noise_budget(ct_d, sk),
    "budget_drot": bfv.noise_budget(bfv.drot(ct_d, 37), sk),
    "budget_cmult127": bfv.noise_budget(bfv.cmult(ct_d, 127, P), sk),
    "h:drot37": h(cts_array([bfv.drot(ct_d, 37)])),
    "h:drot_neg5": h(cts_array([bfv.drot(ct_d, -5)])),
    "h:cmult": h(cts_array([bfv.cmult(ct_d, k, P)])),
    "h:hadd": h(cts_array([bfv.hadd(ct_d, onl)])),
    "h:psub": h(cts_array([bfv.psub(ct_d, onl)])),
    "h:online": h(cts_array([onl])),
    "h:plain_add_d": h(cts_array([bfv.plain_add(ct_d, bfv.encode_direct(msg[::-1].copy(), P), P)])),
    "h:plain_add_b": h(cts_array([bfv.plain_add(ct_b, bfv.encode_batch(msg[::-1].copy(), P), P)])),
    "h:pmult": h(cts_array([bfv.pmult(ct_b, bfv.encode_batch(msg[::-1].copy(), P), P)])),
    "h:decrypt_d": h(bfv.decrypt(ct_d, sk).poly.coeffs),
    "h:decode_b": h(bfv.decode_batch(bfv.decrypt(ct_b, sk), P)),
    "hrot_dec": {str(s): h(bfv.decode_batch(bfv.decrypt(c, sk), P)) for s, c in hr.items()},
    "budget_hrot1": bfv.noise_budget(hr[1], sk),
    "h:encode_batch": h(bfv.encode_batch(msg, P).poly.coeffs),
    "h:automorphism3": h(ring.automorphism(sk.s, 3).coeffs),
}
meta["ops"] = ops

# ------------------------------------------------------- conv goldens
GEOMS = [
    # name, H, W, f_w, c_i, c_o, bias, full_store
    ("cfg1", 32, 32, 3, 16, 16, False, True),
    ("r20_stem", 32, 32, 3, 3, 16, False, False),
    ("r20_s2", 16, 16, 3, 32, 32, False, False),
    ("r20_s3", 8, 8, 3, 64, 64, False, False),
    ("proj1x1", 32, 32, 1, 16, 32, False, False),
    ("frag64", 64, 64, 3, 3, 8, False, False),
    ("frag64_bias", 64, 64, 3, 4, 3, True, False),
    ("packed16_bias", 16, 16, 3, 8, 8, True, False),
    ("r18_8x8_512", 8, 8, 3, 512, 4, False, False),
    ("vgg4x4", 4, 4, 3, 64, 8, False, False),
    ("stem7x7_224", 224, 224, 7, 3, 2, False, False),
]
convs = {}
for gi, (name, H, W, f_w, c_i, c_o, bias, full) in enumerate(GEOMS):
    seed = 300 + gi
    r = np.random.default_rng(seed)
    lay = conv.layout_direct(P, H, W, f_w)
    n_in = lay.ct_count(c_i)
    arr = r.integers(0, P.q, (n_in, 2, P.n), dtype=np.int64)
    wts = r.integers(-127, 128, (c_o, c_i, f_w, f_w), dtype=np.int64)
    b = r.integers(-1000, 1000, c_o, dtype=np.int64) if bias else None
    spec = conv.ConvLayerSpec(H, W, f_w, c_i, c_o, wts, bias=b)
    x = conv.PackedTensor(make_cts(arr, q=P.q), lay, c_i)
    t0 = time.time()
    y = conv.conv_proposed(x, spec, P)
    dt = time.time() - t0
    out = cts_array(y.cts)
    convs[name] = {"seed": seed, "H": H, "W": W, "f_w": f_w, "c_i": c_i, "c_o": c_o, "bias": bias,
                   "layout": layout_dict(lay), "out_layout": layout_dict(y.layout), "n_in": n_in,
                   "n_out": len(y.cts), "h:in": h(arr), "h:w": h(wts), "h:out": h(out),
                   "ref_seconds": round(dt, 3)}
    if full:
        np.savez_compressed(OUT / f"conv_{name}.npz", cts=arr, weights=wts, out=out)
    print("conv", name, dt, flush=True)
meta["conv"] = convs

# ---------------------------------------- config 1 end-to-end (real encryption)
r = np.random.default_rng(1)
sk1 = bfv.keygen(P, r)
xin = r.integers(0, 8, (16, 32, 32), dtype=np.int64)
w1 = r.integers(-127, 128, (16, 16, 3, 3), dtype=np.int64)
x1 = conv.pack_input(xin, P, 3, lambda pt: bfv.encrypt_private(pt, sk1, r))
y1 = conv.conv_proposed(x1, conv.ConvLayerSpec(32, 32, 3, 16, 16, w1), P)
dec1 = conv.unpack(y1, sk1)
np.savez_compressed(OUT / "config1_e2e.npz", s=sk1.s.coeffs, x=xin, w=w1, cts=cts_array(x1.cts),
                    out=cts_array(y1.cts), dec=dec1)
meta["config1_e2e"] = {"seed": 1, "budget_out": [bfv.noise_budget(c, sk1) for c in y1.cts[:2]]}

# avg_pool + fully_connected (config-3 tail geometry, c reduced)
r = np.random.default_rng(77)
lay8 = conv.replace(conv.layout_direct(P, 8, 8, 3), c_n=1)
arr8 = r.integers(0, P.q, (8, 2, P.n), dtype=np.int64)
x8 = conv.PackedTensor(make_cts(arr8, q=P.q), lay8, 8)
pooled = conv.avg_pool(x8, 8, P)
fcw = r.integers(-127, 128, (10, 8), dtype=np.int64)
fcb = r.integers(-100, 100, 10, dtype=np.int64)
fco = conv.fully_connected(pooled, fcw, P, bias=fcb)
meta["pool_fc"] = {"seed": 77, "h:in": h(arr8), "h:pool": h(cts_array(pooled.cts)), "h:fcw": h(fcw),
                   "h:fcb": h(fcb), "h:fc": h(cts_array(fco)), "pool_layout": layout_dict(pooled.layout)}

# small ring (n=256): packed conv with many channels per ciphertext
P256 = rparams.make_params(256)
r = np.random.default_rng(88)
lay = conv.layout_direct(P256, 4, 4, 3)
arr = r.integers(0, P256.q, (lay.ct_count(9), 2, 256), dtype=np.int64)
wts = r.integers(-127, 128, (5, 9, 3, 3), dtype=np.int64)
y = conv.conv_proposed(conv.PackedTensor(make_cts(arr, q=P256.q), lay, 9), conv.ConvLayerSpec(4, 4, 3, 9, 5, wts), P256)
meta["conv_n256"] = {"seed": 88, "params": P256.to_dict(), "layout": layout_dict(lay), "h:in": h(arr),
                     "h:w": h(wts), "h:out": h(cts_array(y.cts))}

# conventional conv, config-1 geometry (T=4 keys as the reference engine uses)
r = np.random.default_rng(9)
skc = bfv.keygen(P, r)
xc = r.integers(0, 8, (4, 16, 16), dtype=np.int64)
wc = r.integers(-127, 128, (4, 4, 3, 3), dtype=np.int64)
specc = conv.ConvLayerSpec(16, 16, 3, 4, 4, wc)
swc = bfv.gen_switching_keys(skc, conv.conventional_steps(specc, P), r, decomp_log=conv.CONV_DECOMP_LOG)
xcb = conv.pack_input(xc, P, 3, lambda pt: bfv.encrypt_private(pt, skc, r), batch=True)
t0 = time.time()
yc = conv.conv_conventional(xcb, specc, swc, P)
meta["conv_conventional"] = {"seed": 9, "steps": conv.conventional_steps(specc, P),
                             "h:in": h(cts_array(xcb.cts)), "h:out": h(cts_array(yc.cts)),
                             "dec": conv.unpack(yc, skc).tolist(), "ref_seconds": round(time.time() - t0, 2)}

# fragmented conventional conv (needs the harness-side _galois_element shim above), with bias
r = np.random.default_rng(10)
skf = bfv.keygen(P, r)
xf = r.integers(0, 8, (2, 32, 32), dtype=np.int64)
wf = r.integers(-127, 128, (3, 2, 3, 3), dtype=np.int64)
bf = np.array([5, 0, -7], dtype=np.int64)
specf = conv.ConvLayerSpec(32, 32, 3, 2, 3, wf, bias=bf)
swf = bfv.gen_switching_keys(skf, conv.conventional_steps(specf, P), r, decomp_log=conv.CONV_DECOMP_LOG)
xfb = conv.pack_input(xf, P, 3, lambda pt: bfv.encrypt_private(pt, skf, r), batch=True)
t0 = time.time()
yf = conv.conv_conventional(xfb, specf, swf, P)
meta["conv_conventional_frag"] = {"seed": 10, "steps": conv.conventional_steps(specf, P),
                                  "h:in": h(cts_array(xfb.cts)), "h:out": h(cts_array(yf.cts)),
                                  "dec": conv.unpack(yf, skf).tolist(), "ref_seconds": round(time.time() - t0, 2)}

(OUT / "golden.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
print("wrote", OUT / "golden.json")
