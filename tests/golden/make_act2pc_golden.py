"""Reference transcripts of the x²+x share protocol,
composed from the REFERENCE's own bfv / conv primitives — privinfer ships no
act2pc module, so these transcripts are how the GPU protocol is pinned:
  server r1  bfv.plain_add(⟦a⟧, encode_direct(r))                  (bfv.py:330-340, 142-147)
  client r1  w = decode_direct(decrypt(m1)) (repacked into the next layout with
             conv.channel_positions / conv.pack_vectors, conv.py:162-197);
             encrypt_online(encode_direct(w² + w·2^f)), encrypt_online(encode_batch(w))
                                                                    (bfv.py:248-263, 124-133)
  server r2  plain_add(pmult(to_eval(⟦w⟧), encode_batch(2r)), encode_batch(v))
                                                                    (bfv.py:503-512, 359-372)
  client r2  encrypt_online(encode_direct(decode_batch(decrypt(m2))))  (bfv.py:296-297, 135-139)
  finalize   plain_add(psub(ct_sq, back), encode_direct(r² − r·2^f + v))  (bfv.py:323-327)
The zero-ciphertext pool is consumed in the GPU layer protocol's order:
k_dst squares, k_dst batch messages, then k_dst round-2 replies.

Run in the build container (needs /root/reference, read-only):
    python tests/golden/make_act2pc_golden.py
Writes tests/golden/act2pc.json (sha256 of every message, little-endian int64).
"""

from __future__ import annotations

import dataclasses
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)

from privinfer import bfv, conv, params as rparams  # noqa: E402


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a, dtype=np.int64)).astype("<i8").tobytes()).hexdigest()


def rows(cts) -> np.ndarray:
    return np.stack([np.stack([c.c0.coeffs, c.c1.coeffs]) for c in cts]).astype(np.int64)


P = rparams.default_params()
p, n = P.p, P.n

# Layer cases: (name, seed, H, channels, f_w of the next conv, stride, frac bits)
CASES = [
    ("packed16_s2", 11, 16, 3, 3, 2, 0),   # 3 output cts (c_n 1) -> 8x8 next layout (c_n 20), stride 2
    ("frag64", 12, 64, 2, 3, 1, 1),        # 3 fragments per channel in and out, f = 1
    ("one_ct", 13, 32, 1, 3, 1, 0),        # one 32x32 channel (the single-ciphertext case)
    ("into_1x1", 14, 16, 4, 1, 2, 2),      # stride 2 into a 1x1 conv's layout (pad 0), f = 2
]

out = {}
for name, seed, H, c, f_next, stride, f in CASES:
    rng = np.random.default_rng(seed)
    sk = bfv.keygen(P, rng)
    src0 = dataclasses.replace(conv.layout_direct(P, H, H, 3), c_n=1)  # conv output layout
    a = rng.integers(-60, 60, (c, H, H), dtype=np.int64)
    conv_out = [bfv.encrypt_private(bfv.encode_direct(v, P), sk, rng) for v in conv.pack_vectors(a, src0, p)]
    src = dataclasses.replace(src0, stride=stride)
    ho = H // stride
    dst = conv.layout_direct(P, ho, ho, f_next)
    k_src, k_dst = len(conv_out), dst.ct_count(c)
    pool = bfv.precompute_zero(sk, rng, 3 * k_dst)
    r = rng.integers(0, p, (k_src, n), dtype=np.int64)
    v = rng.integers(0, p, (k_dst, n), dtype=np.int64)

    def repack(flat_slots):
        """values at the readable positions of `src` -> next-layout slot vectors."""
        vals = np.empty((c, ho * ho), dtype=np.int64)
        for j in range(c):
            ci, si = conv.channel_positions(src, j)
            vals[j] = flat_slots[ci, si]
        return np.stack(conv.pack_vectors(vals.reshape(c, ho, ho), dst, p))

    r_dst = repack(r)
    # server round 1
    m1 = [bfv.plain_add(ct, bfv.encode_direct(r[k], P), P) for k, ct in enumerate(conv_out)]
    # client round 1
    w = np.stack([bfv.decode_direct(bfv.decrypt(m, sk)) for m in m1])
    w_dst = repack(w)
    zs = [pool.take() for _ in range(3 * k_dst)]
    sq = [bfv.encrypt_online(bfv.encode_direct((wd * wd + wd * (1 << f)) % p, P), zs[k], P)
          for k, wd in enumerate(w_dst)]
    ctw = [bfv.encrypt_online(bfv.encode_batch(wd, P), zs[k_dst + k], P) for k, wd in enumerate(w_dst)]
    # server round 2
    m2 = [bfv.plain_add(bfv.pmult(bfv.to_eval(ctw[k], P), bfv.encode_batch(2 * r_dst[k] % p, P), P),
                        bfv.encode_batch(v[k], P), P) for k in range(k_dst)]
    # client round 2
    back = [bfv.encrypt_online(bfv.encode_direct(bfv.decode_batch(bfv.decrypt(m, sk), P), P), zs[2 * k_dst + k], P)
            for k, m in enumerate(m2)]
    # finalize
    const = (r_dst * r_dst - r_dst * (1 << f) + v) % p
    fin = [bfv.plain_add(bfv.psub(sq[k], back[k]), bfv.encode_direct(const[k], P), P) for k in range(k_dst)]
    dec = np.stack([bfv.centered(bfv.decode_direct(bfv.decrypt(x, sk)), p) for x in fin])
    a_next = a[:, ::stride, ::stride]
    want = np.stack(conv.pack_vectors(a_next * a_next + a_next * (1 << f), dst, p))
    assert np.array_equal(dec % p, want % p), name
    out[name] = {"seed": seed, "H": H, "channels": c, "f_next": f_next, "stride": stride, "frac_bits": f,
                 "k_src": k_src, "k_dst": k_dst, "h:conv_out": h(rows(conv_out)), "h:m1": h(rows(m1)),
                 "h:w": h(w), "h:sq": h(rows(sq)), "h:ct_w": h(rows(ctw)), "h:m2": h(rows(m2)),
                 "h:back": h(rows(back)), "h:out": h(rows(fin)), "h:dec": h(dec)}
    print(name, k_src, "->", k_dst, flush=True)

# The per-ciphertext SPEC calls (server_round1 ... server_finalize on one
# ciphertext, no layout change): the same composition with w used as is.
seed = 15
rng = np.random.default_rng(seed)
sk = bfv.keygen(P, rng)
a = rng.integers(-300, 300, n, dtype=np.int64)
ct = bfv.encrypt_private(bfv.encode_direct(a, P), sk, rng)
pool = bfv.precompute_zero(sk, rng, 3)
r = rng.integers(0, p, n, dtype=np.int64)
v = rng.integers(0, p, n, dtype=np.int64)
f = 3
m1 = bfv.plain_add(ct, bfv.encode_direct(r, P), P)
w = bfv.decode_direct(bfv.decrypt(m1, sk))
sq = bfv.encrypt_online(bfv.encode_direct((w * w + w * (1 << f)) % p, P), pool.take(), P)
ctw = bfv.encrypt_online(bfv.encode_batch(w, P), pool.take(), P)
m2 = bfv.plain_add(bfv.pmult(bfv.to_eval(ctw, P), bfv.encode_batch(2 * r % p, P), P), bfv.encode_batch(v, P), P)
back = bfv.encrypt_online(bfv.encode_direct(bfv.decode_batch(bfv.decrypt(m2, sk), P), P), pool.take(), P)
fin = bfv.plain_add(bfv.psub(sq, back), bfv.encode_direct((r * r - r * (1 << f) + v) % p, P), P)
dec = bfv.centered(bfv.decode_direct(bfv.decrypt(fin, sk)), p)
assert np.array_equal(dec, bfv.centered(a * a + a * (1 << f), p))
out["single_ct"] = {"seed": seed, "frac_bits": f, "h:ct": h(rows([ct])), "h:m1": h(rows([m1])),
                    "h:sq": h(rows([sq])), "h:ct_w": h(rows([ctw])), "h:m2": h(rows([m2])),
                    "h:back": h(rows([back])), "h:out": h(rows([fin])), "h:dec": h(dec)}

(OUT / "act2pc.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
print("wrote", OUT / "act2pc.json")
