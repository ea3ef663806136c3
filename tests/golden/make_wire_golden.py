"""Wire frames produced by the REFERENCE's bfv.ct_to_bytes (bfv.py:530-535)
for ciphertexts made by its own keygen / encrypt_private / to_eval / hadd.

Run in the build container (needs /root/reference, read-only):
    python tests/golden/make_wire_golden.py
Writes tests/golden/wire.npz (the ciphertext arrays and seeds) and wire.json
(sha256 and length of every frame; the concatenated unseeded frames of a
batch). tests/test_host.py rebuilds the same ciphertexts from the arrays and
checks the package's frames and parser against them (CPU only).
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)

from privinfer import bfv, params as rparams  # noqa: E402

P = rparams.default_params()
rng = np.random.default_rng(21)
sk = bfv.keygen(P, rng)
m = rng.integers(0, P.p, P.n, dtype=np.int64)
fresh = bfv.encrypt_private(bfv.encode_direct(m, P), sk, rng)                       # fresh: seed-compressible
batch_eval = bfv.to_eval(bfv.encrypt_private(bfv.encode_batch(m, P), sk, rng), P)   # EVAL: never seeded
summed = bfv.hadd(fresh, bfv.encrypt_private(bfv.encode_direct(m[::-1].copy(), P), sk, rng))  # not fresh

cases = {"fresh": fresh, "batch_eval": batch_eval, "summed": summed}
meta = {}
arrays = {}
for name, ct in cases.items():
    arrays[f"{name}_c0"] = ct.c0.coeffs.astype(np.int64)
    arrays[f"{name}_c1"] = ct.c1.coeffs.astype(np.int64)
    seed = ct.seed if ct.seed is not None else b""
    arrays[f"{name}_seed"] = np.frombuffer(seed, dtype=np.uint8).copy()
    frames = {"seeded": bfv.ct_to_bytes(ct), "full": bfv.ct_to_bytes(ct, seed_compress=False)}
    meta[name] = {"encoding": ct.encoding.value, "domain": int(ct.domain.value != bfv.Domain.COEFF.value),
                  "fresh": bool(ct.fresh),
                  **{f"h:{k}": hashlib.sha256(v).hexdigest() for k, v in frames.items()},
                  **{f"len:{k}": len(v) for k, v in frames.items()},
                  "head": list(frames["seeded"][:3])}
    # the reference parser's view of its own frame
    back = bfv.ct_from_bytes(frames["seeded"], P)
    assert np.array_equal(back.c0.coeffs, ct.c0.coeffs) and np.array_equal(back.c1.coeffs, ct.c1.coeffs)
blob = b"".join(bfv.ct_to_bytes(c, seed_compress=False) for c in cases.values())
meta["batch"] = {"order": list(cases), "h": hashlib.sha256(blob).hexdigest(), "len": len(blob)}
meta["wire_size"] = {"seeded": bfv.ct_wire_size(P, True), "full": bfv.ct_wire_size(P, False)}
np.savez_compressed(OUT / "wire.npz", **arrays)
(OUT / "wire.json").write_text(json.dumps(meta, indent=1, sort_keys=True) + "\n")
print(json.dumps(meta["batch"]), meta["wire_size"])
