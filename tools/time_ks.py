"""Event-timed hoisted key switch of the bench's config-2 shape (N=16384,
4 limbs, 64 ciphertexts, 13 steps, L2 flushed): the 13 per-step launches
(fhe_keyswitch_apply) against the one multi-step launch
(fhe_keyswitch_multi). Development tool; --once runs each form once (ncu).

    python tools/time_ks.py [--once]
"""

import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, device, params  # noqa: E402

once = "--once" in sys.argv
N, L, B, T, l = 16384, 4, 64, 16, 4
p = params.find_plaintext_modulus(N)
limbs = params.limb_primes(N, p, L)
rng = np.random.default_rng(2)
t = torch.from_numpy(np.stack([rng.integers(0, q, (B, 2, N), dtype=np.int64) for q in limbs], axis=1)).cuda()
dig = torch.from_numpy(np.stack([rng.integers(0, q, (B, l, N), dtype=np.int64) for q in limbs], axis=1)).cuda()
rsteps = [1 << i for i in range(N.bit_length() - 2)]
S = len(rsteps)
keys = {s: torch.from_numpy(np.stack([rng.integers(0, q, (l, 2, N), dtype=np.int64) for q in limbs])).cuda()
        for s in rsteps}
rot = torch.empty((B, L, 2, N), dtype=torch.int64, device="cuda")
rots = [torch.empty((B, L, 2, N), dtype=torch.int64, device="cuda") for _ in rsteps]
mods = _native.u64_array(limbs)
flush = torch.empty(2**25, dtype=torch.int64, device="cuda")
st = device.stream()
kptr = (ctypes.c_void_p * S)(*[keys[s].data_ptr() for s in rsteps])
gp = (ctypes.c_uint64 * S)(*[pow(3, s, 2 * N) for s in rsteps])
optr = (ctypes.c_void_p * S)(*[r.data_ptr() for r in rots])


def per_step():
    for s in rsteps:
        _native.call("fhe_keyswitch_apply", mods, L, B, N, t.data_ptr(), dig.data_ptr(), keys[s].data_ptr(), l,
                     pow(3, s, 2 * N), rot.data_ptr(), st)


def multi():
    _native.call("fhe_keyswitch_multi", mods, L, B, N, t.data_ptr(), dig.data_ptr(), l, S, kptr, gp, optr, st)


for name, fn in (("per-step", per_step), ("multi", multi)):
    if once:
        fn()
        torch.cuda.synchronize()
        continue
    ts = []
    for i in range(8):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    row = 8 * N
    alg = S * (B * L * row * 4 + L * 2 * l * row)
    moved = B * L * row * (1 + l) + S * L * 2 * l * row + S * B * L * 2 * row
    print(f"{name:9s} 13 steps: {ms:.3f} ms  §8d {alg / ms / 1e6:7.1f} GB/s  moved-min {moved / ms / 1e6:7.1f} GB/s")
