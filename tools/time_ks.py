"""Event-timed hoisted key switch of the bench's config-2 shape (13 steps, L2 flushed). Development tool."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, device, params  # noqa: E402

N, L, B, T, l = 16384, 4, 64, 16, 4
p = params.find_plaintext_modulus(N)
limbs = params.limb_primes(N, p, L)
rng = np.random.default_rng(2)
t = torch.from_numpy(np.stack([rng.integers(0, q, (B, 2, N), dtype=np.int64) for q in limbs], axis=1)).cuda()
dig = torch.from_numpy(np.stack([rng.integers(0, q, (B, l, N), dtype=np.int64) for q in limbs], axis=1)).cuda()
rsteps = [1 << i for i in range(N.bit_length() - 2)]
keys = {s: torch.from_numpy(np.stack([rng.integers(0, q, (l, 2, N), dtype=np.int64) for q in limbs])).cuda()
        for s in rsteps}
rot = torch.empty((B, L, 2, N), dtype=torch.int64, device="cuda")
mods = _native.u64_array(limbs)
flush = torch.empty(2**25, dtype=torch.int64, device="cuda")
st = device.stream()
ts = []
for i in range(8):
    flush.fill_(i)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in rsteps:
        _native.call("fhe_keyswitch_apply", mods, L, B, N, t.data_ptr(), dig.data_ptr(), keys[s].data_ptr(), l,
                     pow(3, s, 2 * N), rot.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    if i >= 2:
        ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
alg = len(rsteps) * (B * L * 8 * N * (1 + l + 2) + L * 2 * l * 8 * N)
print(f"keyswitch 13 steps: {ms:.3f} ms, {alg / ms / 1e6:.1f} GB/s, checksum {int(rot.sum().item()) & 0xffffffff}")
