"""Event-timed batched NTT fwd/inv of the bench's config-2 shape (L2 flushed). Development tool."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, device, params  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
L, B = 4, 64
p = params.find_plaintext_modulus(N)
limbs = params.limb_primes(N, p, L)
rng = np.random.default_rng(2)
x = np.stack([rng.integers(0, q, (B, 2, N), dtype=np.int64) for q in limbs], axis=1)
t = torch.from_numpy(x).cuda()
out = torch.empty_like(t)
flush = torch.empty(2**25, dtype=torch.int64, device="cuda")
plans = device.plan_array(N, limbs)
res = {}
for fn in ("fhe_ntt_forward", "fhe_ntt_inverse"):
    ts = []
    for i in range(13):
        flush.fill_(i)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _native.call(fn, plans, L, B, 2, t.data_ptr(), out.data_ptr(), device.stream())
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    res[fn[8:]] = round(float(np.median(ts)), 1)
print(N, res)
