"""One batched forward NTT of the bench's config-2 shape (for ncu). Development tool."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, device, params  # noqa: E402

N = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
L, B = 4, 64
p = params.find_plaintext_modulus(N)
limbs = params.limb_primes(N, p, L)
rng = np.random.default_rng(2)
x = np.stack([rng.integers(0, q, (B, 2, N), dtype=np.int64) for q in limbs], axis=1)
t = torch.from_numpy(x).cuda()
out = torch.empty_like(t)
plans = device.plan_array(N, limbs)
fn = "fhe_ntt_inverse" if len(sys.argv) > 1 and sys.argv[1] == "inv" else "fhe_ntt_forward"
for _ in range(2):
    _native.call(fn, plans, L, B, 2, t.data_ptr(), out.data_ptr(), device.stream())
torch.cuda.synchronize()
print("ok")
