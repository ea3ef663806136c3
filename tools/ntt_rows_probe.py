"""n = 2048 row NTT and fused-decryption throughput at several row counts (development probe)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2401_16732_b200 import _native, bfv, device, params, ring  # noqa: E402

P = params.default_params()
n = P.n
rng = np.random.default_rng(1)
sk = bfv.keygen(P, rng)


def t_events(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


for rows in (512, 2048, 10240):
    x = torch.from_numpy(rng.integers(0, P.q, (rows, n), dtype=np.int64)).cuda()
    out = torch.empty_like(x)
    us = t_events(lambda: ring.ntt_rows(x, n, [P.q], out=out))
    bf = rows * (n // 2) * 11 / (us * 1e-6)
    print(f"ntt fwd rows {rows:6d}: {us:8.1f} us  {bf / 1e12:.3f} T butterflies/s ({bf / 0.862e12:.0%} of 0.862)")
for k in (192, 5120):
    cts = bfv.cts_from_rows(torch.from_numpy(rng.integers(0, P.q, (k, 2, n), dtype=np.int64)).cuda(), P.q,
                            bfv.Encoding.DIRECT, ring.Domain.COEFF)
    acc = bfv.MaxAcc()
    us = t_events(lambda: bfv.decrypt_rows_max(cts, sk, acc))
    bf = k * 2 * (n // 2) * 11 / (us * 1e-6)
    print(f"decrypt fused k {k:6d}: {us:8.1f} us  {bf / 1e12:.3f} T butterflies/s (2 transforms per ct)")
