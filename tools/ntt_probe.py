"""NTT timing at the reference's default n = 2048 (and config-2 sizes):
forward / inverse over `rows` rows, CUDA-graph timed (development probe; run
under ncu with --once for a capture of one launch each).

    python tools/ntt_probe.py [--n 2048] [--rows 512] [--once]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, device, params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2048)
    ap.add_argument("--rows", type=int, default=512)
    ap.add_argument("--once", action="store_true")
    args = ap.parse_args()
    n, rows = args.n, args.rows
    q = params.default_params().q if n == 2048 else params.limb_primes(n, params.find_plaintext_modulus(n), 1)[0]
    plans = device.plan_array(n, [q])
    x = torch.from_numpy(np.random.default_rng(1).integers(0, q, (rows, n), dtype=np.int64)).cuda()
    y = torch.empty_like(x)
    for name in ("fhe_ntt_forward", "fhe_ntt_inverse"):
        fn = lambda: _native.call(name, plans, 1, rows, 1, x.data_ptr(), y.data_ptr(), device.stream())  # noqa: E731
        fn()
        torch.cuda.synchronize()
        if args.once:
            continue
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
            for _ in range(20):
                fn()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 20 * 1e3)
        us = sorted(ts)[2]
        bfly = rows * (n // 2) * (n.bit_length() - 1)
        print(f"{name:16s} n={n} rows={rows}: {us:7.2f} us  {bfly / us / 1e6:7.3f} T butterflies/s  "
              f"{rows * n * 16 / us / 1e3:7.1f} GB/s")


if __name__ == "__main__":
    main()
