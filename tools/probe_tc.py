"""Per-kernel timing of the K1-TC path (prep vs MMA kernel) on config-4 layers.

Development probe (not part of the product or the bench contract):
    python tools/probe_tc.py
"""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, conv, device, params, stacks  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    P = params.default_params()
    rng = np.random.default_rng(0)
    seen = set()
    for l in stacks.conv_layers(stacks.config4()):
        key = (l.H, l.f_w, l.c_i, l.c_o)
        if key in seen:
            continue
        seen.add(key)
        lay = conv.layout_direct(P, l.H, l.W, l.f_w)
        w = rng.integers(-127, 128, (l.c_o, l.c_i, l.f_w, l.f_w))
        spec = conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, w)
        plan = conv.conv_plan(spec, lay, P)
        inp = torch.from_numpy(rng.integers(0, P.q, (lay.ct_count(l.c_i), 2, P.n))).cuda()
        out = torch.empty((plan.n_out, 2, P.n), dtype=torch.int64, device="cuda")
        if plan.tc is None:
            plan.run(inp, out)
            torch.cuda.synchronize()
            e0, e1 = ev(), ev()
            e0.record()
            for _ in range(10):
                plan.run(inp, out)
            e1.record()
            torch.cuda.synchronize()
            print(f"{l.name:10s} int  total {e0.elapsed_time(e1) / 10 * 1e3:8.1f} us")
            continue
        tc = plan.tc
        st = device.stream()

        def prep():
            _native.call("fhe_conv_tc_prep", tc.q, tc.n, inp.data_ptr(), tc.c_i, tc.frags, tc.fstride,
                         tc.chan.data_ptr(), tc.h, tc.X.data_ptr(), st)

        def mma():
            _native.call("fhe_conv_tc", tc.q, tc.n, tc.X.data_ptr(), tc.c_i, tc.frags, tc.h, tc.w.data_ptr(),
                         tc.c_o, tc.taps, tc.n_tile, tc.steps, None, None, out.data_ptr(), st)

        prep()
        mma()
        torch.cuda.synchronize()
        res = []
        for fn in (prep, mma):
            e0, e1 = ev(), ev()
            e0.record()
            for _ in range(10):
                fn()
            e1.record()
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / 10 * 1e3)
        macs = plan.n_out * plan.K * 2 * P.n
        print(f"{l.name:10s} tc N={tc.n_tile:3d} prep {res[0]:7.1f} us  mma {res[1]:7.1f} us  "
              f"X {tc.X.numel() / 1e6:6.1f} MB  {macs / res[1] / 1e6:7.1f} TMAC60/s(mma)")


if __name__ == "__main__":
    main()
