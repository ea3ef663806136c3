"""Host cost of one drop-in call (conv.conv_proposed / ConvPlan.run) against
its device time, for small config layers (development probe).

    python tools/host_overhead.py [--workload config5] [--calls 200]
"""

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import bfv, conv, params, stacks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config5")
    ap.add_argument("--calls", type=int, default=200)
    args = ap.parse_args()
    P = params.default_params()
    rng = np.random.default_rng(0)
    seen = set()
    for l in stacks.conv_layers(stacks.CONFIGS[args.workload]()):
        key = (l.H, l.f_w, l.c_i, l.c_o)
        if key in seen:
            continue
        seen.add(key)
        lay = conv.layout_direct(P, l.H, l.W, l.f_w)
        spec = conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, rng.integers(-127, 128, (l.c_o, l.c_i, l.f_w, l.f_w)))
        plan = conv.conv_plan(spec, lay, P)
        inp = torch.from_numpy(rng.integers(0, P.q, (lay.ct_count(l.c_i), 2, P.n))).cuda()
        out = torch.empty((plan.n_out, 2, P.n), dtype=torch.int64, device="cuda")
        x = conv.PackedTensor(bfv.cts_from_rows(inp, P.q, bfv.Encoding.DIRECT, bfv.Domain.COEFF), lay, l.c_i)
        for _ in range(5):
            plan.run(inp, out)
            conv.conv_proposed(x, spec, P, out=out)
        torch.cuda.synchronize()
        res = {}
        for name, fn in (("plan.run", lambda: plan.run(inp, out)),
                         ("conv_proposed", lambda: conv.conv_proposed(x, spec, P, out=out))):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0.record()
            for _ in range(args.calls):
                fn()
            e1.record()
            host = (time.perf_counter() - t0) / args.calls * 1e6
            torch.cuda.synchronize()
            res[name] = (host, e0.elapsed_time(e1) / args.calls * 1e3)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20):
                plan.run(inp, out)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        dev = e0.elapsed_time(e1) / 20 * 1e3
        print(f"{l.name:9s} device (graph) {dev:6.1f} us | plan.run host {res['plan.run'][0]:6.1f} us, "
              f"stream {res['plan.run'][1]:6.1f} us | conv_proposed host {res['conv_proposed'][0]:6.1f} us, "
              f"stream {res['conv_proposed'][1]:6.1f} us")


if __name__ == "__main__":
    main()
