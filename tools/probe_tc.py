"""Per-layer timing of K1 (tensor-core or integer path) on a config's conv layers.

Development probe (not part of the product or the bench contract):
    python tools/probe_tc.py [--workload config4] [--layer NAME] [--once]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import conv, params, stacks  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default=None, help="only this config-4 layer name")
    ap.add_argument("--once", action="store_true", help="one launch per layer (for ncu)")
    ap.add_argument("--workload", default="config4")
    ap.add_argument("--int", action="store_true", help="also time the integer-pipe kernel")
    args = ap.parse_args()
    P = params.default_params()
    rng = np.random.default_rng(0)
    seen = set()
    for l in stacks.conv_layers(stacks.CONFIGS[args.workload]()):
        key = (l.H, l.f_w, l.c_i, l.c_o)
        if key in seen or (args.layer and l.name != args.layer):
            continue
        seen.add(key)
        lay = conv.layout_direct(P, l.H, l.W, l.f_w)
        w = rng.integers(-127, 128, (l.c_o, l.c_i, l.f_w, l.f_w))
        plan = conv.conv_plan(conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, w), lay, P)
        inp = torch.from_numpy(rng.integers(0, P.q, (lay.ct_count(l.c_i), 2, P.n))).cuda()
        out = torch.empty((plan.n_out, 2, P.n), dtype=torch.int64, device="cuda")
        plan.run(inp, out)
        torch.cuda.synchronize()
        if args.once:
            print(l.name, "ran once via", plan.path)
            continue
        for path in ([plan.path, "int"] if args.int and plan.path == "tc" else [plan.path]):
            plan.run(inp, out, path=path)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(10):
                    plan.run(inp, out, path=path)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 10 * 1e3
            macs = plan.n_out * plan.K * 2 * P.n
            print(f"{l.name:10s} {path:3s} {us:8.1f} us  {macs / us / 1e6:7.1f} TMAC60/s  "
                  f"{16 * macs / us / 1e6:8.1f} int8 TOPS-equiv  {macs / 1e6:8.1f} M MAC60")


if __name__ == "__main__":
    main()
