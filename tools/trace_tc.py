"""Timeline of the K1-TC pipeline on one config-4 layer (CTA 0), via fhe_debug_trace.

Development probe:  python tools/trace_tc.py [--layer s4b1c2]

Needs a trace build of the library (the default build keeps only the per-CTA
start/end stamps):  python tools/build_probe.py trace -DFHE_TC_TRACE=1, then run
with FLASHHE_LIB=tools/_lib_trace.so.
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, conv, params, stacks  # noqa: E402

KINDS = ["mma_full_ok", "mma_commit", "relayout_start", "relayout_warp_done", "load_issue", "epi_full_ok", "epi_done", "grid_barrier_done"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", default="s4b1c2")
    args = ap.parse_args()
    P = params.default_params()
    rng = np.random.default_rng(0)
    l = [x for x in stacks.conv_layers(stacks.config4()) if x.name == args.layer][0]
    lay = conv.layout_direct(P, l.H, l.W, l.f_w)
    w = rng.integers(-127, 128, (l.c_o, l.c_i, l.f_w, l.f_w))
    plan = conv.conv_plan(conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, w), lay, P)
    inp = torch.from_numpy(rng.integers(0, P.q, (lay.ct_count(l.c_i), 2, P.n))).cuda()
    out = torch.empty((plan.n_out, 2, P.n), dtype=torch.int64, device="cuda")
    plan.run(inp, out)
    buf = torch.zeros(25 * 4096, dtype=torch.int64, device="cuda")  # (the trace area fhe_debug_trace needs)
    _native.call("fhe_debug_trace", buf.data_ptr())
    plan.run(inp, out)
    torch.cuda.synchronize()
    _native.call("fhe_debug_trace", None)
    t = buf.cpu().numpy().reshape(8, 4096)
    t0 = t[t > 0].min()
    print("layer", l.name, "path", plan.path)
    st = t[4][t[4] > 0] - t0
    li = t[2][64:64 + 4000]
    li = li[li > 0] - t0
    if len(st) > 8:
        full, issued = st[0::2], st[1::2]
        m = min(len(full), len(issued), len(li))
        print("stage: load_issue, full_ok, mma_issued (first 6):")
        for k in range(min(6, m)):
            print(f"   {k:3d} {li[k]:8d} {full[k]:8d} {issued[k]:8d}  load->full {full[k] - li[k]:6d}  issue {issued[k] - full[k]:5d}")
        gap = full[1:m] - issued[:m - 1]
        print("median: load->full", int(np.median(full[:m] - li[:m])), "issue", int(np.median(issued[:m] - full[:m])),
              "wait-for-data", int(np.median(gap)))
    for k, name in enumerate(KINDS):
        v = t[k][t[k] > 0] - t0
        print(f"{name:16s} n={len(v):4d} first={v[:12].tolist()}")
        if len(v) > 2:
            print(f"{'':16s} median step={int(np.median(np.diff(v)))} last={int(v[-1])}")


if __name__ == "__main__":
    main()
