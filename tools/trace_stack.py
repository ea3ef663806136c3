"""Timeline of CTA 0 through the stacked K1-TC launch of a bench workload.

Development probe:  python tools/trace_stack.py [--workload config4]
Prints per layer (cycles from kernel start, CTA 0): relayout warp done with
the layer, loader sees the layer's X ready, first MMA tile start, last MMA
commit, last epilogue done.

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

import bench  # noqa: E402
from paper_2401_16732_b200 import _native, conv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config4")
    ap.add_argument("--only", default=None, help="trace this layer alone (a single-layer launch)")
    ap.add_argument("--cta-dump", default=None, help="write per-CTA [start, end] globaltimer ns and the dealing offsets (.npz)")
    ap.add_argument("--detail", default=None, help="per-epilogue-warp timing of this layer's tiles (CTA 0)")
    args = ap.parse_args()
    P, layers = bench.build_stack(args.workload)
    if args.only:  # one layer alone: the drop-in single-layer launch (conv_proposed's path)
        layers = [L for L in layers if L["layer"].name == args.only]
    items = [(L["plan"], L["dev"], None, L["out"]) for L in layers]
    conv.issue_k1(items)
    torch.cuda.synchronize()
    buf = torch.full((25 * 4096,), -1, dtype=torch.int64, device="cuda")
    buf[: 7 * 4096].zero_()
    _native.call("fhe_debug_trace", buf.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    conv.issue_k1(items)
    e1.record()
    torch.cuda.synchronize()
    _native.call("fhe_debug_trace", None)
    allb = buf.cpu().numpy().astype(np.int64)
    t = allb[: 8 * 4096].reshape(8, 4096)
    ct = allb[8 * 4096 : 8 * 4096 + 2 * 148].reshape(148, 2)
    print(f"traced launch: {e0.elapsed_time(e1) * 1e3:.1f} us (events)")
    cc = allb[8 * 4096 + 512 : 8 * 4096 + 512 + 2 * 148].reshape(148, 2)
    mhz = (cc[:, 1] - cc[:, 0]) / ((ct[:, 1] - ct[:, 0]) / 1e3)
    print(f"SM clock during the launch (clock64 / globaltimer): median {np.median(mhz):.0f} MHz "
          f"(min {mhz.min():.0f}, max {mhz.max():.0f})")
    if args.cta_dump:
        np.savez(args.cta_dump, ct=ct, toff=allb[7 * 4096 + 2048 : 7 * 4096 + 2048 + 24])
    t0g = ct[:, 0].min()
    rd = allb[8 * 4096 + 1024 : 8 * 4096 + 1024 + 2 * 148].reshape(148, 2)
    for k in range(2):
        v = (rd[:, k] - t0g) / 1e3
        v = v[rd[:, k] > 0]
        if len(v):
            print(f"layer {k} relayout done per CTA (us): min {v.min():.1f} p50 {np.median(v):.1f} p90 "
                  f"{np.percentile(v, 90):.1f} max {v.max():.1f}")
    ends = (ct[:, 1] - t0g) / 1e3
    print(f"per-CTA globaltimer (us from the first CTA start): start spread {(ct[:, 0].max() - t0g) / 1e3:.1f}, "
          f"end min {ends.min():.1f} median {np.median(ends):.1f} max {ends.max():.1f} (CTA {int(ends.argmax())})")
    if conv._stack_order():  # issue_k1's launch order
        order = conv._stack_schedule([(L["plan"], k) for k, L in enumerate(layers)])
        layers = [layers[k] for _, k in order]
    t0 = t[2][0]
    rel = lambda v: int(v - t0) if v else -1  # noqa: E731
    tl = 0
    toff = 0
    print(f"{'layer':10s} {'rel_start':>9s} {'rel_done':>9s} {'x_ready':>9s} {'mma0':>9s} {'mma_end':>9s} {'epi_end':>9s} tiles(CTA0)"
          f" {'mma/tile':>9s} {'wait/tile':>9s} {'epi/tile':>9s} {'commit->epi':>11s}")
    for l, L in enumerate(layers):
        d = L["plan"].tc
        seq = t[7][1024:2048]  # the layer of each tile CTA 0 ran (the kernel's tile sequence)
        idx = np.nonzero(seq[: int(np.count_nonzero(t[0][:1024]))] == l)[0]
        mine = len(idx)
        first, last = (int(idx[0]), int(idx[-1])) if mine else (tl, tl - 1)
        print(f"{L['layer'].name:10s} {rel(t[2][64 + l]) if l else -1:9d} {rel(t[3][l]) if l else -1:9d} {rel(t[7][l]):9d} {rel(t[0][first]) if mine else -1:9d} "
              f"{rel(t[1][last]) if mine else -1:9d} {rel(t[6][last]) if mine else -1:9d} {mine:11d}"
              f" {int(np.mean([t[1][i] - t[0][i] for i in range(first, last + 1)])) if mine else -1:9d}"
              f" {int(np.mean([t[4][i] - t[0][i] for i in range(first, last + 1)])) if mine else -1:9d}"
              f" {int(np.mean([t[6][i] - t[5][i] for i in range(first, last + 1)])) if mine else -1:9d}"
              f" {int(np.mean([t[5][i] - t[1][i] for i in range(first, last + 1)])) if mine else -1:11d}")
        if args.detail == L["layer"].name and mine:
            W = allb[9 * 4096 : 25 * 4096].reshape(16, 4096)
            for i in range(first, min(last + 1, first + 12)):
                seen = W[:8, i] - t[0][first]
                done = W[8:, i] - t[0][first]
                print(f"  tile {i - first:3d}: mma start {int(t[0][i] - t[0][first]):7d} tempty {int(t[4][i] - t[0][first]):7d} "
                      f"commit {int(t[1][i] - t[0][first]):7d} | tfull seen per warp " + " ".join(f"{int(v):7d}" for v in seen)
                      + " | done " + " ".join(f"{int(v):7d}" for v in done))
        tl += mine



if __name__ == "__main__":
    main()
