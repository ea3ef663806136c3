"""Per-kernel device timeline of one bench step (development tool).

Builds the bench stack, captures one CUDA graph with external event nodes
around every K1 launch (prep / GEMM / integer path), replays it after an L2
flush and prints each launch's duration and the gaps between launches.

    python tools/step_breakdown.py [--workload config4] [--reps 5]
"""

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2401_16732_b200 import _native, device  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config4")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--overlap", action="store_true", help="bench schedule (conv.issue_k1): GEMM times only")
    args = ap.parse_args()
    P, layers = bench.build_stack(args.workload)
    flush = torch.empty(2**25, dtype=torch.int64, device="cuda")
    rec = _native.fn("fhe_record_event")
    marks = []  # (label, event)

    def mk(label):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((label, e))
        return e

    def step(capture):
        for L in layers:
            plan = L["plan"]
            name = L["layer"].name
            if capture:
                e0 = mk(f"{name}:start")
                rec(e0.cuda_event, device.stream())
            plan.run(L["dev"], L["out"])
        if capture:
            e = mk("end")
            rec(e.cuda_event, device.stream())

    if args.overlap:
        from paper_2401_16732_b200 import conv

        gev = {}

        def on_gemm(i, what):
            e = gev.setdefault((i, what), torch.cuda.Event(enable_timing=True))
            rec(e.cuda_event, device.stream())

        def step(capture):  # noqa: F811
            if capture:
                rec(mk("start").cuda_event, device.stream())
            conv.issue_k1([(L["plan"], L["dev"], None, L["out"]) for L in layers],
                          on_gemm=on_gemm if capture else None)
            if capture:
                rec(mk("end").cuda_event, device.stream())

        for i, L in enumerate(layers):
            if L["plan"].path == "tc":
                for w in ("start", "end"):
                    gev[(i, w)] = torch.cuda.Event(enable_timing=True)
                    gev[(i, w)].record()
    for _ in range(3):
        step(False)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step(True)
    acc = np.zeros(len(marks) - 1)
    for _ in range(args.reps):
        bench.flush_l2(flush)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        acc += [marks[i][1].elapsed_time(marks[i + 1][1]) for i in range(len(marks) - 1)]
    acc /= args.reps
    total = acc.sum()
    if args.overlap:
        print(f"step {total * 1e3:.1f} us (overlapped schedule, graph replay after L2 flush)")
        t0 = marks[0][1]
        for i, L in enumerate(layers):
            if (i, "start") in gev:
                g0, g1 = gev[(i, "start")], gev[(i, "end")]
                print(f"  {L['layer'].name:10s} k1-tc [{t0.elapsed_time(g0) * 1e3:7.1f}, {t0.elapsed_time(g1) * 1e3:7.1f}]"
                      f" = {g0.elapsed_time(g1) * 1e3:6.1f} us")
        return
    print(f"step {total * 1e3:.1f} us (graph replay after L2 flush, event nodes between launches)")
    for (label, _), ms in zip(marks[:-1], acc):
        print(f"  {label.split(':')[0]:10s} {ms * 1e3:8.1f} us")


if __name__ == "__main__":
    main()
