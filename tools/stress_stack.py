"""Repeated stacked launches compared with single-layer launches (race hunting).

    python tools/stress_stack.py [--reps 20] [--workloads config4,config3] [--order given|johnson]
"""

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2401_16732_b200 import conv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--workloads", default="config4,config3")
    ap.add_argument("--poison", action="store_true", help="fill the digit-plane scratch before every launch")
    args = ap.parse_args()
    layers = []
    for k, w in enumerate(args.workloads.split(",")):
        layers += [dict(L, name=f"{w}:{L['layer'].name}") for L in bench.build_stack(w, seed=41 + k)[1]]
    refs = [L["plan"].run(L["dev"], torch.empty_like(L["out"])) for L in layers]
    items = [(L["plan"], L["dev"], None, L["out"]) for L in layers]
    bad = 0
    from paper_2401_16732_b200 import device

    conv.issue_k1(items)
    torch.cuda.synchronize()
    scratch = device._scratch[(torch.cuda.current_device(), "conv_tc_x")]
    for rep in range(args.reps):
        for L in layers:
            L["out"].fill_(-1)
        if args.poison:
            scratch.fill_(rep & 0xFF)  # stale digit-plane reads would now produce wrong outputs
        conv.issue_k1(items)
        torch.cuda.synchronize()
        wrong = [L["name"] for L, r in zip(layers, refs) if not torch.equal(L["out"], r)]
        if wrong:
            bad += 1
            print(f"rep {rep}: {len(wrong)} layers differ: {wrong[:6]}")
    print(f"{bad} of {args.reps} repetitions wrong ({len(layers)} layers per repetition)")


if __name__ == "__main__":
    main()
