"""One stacked K1-TC launch of a bench workload (for ncu). Development tool."""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2401_16732_b200 import conv  # noqa: E402

args = [a for a in sys.argv[1:] if a != "--workload"]
only = None
if "--only" in args:  # one layer of the workload by name (e.g. --only stem)
    only = args[args.index("--only") + 1]
    args = args[: args.index("--only")]
P, layers = bench.build_stack(args[0] if args else "config5")
if only:
    layers = [L for L in layers if L["layer"].name == only]
items = [(L["plan"], L["dev"], None, L["out"]) for L in layers]
conv.issue_k1(items)
torch.cuda.synchronize()
conv.issue_k1(items)
torch.cuda.synchronize()
print("ok")
