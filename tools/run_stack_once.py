"""One stacked K1-TC launch of a bench workload (for ncu). Development tool."""

import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2401_16732_b200 import conv  # noqa: E402

P, layers = bench.build_stack(sys.argv[1] if len(sys.argv) > 1 else "config4")
items = [(L["plan"], L["dev"], None, L["out"]) for L in layers]
conv.issue_k1(items)
torch.cuda.synchronize()
conv.issue_k1(items)
torch.cuda.synchronize()
print("ok")
