"""Stack order vs K1-TC launch time (independent layers; development tool)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2401_16732_b200 import conv  # noqa: E402

P, layers = bench.build_stack("config4")
flush = torch.empty(2**25, dtype=torch.int64, device="cuda")
macs = [L["macs"] for L in layers]
idx = list(range(len(layers)))
big_first = sorted(idx, key=lambda i: -macs[i])
inter = []
a, b = big_first[:], big_first[::-1]
while a:
    inter.append(a.pop(0))
    if a:
        inter.append(a.pop())
orders = {"network": idx, "reverse": idx[::-1], "big_first": big_first, "small_first": big_first[::-1],
          "interleaved": inter}
for name, order in orders.items():
    items = [(layers[i]["plan"], layers[i]["dev"], None, layers[i]["out"]) for i in order]
    for _ in range(3):
        conv.issue_k1(items)
    torch.cuda.synchronize()
    ts = []
    for _ in range(15):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        conv.issue_k1(items)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{name:12s} {sorted(ts)[7]:.4f} ms")
