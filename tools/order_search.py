"""Measured local search over the job order of the config-5 stacked K1-TC
launch (development probe for the schedule's cost model, conv._stage_times):
prints the time of the Johnson orders under several model constants and the
best order a first-improvement insertion search finds."""

import os
import random
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import bench  # noqa: E402
from paper_2401_16732_b200 import conv  # noqa: E402

P, layers = bench.build_stack(os.environ.get("WL", "config5"))
names = [L["layer"].name for L in layers]
items = [(L["plan"], L["dev"], None, L["out"]) for L in layers]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
johnson = conv._stack_schedule
perm_now = None


def fixed(its):
    return [its[k] for k in perm_now]


def t_order(perm, steps=12):
    global perm_now
    perm_now = perm
    conv._stack_schedule = fixed
    ts = bench.time_steps(lambda: conv.issue_k1(items), steps, 3, flush)
    return float(np.median(ts))


def johnson_perm():
    conv._stack_schedule = johnson
    order = johnson(items)
    return [next(k for k, it in enumerate(items) if it is o) for o in order]


for fill in (0, 2, 4, 6):
    conv._RELAYOUT_FILL_S = fill * 1e-6
    p = johnson_perm()
    print(f"johnson fill={fill}us: {t_order(p, 20):.4f} ms", [names[k] for k in p], flush=True)
conv._RELAYOUT_FILL_S = 4e-6
best = johnson_perm()
bt = t_order(best, 20)
rnd = random.Random(1)
for it in range(int(os.environ.get("ITERS", "120"))):
    cand = best[:]
    i, j = rnd.randrange(len(cand)), rnd.randrange(len(cand))
    cand.insert(j, cand.pop(i))
    if cand == best:
        continue
    t = t_order(cand)
    if t < bt * 0.997:
        t = t_order(cand, 20)  # confirm
        if t < bt * 0.997:
            best, bt = cand, t
            print(f"iter {it}: {bt:.4f} ms", [names[k] for k in best], flush=True)
print(f"best {bt:.4f} ms", [names[k] for k in best])
print("johnson fill=4 again:", round(t_order(johnson_perm(), 20), 4))
