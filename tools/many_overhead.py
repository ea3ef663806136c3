"""Host cost of conv.conv_proposed_many (one stacked launch for R inputs of one
layer) against its device time (development probe)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2401_16732_b200 import bfv, conv, params  # noqa: E402

P = params.default_params()
rng = np.random.default_rng(0)
for (H, f_w, c_i, c_o, R) in [(56, 3, 64, 64, 4), (14, 3, 256, 256, 4), (7, 3, 512, 512, 4)]:
    lay = conv.layout_direct(P, H, H, f_w)
    spec = conv.ConvLayerSpec(H, H, f_w, c_i, c_o, rng.integers(-127, 128, (c_o, c_i, f_w, f_w)))
    xs = [conv.PackedTensor(bfv.cts_from_rows(torch.from_numpy(rng.integers(0, P.q, (lay.ct_count(c_i), 2, P.n))).cuda(),
                                              P.q, bfv.Encoding.DIRECT, bfv.Domain.COEFF), lay, c_i) for _ in range(R)]
    for _ in range(5):
        conv.conv_proposed_many(xs, spec, P)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        conv.conv_proposed_many(xs, spec, P)
    host = (time.perf_counter() - t0) / 50 * 1e6
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / 50 * 1e6
    plan = conv.conv_plan(spec, lay, P)
    outs = [torch.empty((plan.n_out, 2, P.n), dtype=torch.int64, device="cuda") for _ in range(R)]
    items = [(plan, bfv.cts_rows(x.cts), None, o) for x, o in zip(xs, outs)]
    g = torch.cuda.CUDAGraph()
    conv.issue_k1(items)
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        conv.issue_k1(items)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{H}x{H} {c_i}->{c_o} x{R}: host {host:.1f} us/call, wall {wall:.1f} us/call, device (graph) "
          f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us/launch")
