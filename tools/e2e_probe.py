"""Where the e2e step's time goes: host enqueue time vs device copy/compute (development tool)."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2401_16732_b200 import bfv, conv  # noqa: E402
from paper_2401_16732_b200.device import DeviceRows  # noqa: E402
from paper_2401_16732_b200.ring import Domain  # noqa: E402

P, layers = bench.build_stack("config4")
pinned = [torch.from_numpy(L["host"].reshape(-1, P.n)).pin_memory() for L in layers]


def jobs():
    out = []
    for L, pt in zip(layers, pinned):
        cts = bfv.CtStack(DeviceRows(host=pt.numpy(), pinned=pt), P.q, bfv.Encoding.DIRECT, Domain.COEFF)
        out.append((conv.PackedTensor(cts, L["layout"], L["spec"].c_i), L["spec"]))
    return out


orig_sync = torch.cuda.Stream.synchronize
marks = {}


def timed_sync(self):
    marks["enqueued"] = time.perf_counter()
    return orig_sync(self)


for it in range(4):
    js = jobs()
    torch.cuda.synchronize()
    torch.cuda.Stream.synchronize = timed_sync
    t0 = time.perf_counter()
    outs = conv.conv_proposed_stream(js, P)
    t1 = time.perf_counter()
    torch.cuda.Stream.synchronize = orig_sync
    print(f"total {1e3 * (t1 - t0):.3f} ms, host enqueue {1e3 * (marks['enqueued'] - t0):.3f} ms")

if len(sys.argv) > 1 and sys.argv[1] == "profile":
    import cProfile
    import pstats

    pr = cProfile.Profile()
    for it in range(5):
        js = jobs()
        torch.cuda.synchronize()
        pr.enable()
        outs = conv.conv_proposed_stream(js, P)
        pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)

if len(sys.argv) > 1 and sys.argv[1] == "pieces":
    import collections

    acc = collections.defaultdict(float)
    comp = torch.cuda.current_stream()
    up, down = conv._streams()
    for it in range(5):
        js = jobs()
        torch.cuda.synchronize()
        for x, layer in js:
            t0 = time.perf_counter()
            plan = conv._proposed_plan(x, layer, P)
            t1 = time.perf_counter()
            inp, ready = x.cts.rows.upload_on(up)
            t2 = time.perf_counter()
            inp = inp.reshape(-1, 2, P.n)
            out = torch.empty((plan.n_out, 2, P.n), dtype=torch.int64, device=inp.device)
            t3 = time.perf_counter()
            (ev,) = conv.issue_k1([(plan, inp, ready, out)])
            t4 = time.perf_counter()
            down.wait_event(ev)
            rows = conv.device.DeviceRows.download_on(out, down)
            t5 = time.perf_counter()
            if it:
                for k, v in zip(("plan", "upload", "empty", "issue_k1", "download"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
                    acc[k] += v
        down.synchronize()
    print({k: round(v / 4 / 20 * 1e6, 1) for k, v in acc.items()}, "us per job")
