"""Per-conv device timing inside the config-3/4/5 inference chain (development
probe): wraps conv.conv_proposed with synchronised wall clocks and CUDA events
and prints each call's time, its K1 path and the layer geometry.

    python tools/chain_probe.py [--config config5] [--runs 2]
"""

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import bfv, conv, inference, params  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config5")
    ap.add_argument("--runs", type=int, default=2)
    args = ap.parse_args()
    P = params.default_params()
    layers = inference.config_layers(args.config)
    rng = np.random.default_rng(77)
    weights = inference.random_weights(layers, rng)
    specs = inference.layer_specs(layers, weights)
    sk = bfv.keygen(P, np.random.default_rng(78))
    orig = conv.conv_proposed
    log = []

    def timed(x, layer, params_, *a, **k):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        y = orig(x, layer, params_, *a, **k)
        e1.record()
        torch.cuda.synchronize()
        plan = conv.conv_plan(layer, x.layout, params_)
        log.append((f"{layer.height}x{layer.width} f{layer.f_w} {layer.c_i}->{layer.c_o}", plan.path,
                    (time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1), torch.cuda.memory_allocated() >> 20))
        return y

    conv.conv_proposed = timed
    for it in range(args.runs):
        log.clear()
        r = np.random.default_rng(78 + it)
        x = r.integers(0, 8, (3, layers[0].H, layers[0].W), dtype=np.int64)
        t = {}
        got = inference.he_forward(layers, x, weights, sk, r, P, timings=t, specs=specs)
        ok = bool(np.array_equal(got, inference.plain_forward(layers, x, weights, P.p)))
        print(f"run {it}: ok={ok} " + " ".join(f"{k}={v * 1e3:.2f}ms" for k, v in t.items()))
        for g, path, wall, dev, mb in log:
            print(f"   {g:24s} {path:3s} wall {wall:8.3f} ms  device {dev:8.3f} ms  alloc {mb} MiB")


if __name__ == "__main__":
    main()
