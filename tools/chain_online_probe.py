"""Per-step device time of inference.he_forward_online (CUDA events between
the enqueued steps; development probe):  python tools/chain_online_probe.py [config5]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2401_16732_b200 import act2pc, bfv, conv, inference, params  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config5"
P = params.default_params()
rng = np.random.default_rng(5)
layers = inference.config_layers(name)
seq, pool, fc = inference.main_path(layers)
weights = inference.random_weights(layers, rng)
specs = inference.layer_specs(layers, weights)
sk = bfv.keygen(P, rng)
marks = []
orig_act, orig_conv = act2pc.run_layer_activation, conv.conv_proposed


def ev(tag):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((tag, e))


def act(*a, **k):
    ev("conv/pool")
    r = orig_act(*a, **k)
    ev("act")
    return r


act2pc.run_layer_activation = act
for it in range(2):
    marks.clear()
    x = rng.integers(0, 8, (seq[0].c_i, seq[0].H, seq[0].W), dtype=np.int64)
    prepared = inference.he_prepare(layers, P, sk, rng)
    cur = conv.pack_input(x, P, seq[0].f_w, lambda pt: bfv.encrypt_private(pt, sk, rng))
    rows = bfv.cts_rows(cur.cts).contiguous()
    cur = conv.PackedTensor(bfv.cts_from_rows(rows, P.q, bfv.Encoding.DIRECT, bfv.Domain.COEFF), cur.layout,
                            cur.channels, cur.scale)
    torch.cuda.synchronize()
    ev("start")
    inference.he_forward_online(layers, cur, weights, sk, P, prepared, specs=specs)
    ev("end")
    torch.cuda.synchronize()
tot = {}
convs = [l for l in seq if l.kind == "conv"]
ci = 0
for (t0, e0), (t1, e1) in zip(marks, marks[1:]):
    ms = e0.elapsed_time(e1)
    tot[t1] = tot.get(t1, 0) + ms
    if t1 == "act":
        print(f"  act after {convs[ci].name:9s} {ms * 1e3:8.1f} us")
        ci += 1
print({k: round(v, 3) for k, v in tot.items()}, "ms total", round(sum(tot.values()), 3))
