"""Johnson order and estimated flow-shop makespan of the config-5 stacked launch for several cost-model constants (development probe)."""
import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2401_16732_b200 import conv, params, stacks
P = params.default_params()
rng = np.random.default_rng(0)
items = []
for l in stacks.conv_layers(stacks.config5()):
    w = rng.integers(-127, 128, (l.c_o, l.c_i, l.f_w, l.f_w))
    spec = conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, w)
    lay = conv.layout_direct(P, l.H, l.W, l.f_w)
    plan = conv.conv_plan(spec, lay, P)
    items.append((plan, l.name))
import itertools
for fill, bps, gf in [(0,.9e12,2e-6),(2e-6,.9e12,2e-6),(4e-6,.9e12,2e-6),(4e-6,1.2e12,2e-6),(4e-6,.9e12,4e-6),(2e-6,1.2e12,2e-6),(6e-6,1.2e12,3e-6)]:
    conv._RELAYOUT_BPS = bps; conv._LAYER_FILL_S = gf
    conv._RELAYOUT_FILL_S = fill
    order = conv._stack_schedule(items)
    t = [conv._stage_times(p) for p, _ in order]
    # flow shop makespan estimate
    a = b = 0.0
    for r, g in t:
        a += r; b = max(a, b) + g
    print(fill, round(b*1e6,1), [n for _, n in order])
