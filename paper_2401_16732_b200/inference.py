"""Configs 3 and 4 end to end on the device — the caller of the hot path.

The conv stack of `stacks.py` run as a chain, both parties in-process:
Flash conv (K1, conv.conv_proposed) -> x²+x on shares with the client's
repack into the next conv's layout (act2pc layer protocol, SPEC.md:304-331,
conv.py:162-197; strided convs are subsampled there) -> ... -> avg_pool ->
fully_connected -> decrypt. The reference has no model module (SPEC's absent
`model` lists ResidualAdd), so shortcut projections and residual additions
are not modelled: the chain is the ResNet's main path. Config 5's 2x2 pool
after the stem would need a server-side repack between two linear layers and
is not covered. The integer model `plain_forward` is the parity reference:
decrypted logits equal it mod p.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

from . import act2pc, bfv, conv, stacks
from .params import RingParams


def main_path(layers):
    """The convs of the ResNet main path (no projections), the final pool and FC."""
    convs = [l for l in layers if l.kind == "conv" and not l.name.endswith("proj")]
    pool = next(l for l in layers if l.kind == "pool" and l.name == "avgpool")
    fc = next(l for l in layers if l.kind == "fc")
    return convs, pool, fc


def random_weights(layers, rng, bound: int = 127) -> dict:
    convs, pool, fc = main_path(layers)
    w = {l.name: rng.integers(-bound, bound + 1, (l.c_o, l.c_i, l.f_w, l.f_w), dtype=np.int64) for l in convs}
    w["fc"] = rng.integers(-bound, bound + 1, (fc.c_o, fc.c_i), dtype=np.int64)
    return w


def _conv_same(a: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Zero-padded correlation, the closed form of conv.conv_proposed's slots."""
    f = w.shape[-1]
    p = f // 2
    c, h, wd = a.shape
    pad = np.pad(a, ((0, 0), (p, p), (p, p)))
    out = np.zeros((w.shape[0], h, wd), dtype=np.int64)
    for dy in range(f):
        for dx in range(f):
            out += np.einsum("oi,ihw->ohw", w[:, :, dy, dx], pad[:, dy : dy + h, dx : dx + wd])
    return out


def plain_forward(layers, x: np.ndarray, weights: dict, p: int, frac_bits: int = 0) -> np.ndarray:
    """Integer model mod p: conv, stride subsample, a² + a·2^f, window sum, FC."""
    convs, pool, fc = main_path(layers)
    a = np.asarray(x, dtype=np.int64) % p
    for l in convs:
        a = _conv_same(a, weights[l.name]) % p
        a = a[:, :: l.stride, :: l.stride]
        a = (a * a + a * (1 << frac_bits)) % p
    pooled = a.reshape(a.shape[0], -1).sum(axis=1) % p
    return (weights["fc"] @ pooled) % p


def layer_specs(layers, weights: dict) -> dict:
    """ConvLayerSpec per main-path conv (they cache their K1 plans: build once, reuse)."""
    convs, _, _ = main_path(layers)
    return {l.name: conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, weights[l.name]) for l in convs}


def he_forward(layers, x: np.ndarray, weights: dict, sk: bfv.SecretKey, rng, params: RingParams,
               frac_bits: int = 0, timings: dict | None = None, specs: dict | None = None) -> np.ndarray:
    """The encrypted chain on the device; returns the decrypted logits mod p."""
    import time

    import torch

    P = params
    convs, pool, fc = main_path(layers)
    specs = specs if specs is not None else layer_specs(layers, weights)
    t_conv = t_act = t_off = 0.0
    cur = conv.pack_input(x, P, convs[0].f_w, lambda pt: bfv.encrypt_private(pt, sk, rng))
    for i, l in enumerate(convs):
        spec = specs[l.name]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y = conv.conv_proposed(cur, spec, P)
        torch.cuda.synchronize()
        t_conv += time.perf_counter() - t0
        if l.stride > 1:  # subsampled by the client's repack below
            y = conv.PackedTensor(y.cts, replace(y.layout, stride=l.stride), y.channels, y.scale)
        h = l.H // l.stride
        nxt = convs[i + 1].f_w if i + 1 < len(convs) else 3
        t0 = time.perf_counter()
        plan = act2pc.RepackPlan(y.layout, l.c_o, conv.layout_direct(P, h, h, nxt), P)
        sess = act2pc.offline_prepare_layer(plan, P, rng, frac_bits=frac_bits)
        zeros = bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        cur = act2pc.run_layer_activation(y, sess, sk, zeros, P)
        torch.cuda.synchronize()
        t_off += t1 - t0
        t_act += time.perf_counter() - t1
    t0 = time.perf_counter()
    pooled = conv.avg_pool(cur, pool.f_w, P)
    logits = conv.fully_connected(pooled, weights["fc"], P)
    out = bfv.centered(conv.read_scalar_outputs(logits, sk), P.p) % P.p
    t_tail = time.perf_counter() - t0
    if timings is not None:
        timings.update(conv_s=t_conv, act_s=t_act, offline_s=t_off, tail_s=t_tail)
    return out


def config_layers(name: str):
    return stacks.CONFIGS[name]()
