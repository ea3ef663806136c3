"""Configs 3, 4 and 5 end to end on the device — the caller of the hot path.

The conv stack of `stacks.py` run as a chain, both parties in-process:
Flash conv (K1, conv.conv_proposed) -> x²+x on shares with the client's
repack into the next conv's layout (act2pc layer protocol, SPEC.md:304-331,
conv.py:162-197; strided convs are subsampled there) -> ... -> avg_pool ->
fully_connected -> decrypt. The reference has no model module (SPEC's absent
`model` lists ResidualAdd); the basic blocks' shortcuts are added here on the
server before the block's second activation (`residual=True`, the default):
an identity shortcut is the block input itself, moved into the conv output
layout by DRot and added in one launch (conv.residual_add); a 1x1 stride-2
projection runs on the block input after a masked repack round applies the
stride (its 1x1 weights as the centre tap of a 3x3 conv_proposed, so its
output layout is the second conv's). Config 5's 2x2 pool
after the stem is evaluated by the server and its stride applied by one
masked repack round (act2pc.run_repack_round). The integer model
`plain_forward` is the parity reference: decrypted logits equal it mod p.
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

from . import act2pc, bfv, conv, device, stacks
from .errors import EncodingError
from .params import RingParams


def main_path(layers):
    """The ResNet main path in order (convs without projections, any pool
    between convs, the final pool and FC) and the final pool / FC layers."""
    seq = [l for l in layers if not (l.kind == "conv" and l.name.endswith("proj"))]
    pool = next(l for l in layers if l.kind == "pool" and l.name == "avgpool")
    fc = next(l for l in layers if l.kind == "fc")
    return seq, pool, fc


def _convs(layers):
    return [l for l in main_path(layers)[0] if l.kind == "conv"]


def blocks(layers) -> dict:
    """Basic blocks: second conv's name -> (first conv's name, projection
    Layer or None for an identity shortcut)."""
    convs = {l.name: l for l in layers if l.kind == "conv"}
    return {name: (name[:-2] + "c1", convs.get(name[:-2] + "proj"))
            for name in convs if name.endswith("c2") and name[:-2] + "c1" in convs}


def random_weights(layers, rng, bound: int = 127) -> dict:
    _, _, fc = main_path(layers)
    w = {l.name: rng.integers(-bound, bound + 1, (l.c_o, l.c_i, l.f_w, l.f_w), dtype=np.int64)
         for l in _convs(layers)}
    w["fc"] = rng.integers(-bound, bound + 1, (fc.c_o, fc.c_i), dtype=np.int64)
    for l in layers:  # projection shortcuts last (the main-path draws above keep their values)
        if l.kind == "conv" and l.name.endswith("proj"):
            w[l.name] = rng.integers(-bound, bound + 1, (l.c_o, l.c_i, l.f_w, l.f_w), dtype=np.int64)
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


def plain_forward(layers, x: np.ndarray, weights: dict, p: int, frac_bits: int = 0,
                  residual: bool = True) -> np.ndarray:
    """Integer model mod p: conv, stride subsample, [+ the block's shortcut:
    its input, or the strided 1x1 projection of it], a² + a·2^f, window sums
    (pools: sum of each k x k block), FC."""
    seq, pool, fc = main_path(layers)
    blk = blocks(layers) if residual else {}
    firsts = {c1 for c1, _ in blk.values()}
    a = np.asarray(x, dtype=np.int64) % p
    a_in = None
    for l in seq:
        if l.kind == "conv":
            if l.name in firsts:
                a_in = a
            a = _conv_same(a, weights[l.name]) % p
            a = a[:, :: l.stride, :: l.stride]
            if l.name in blk:
                proj = blk[l.name][1]
                if proj is None:
                    sc = a_in
                else:
                    s = proj.stride
                    sc = np.einsum("oi,ihw->ohw", weights[proj.name][:, :, 0, 0], a_in[:, ::s, ::s])
                a = (a + sc) % p
            a = (a * a + a * (1 << frac_bits)) % p
        elif l.kind == "pool":
            k = l.f_w
            c, h, w = a.shape
            a = a.reshape(c, h // k, k, w // k, k).sum(axis=(2, 4)) % p
    return (weights["fc"] @ a.reshape(a.shape[0])) % p


def layer_specs(layers, weights: dict) -> dict:
    """ConvLayerSpec per main-path conv (they cache their K1 plans: build once,
    reuse), and per projection shortcut with weights: the 1x1 weights as the
    centre tap of a 3x3 conv at the strided resolution (its input is the
    block input repacked with the stride into a pad-1 layout)."""
    specs = {l.name: conv.ConvLayerSpec(l.H, l.W, l.f_w, l.c_i, l.c_o, weights[l.name]) for l in _convs(layers)}
    for l in layers:
        if l.kind == "conv" and l.name.endswith("proj") and l.name in weights:
            w3 = np.zeros((l.c_o, l.c_i, 3, 3), dtype=np.int64)
            w3[:, :, 1, 1] = np.asarray(weights[l.name]).reshape(l.c_o, l.c_i)
            specs[l.name] = conv.ConvLayerSpec(l.H // l.stride, l.W // l.stride, 3, l.c_i, l.c_o, w3)
    return specs


def _proj_plan(a_layout, proj, P: RingParams):
    """Masked repack of a block input into the projection's strided pad-1 layout."""
    src = replace(a_layout, stride=proj.stride)
    dst = conv.layout_direct(P, proj.H // proj.stride, proj.W // proj.stride, 3)
    return act2pc.repack_plan(src, proj.c_i, dst, P)


def _with_shortcut(y, a_in, sc_in, proj, specs: dict, P: RingParams):
    """y + the block's shortcut: a_in itself (identity) or the projection conv
    of sc_in (a_in repacked with the stride)."""
    sc = a_in if proj is None else conv.conv_proposed(sc_in, specs[proj.name], P)
    return conv.residual_add(y, sc, P)


def he_forward(layers, x: np.ndarray, weights: dict, sk: bfv.SecretKey, rng, params: RingParams,
               frac_bits: int = 0, timings: dict | None = None, specs: dict | None = None,
               residual: bool = True) -> np.ndarray:
    """The encrypted chain on the device; returns the decrypted logits mod p.

    conv -> x²+x layer exchange repacking into the next operation's layout
    (the next conv's input layout, or a pad-1 layout for a pool); a pool
    between convs (config 5) is evaluated by the server and its stride applied
    by a masked repack round (act2pc.run_repack_round) before the next conv."""
    import time

    import torch

    P = params
    seq, pool, fc = main_path(layers)
    specs = specs if specs is not None else layer_specs(layers, weights)
    blk = blocks(layers) if residual else {}
    firsts = {c1 for c1, _ in blk.values()}
    a_in = None
    t = dict(conv_s=0.0, act_s=0.0, offline_s=0.0, repack_s=0.0, shortcut_s=0.0)
    per_conv = []
    first = seq[0]
    t0 = time.perf_counter()
    # the client's encrypted input as one device stack (encryptions batched,
    # bit-identical to encrypt_private per ciphertext)
    cur = conv.pack_input_private(x, P, first.f_w, sk, rng)
    torch.cuda.synchronize()
    t["input_s"] = time.perf_counter() - t0

    def next_layout(i, h):
        nxt = seq[i + 1]
        return conv.layout_direct(P, h, h, nxt.f_w if nxt.kind == "conv" else 3)

    for i, l in enumerate(seq):
        if l.kind == "conv":
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            spec = specs[l.name]
            if l.name in firsts:
                a_in = cur
            buf = spec.__dict__.get("_out_buf")  # reused across inferences: the previous output is consumed
            y = conv.conv_proposed(cur, spec, P, out=buf)
            spec.__dict__["_out_buf"] = bfv.cts_rows(y.cts)
            torch.cuda.synchronize()
            t["conv_s"] += time.perf_counter() - t0
            per_conv.append(time.perf_counter() - t0)
            if l.name in blk:  # the block's shortcut, added before its second activation
                t0 = time.perf_counter()
                proj = blk[l.name][1]
                a_s = None
                if proj is not None:
                    plan = _proj_plan(a_in.layout, proj, P)
                    rs = act2pc.offline_prepare_repack(plan, P, rng)
                    zeros = bfv.precompute_zero_rows(sk, rng, plan.k_dst)
                    torch.cuda.synchronize()
                    t["offline_s"] += time.perf_counter() - t0
                    t0 = time.perf_counter()
                    a_s = act2pc.run_repack_round(a_in, rs, sk, zeros, P)
                y = _with_shortcut(y, a_in, a_s, proj, specs, P)
                torch.cuda.synchronize()
                t["shortcut_s"] += time.perf_counter() - t0
            if l.stride > 1:  # subsampled by the client's repack below
                y = conv.PackedTensor(y.cts, replace(y.layout, stride=l.stride), y.channels, y.scale)
            t0 = time.perf_counter()
            plan = act2pc.repack_plan(y.layout, l.c_o, next_layout(i, l.H // l.stride), P)
            sess = act2pc.offline_prepare_layer(plan, P, rng, frac_bits=frac_bits)
            zeros = bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            cur = act2pc.run_layer_activation(y, sess, sk, zeros, P)
            torch.cuda.synchronize()
            t["offline_s"] += t1 - t0
            t["act_s"] += time.perf_counter() - t1
        elif l.kind == "pool" and l is not pool:
            t0 = time.perf_counter()
            pooled = conv.avg_pool(cur, l.f_w, P)
            h = cur.layout.height // l.f_w
            plan = act2pc.repack_plan(pooled.layout, l.c_o, next_layout(i, h), P)
            rs = act2pc.offline_prepare_repack(plan, P, rng)
            zeros = bfv.precompute_zero_rows(sk, rng, plan.k_dst)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            cur = act2pc.run_repack_round(pooled, rs, sk, zeros, P)
            torch.cuda.synchronize()
            t["offline_s"] += t1 - t0
            t["repack_s"] += time.perf_counter() - t1
    t0 = time.perf_counter()
    pooled = conv.avg_pool(cur, pool.f_w, P)
    logits = conv.fully_connected(pooled, weights["fc"], P)
    out = bfv.centered(conv.read_scalar_outputs(logits, sk), P.p) % P.p
    t["tail_s"] = time.perf_counter() - t0
    if timings is not None:
        timings.update(t)
        timings["per_conv_s"] = per_conv
    return out


def he_forward_many(layers, xs, weights: dict, sk: bfv.SecretKey, rng, params: RingParams, frac_bits: int = 0,
                    timings: dict | None = None, specs: dict | None = None,
                    residual: bool = True) -> list[np.ndarray]:
    """he_forward over several independent requests in lockstep: each conv
    layer of all requests runs as stacked tensor-core launches
    (conv.conv_proposed_many -> conv.issue_k1, up to 24 requests per launch);
    the layer exchanges (act2pc) and the tail stay per request. Returns each
    request's decrypted logits mod p (equal to he_forward's)."""
    import time

    import torch

    P = params
    seq, pool, fc = main_path(layers)
    specs = specs if specs is not None else layer_specs(layers, weights)
    blk = blocks(layers) if residual else {}
    firsts = {c1 for c1, _ in blk.values()}
    a_ins = None
    t = dict(conv_s=0.0, act_s=0.0, offline_s=0.0, repack_s=0.0, shortcut_s=0.0)
    per_conv = []
    first = seq[0]
    t0 = time.perf_counter()
    curs = [conv.pack_input_private(x, P, first.f_w, sk, rng) for x in xs]
    torch.cuda.synchronize()
    t["input_s"] = time.perf_counter() - t0

    def next_layout(i, h):
        nxt = seq[i + 1]
        return conv.layout_direct(P, h, h, nxt.f_w if nxt.kind == "conv" else 3)

    for i, l in enumerate(seq):
        if l.kind == "conv":
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if l.name in firsts:
                a_ins = curs
            e0.record()
            ys = conv.conv_proposed_many(curs, specs[l.name], P)
            e1.record()
            torch.cuda.synchronize()
            t["conv_s"] += time.perf_counter() - t0
            t["conv_gpu_s"] = t.get("conv_gpu_s", 0.0) + e0.elapsed_time(e1) / 1e3  # device time of the launches
            per_conv.append(time.perf_counter() - t0)
            if l.name in blk:  # each request's shortcut (projections stacked across requests)
                t0 = time.perf_counter()
                proj = blk[l.name][1]
                if proj is None:
                    ys = [conv.residual_add(y, a, P) for y, a in zip(ys, a_ins)]
                else:
                    a_ss = []
                    for a in a_ins:
                        plan = _proj_plan(a.layout, proj, P)
                        rs = act2pc.offline_prepare_repack(plan, P, rng)
                        a_ss.append(act2pc.run_repack_round(a, rs, sk, bfv.precompute_zero_rows(sk, rng, plan.k_dst), P))
                    scs = conv.conv_proposed_many(a_ss, specs[proj.name], P)
                    ys = [conv.residual_add(y, sc, P) for y, sc in zip(ys, scs)]
                torch.cuda.synchronize()
                t["shortcut_s"] += time.perf_counter() - t0
            nxt = []
            for y in ys:
                if l.stride > 1:  # subsampled by the client's repack below
                    y = conv.PackedTensor(y.cts, replace(y.layout, stride=l.stride), y.channels, y.scale)
                t0 = time.perf_counter()
                plan = act2pc.repack_plan(y.layout, l.c_o, next_layout(i, l.H // l.stride), P)
                sess = act2pc.offline_prepare_layer(plan, P, rng, frac_bits=frac_bits)
                zeros = bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst)
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                nxt.append(act2pc.run_layer_activation(y, sess, sk, zeros, P))
                torch.cuda.synchronize()
                t["offline_s"] += t1 - t0
                t["act_s"] += time.perf_counter() - t1
            curs = nxt
        elif l.kind == "pool" and l is not pool:
            nxt = []
            for cur in curs:
                t0 = time.perf_counter()
                pooled = conv.avg_pool(cur, l.f_w, P)
                h = cur.layout.height // l.f_w
                plan = act2pc.repack_plan(pooled.layout, l.c_o, next_layout(i, h), P)
                rs = act2pc.offline_prepare_repack(plan, P, rng)
                zeros = bfv.precompute_zero_rows(sk, rng, plan.k_dst)
                torch.cuda.synchronize()
                t1 = time.perf_counter()
                nxt.append(act2pc.run_repack_round(pooled, rs, sk, zeros, P))
                torch.cuda.synchronize()
                t["offline_s"] += t1 - t0
                t["repack_s"] += time.perf_counter() - t1
            curs = nxt
    t0 = time.perf_counter()
    outs = []
    for cur in curs:
        pooled = conv.avg_pool(cur, pool.f_w, P)
        logits = conv.fully_connected(pooled, weights["fc"], P)
        outs.append(bfv.centered(conv.read_scalar_outputs(logits, sk), P.p) % P.p)
    t["tail_s"] = time.perf_counter() - t0
    if timings is not None:
        timings.update(t)
        timings["per_conv_s"] = per_conv
    return outs


def he_prepare(layers, params: RingParams, sk: bfv.SecretKey, rng, frac_bits: int = 0,
               residual: bool = True) -> list:
    """The chain's offline phase up front: for every activation exchange and
    pool repack of the main path, its repack plan, masks (act2pc sessions) and
    encryptions of zero, in chain order. The layouts follow from the geometry
    alone (conv output = input layout with one channel per ciphertext, stride
    pending; exchange output = the plan's destination), so no ciphertext is
    needed. Sessions are single-use: prepare once per inference."""
    P = params
    seq, pool, _ = main_path(layers)

    def next_layout(i, h):
        nxt = seq[i + 1]
        return conv.layout_direct(P, h, h, nxt.f_w if nxt.kind == "conv" else 3)

    blk = blocks(layers) if residual else {}
    firsts = {c1 for c1, _ in blk.values()}
    steps = []
    lay = conv.layout_direct(P, seq[0].H, seq[0].W, seq[0].f_w)
    a_lay = None
    for i, l in enumerate(seq):
        if l.kind == "conv":
            if l.name in firsts:
                a_lay = lay
            if l.name in blk and blk[l.name][1] is not None:  # the projection's repack round
                plan = _proj_plan(a_lay, blk[l.name][1], P)
                steps.append(("shortcut", plan, act2pc.offline_prepare_repack(plan, P, rng),
                              bfv.precompute_zero_rows(sk, rng, plan.k_dst)))
            y_lay = replace(lay, c_n=1, stride=l.stride) if l.stride > 1 else replace(lay, c_n=1)
            plan = act2pc.repack_plan(y_lay, l.c_o, next_layout(i, l.H // l.stride), P)
            sess = act2pc.offline_prepare_layer(plan, P, rng, frac_bits=frac_bits)
            steps.append(("act", plan, sess, bfv.precompute_zero_rows(sk, rng, 3 * plan.k_dst)))
            lay = plan.dst
        elif l.kind == "pool" and l is not pool:
            pooled = replace(lay, stride=l.f_w)
            plan = act2pc.repack_plan(pooled, l.c_o, next_layout(i, lay.height // l.f_w), P)
            steps.append(("repack", plan, act2pc.offline_prepare_repack(plan, P, rng),
                          bfv.precompute_zero_rows(sk, rng, plan.k_dst)))
            lay = plan.dst
    return steps


def he_forward_online(layers, cur, weights: dict, sk: bfv.SecretKey, params: RingParams, prepared: list,
                      specs: dict | None = None, residual: bool = True) -> np.ndarray:
    """The online phase of he_forward with the offline material of he_prepare:
    convs, activation exchanges and repacks enqueued back to back on the
    stream with no host synchronisation until the logits are read; the
    client's noise-budget checks are deferred to one read at the end
    (act2pc.check_deferred_budgets). `cur`: the uploaded input (a device
    PackedTensor). Returns the decrypted logits mod p (equal to he_forward's)."""
    P = params
    seq, pool, _ = main_path(layers)
    specs = specs if specs is not None else layer_specs(layers, weights)
    blk = blocks(layers) if residual else {}
    firsts = {c1 for c1, _ in blk.values()}
    a_in = None
    residuals = device.zeros_i64(max(1, len(prepared)))  # (cudaMemsetAsync, no fill kernel)
    k = 0
    for l in seq:
        if l.kind == "conv":
            spec = specs[l.name]
            if l.name in firsts:
                a_in = cur
            buf = spec.__dict__.get("_out_buf")  # reused across inferences: the previous output is consumed
            y = conv.conv_proposed(cur, spec, P, out=buf)
            spec.__dict__["_out_buf"] = bfv.cts_rows(y.cts)
            if l.name in blk:
                proj = blk[l.name][1]
                a_s = None
                if proj is not None:
                    kind, plan, rs, zeros = prepared[k]
                    if kind != "shortcut" or plan.src != replace(a_in.layout, stride=proj.stride):
                        raise EncodingError("prepared material does not match the chain (he_prepare for these layers)")
                    a_s = act2pc.run_repack_round(a_in, rs, sk, zeros, P, budget_into=(residuals, k))
                    k += 1
                y = _with_shortcut(y, a_in, a_s, proj, specs, P)
            if l.stride > 1:  # subsampled by the client's repack below
                y = conv.PackedTensor(y.cts, replace(y.layout, stride=l.stride), y.channels, y.scale)
            kind, plan, sess, zeros = prepared[k]
            if kind != "act" or plan.src != y.layout:
                raise EncodingError("prepared material does not match the chain (he_prepare for these layers)")
            cur = act2pc.run_layer_activation(y, sess, sk, zeros, P, budget_into=(residuals, k))
            k += 1
        elif l.kind == "pool" and l is not pool:
            pooled = conv.avg_pool(cur, l.f_w, P)
            kind, plan, rs, zeros = prepared[k]
            if kind != "repack" or plan.src != pooled.layout:
                raise EncodingError("prepared material does not match the chain (he_prepare for these layers)")
            cur = act2pc.run_repack_round(pooled, rs, sk, zeros, P, budget_into=(residuals, k))
            k += 1
    pooled = conv.avg_pool(cur, pool.f_w, P)
    logits = conv.fully_connected(pooled, weights["fc"], P)
    out = bfv.centered(conv.read_scalar_outputs(logits, sk), P.p) % P.p
    act2pc.check_deferred_budgets(P, residuals[:k])
    return out


def config_layers(name: str):
    return stacks.CONFIGS[name]()
