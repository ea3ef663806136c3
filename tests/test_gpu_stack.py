"""Parity of the STACKED tensor-core launch — the path bench.py times.

conv.issue_k1 runs up to 24 independent conv layers as ONE
conv_tc_stack_kernel launch: three rotating digit-plane buffers, relayout
running up to three layers ahead of the GEMM, launch epochs on monotonic
counters and tiles dealt round-robin over the whole stack. Every layer's
output must equal (i) the same layer launched alone (nl = 1, the path the
reference goldens pin in test_gpu_conv.py), (ii) the integer-pipe kernel
(conv_flash_kernel, an independent implementation) and (iii) the C oracle
(oracle/conv_oracle.c, pinned against the reference in
test_oracle_golden.py) on sampled output units — eagerly, on repeated
launches (epochs 1, 2, ...) and as CUDA-graph replays.
Reference: privinfer conv.conv_proposed (conv.py:355-411).
"""

import numpy as np
import pytest
import torch

import bench
from oracle import c_oracle

pytestmark = pytest.mark.gpu


def _layout_dict(lay):
    return {"n": lay.n, "w_p": lay.w_p, "tile": lay.tile, "c_n": lay.c_n, "frags": lay.frags}


def _oracle_check(P, L, out, rng, k=3):
    lay, spec = L["layout"], L["spec"]
    n_out = L["plan"].n_out
    sel = np.unique(np.concatenate([[0, n_out - 1], rng.integers(0, n_out, k)]))
    src, step, fstride = c_oracle.conv_terms(_layout_dict(lay), spec.c_i, spec.f_w)
    want = c_oracle.conv(P.q, P.n, L["host"], spec.weights.reshape(spec.c_o, -1), src, step, lay.frags, fstride,
                         threads=8, units=sel)
    got = out[torch.from_numpy(sel).cuda()].cpu().numpy()
    assert np.array_equal(got, want), f"{L['layer'].name}: stacked output differs from the C oracle"


def _compare(layers, refs, tag):
    bad = []
    for k, (L, r) in enumerate(zip(layers, refs)):
        if not torch.equal(L["out"], r):
            rows = (L["out"] != r).reshape(L["out"].shape[0], -1).any(1).nonzero().flatten().tolist()
            o = L["out"].reshape(L["out"].shape[0], -1)
            untouched = int((o == -1).all(1).sum())
            diff = int((L["out"] != r).sum())
            dpos = (L["out"] != r).reshape(L["out"].shape[0], 2, -1).any(0)  # [2, n] positions differing in any ct
            spans = []
            for p in range(2):
                idx = dpos[p].nonzero().flatten().tolist()
                if idx:
                    spans.append(f"poly {p}: {len(idx)} slots in [{idx[0]}, {idx[-1]}]")
            bad.append(f"#{k} {L['layer'].name} ({'; '.join(spans)}): "
                       f"{len(rows)} of {L['out'].shape[0]} output cts differ (first {rows[:4]}), "
                       f"{diff} coefficients, {untouched} rows never written, out[0,0,:3]={o[0, :3].tolist()} "
                       f"ref[0,0,:3]={r.reshape(r.shape[0], -1)[0, :3].tolist()}")
    assert not bad, f"{tag}: " + "; ".join(bad)


@pytest.mark.parametrize("workload", ["config4", "config5", "config3"])
def test_stacked_launch_bit_exact(workload):
    from paper_2401_16732_b200 import conv

    P, layers = bench.build_stack(workload, seed=31)
    assert all(L["plan"].path == "tc" for L in layers)
    refs, ints = [], []
    for L in layers:
        refs.append(L["plan"].run(L["dev"], torch.empty_like(L["out"])))  # nl = 1
        ints.append(L["plan"].run(L["dev"], torch.empty_like(L["out"]), path="int"))
    torch.cuda.synchronize()
    for L, r, i in zip(layers, refs, ints):
        assert torch.equal(r, i), f"{L['layer'].name}: tensor-core and integer-pipe K1 differ"
    items = [(L["plan"], L["dev"], None, L["out"]) for L in layers]
    for rep in range(2):  # launch epochs 1 and 2 of this stack's counters
        for L in layers:
            L["out"].fill_(-1)
        conv.issue_k1(items)
        torch.cuda.synchronize()
        _compare(layers, refs, f"eager launch {rep}")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side), torch.cuda.graph(g, stream=side):
        conv.issue_k1(items)
    torch.cuda.current_stream().wait_stream(side)
    for rep in range(2):
        for L in layers:
            L["out"].fill_(-1)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        _compare(layers, refs, f"graph replay {rep}")
    rng = np.random.default_rng(5)
    for L in layers:
        _oracle_check(P, L, L["out"], rng)


def test_two_stacks_beyond_24_layers():
    """More than MAX_STACK jobs: issue_k1 splits them into consecutive
    launches (config 4's 20 layers + config 3's 21 = 41 jobs, 2 launches)
    that share the digit-plane scratch."""
    from paper_2401_16732_b200 import conv

    _, a = bench.build_stack("config4", seed=41)
    _, b = bench.build_stack("config3", seed=42)
    layers = a + b
    from paper_2401_16732_b200 import device

    refs = [L["plan"].run(L["dev"], torch.empty_like(L["out"])) for L in layers]
    for rep in range(3):
        for L in layers:
            L["out"].fill_(-1)
        if rep == 2:  # poison the digit-plane scratch: a stale operand read would now show
            conv.issue_k1([(L["plan"], L["dev"], None, L["out"]) for L in layers])  # (sizes the scratch)
            torch.cuda.synchronize()
            device._scratch[(torch.cuda.current_device(), "conv_tc_x")].fill_(0x5A)
        ev = conv.issue_k1([(L["plan"], L["dev"], None, L["out"]) for L in layers])
        assert len(set(map(id, ev))) == 2
        torch.cuda.synchronize()
        _compare(layers, refs, f"split launch {rep}")


def test_sync_buffer_shared_by_different_stacks():
    """Dynamic tile counters: the last grab of a launch resets each layer's
    counter, so ONE counter buffer can serve stacks with different per-layer
    tile counts in turn (config 4's layers, then config 3's, then config 4's
    again) and every output still equals the single-layer launches."""
    from paper_2401_16732_b200 import conv, device

    sync = device.zeros_i64(conv.SYNC_WORDS)
    stacks = []
    for w, seed in (("config4", 61), ("config3", 62)):
        P, layers = bench.build_stack(w, seed=seed)
        layers = layers[:12]
        refs = [L["plan"].run(L["dev"], torch.empty_like(L["out"])) for L in layers]
        stacks.append((layers, refs))
    for layers, refs in (stacks[0], stacks[1], stacks[0], stacks[1]):
        for L in layers:
            L["out"].fill_(-1)
        conv.run_tc_stack([(L["plan"].tc, L["dev"], L["out"]) for L in layers], sync=sync)
        torch.cuda.synchronize()
        _compare(layers, refs, "shared counter buffer")


@pytest.mark.parametrize("workload", ["config5", "config4"])
def test_stacked_launch_is_linear_at_full_size(workload):
    """A size-independent property at BASELINE's full sizes: the conv core is
    Z_q-linear in the input ciphertexts (conv.py:326-352 is a signed-weight sum
    of DRot-shifted rows), so without bias
        K1(a) + K1(b) == K1(a + b)  (mod q)
    for whole stacks, on every coefficient of every output ciphertext — no
    oracle involved, every layer geometry of the workload at once."""
    from paper_2401_16732_b200 import conv

    P, layers = bench.build_stack(workload, seed=77)
    rng = np.random.default_rng(78)
    outs = []
    others = [torch.from_numpy(rng.integers(0, P.q, L["host"].shape, dtype=np.int64)).cuda() for L in layers]
    sums = [(L["dev"] + b) % P.q for L, b in zip(layers, others)]  # < 2^61: no int64 overflow
    for inputs in ([L["dev"] for L in layers], others, sums):
        res = [torch.full_like(L["out"], -1) for L in layers]
        conv.issue_k1([(L["plan"], x, None, r) for L, x, r in zip(layers, inputs, res)])
        torch.cuda.synchronize()
        outs.append(res)
    for L, ya, yb, ys in zip(layers, *outs):
        assert int(ys.min()) >= 0 and int(ys.max()) < P.q, f"{L['layer'].name}: output not canonical mod q"
        assert torch.equal((ya + yb) % P.q, ys), f"{L['layer'].name}: stacked launch is not linear mod q"
