"""Small invocations of every kernel family for compute-sanitizer runs
(memcheck / synccheck / racecheck): K1-TC single and stacked launches (with
rep 2/4 position groups, tap folding, fragments, bias), K1 integer pipes,
pool, NTT row and split kernels, hoisted key switch (per-step and
multi-step), the fused conventional conv, and one act2pc layer exchange.
Each result is compared against an independent path so a sanitizer run also
checks values. Development tool (profiles/r02_sanitizer_*.txt)."""

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2401_16732_b200 import _native, act2pc, bfv, conv, device, params  # noqa: E402


def main():
    P = params.default_params()
    rng = np.random.default_rng(3)
    jobs = []
    for H, f_w, c_i, c_o, bias in ((32, 3, 3, 16, False), (16, 3, 8, 8, True), (8, 3, 40, 130, False),
                                   (64, 3, 4, 3, True), (32, 1, 16, 32, False)):
        lay = conv.layout_direct(P, H, H, f_w)
        w = rng.integers(-127, 128, (c_o, c_i, f_w, f_w))
        b = rng.integers(-50, 50, c_o) if bias else None
        spec = conv.ConvLayerSpec(H, H, f_w, c_i, c_o, w, bias=b)
        plan = conv.conv_plan(spec, lay, P)
        inp = torch.from_numpy(rng.integers(0, P.q, (lay.ct_count(c_i), 2, P.n))).cuda()
        tc = plan.run(inp, path="tc") if plan.tc is not None else None
        it = plan.run(inp, path="int")
        assert tc is None or torch.equal(tc, it), (H, f_w, c_i, c_o)
        if plan.tc is not None:
            jobs.append((plan, inp, None, torch.empty_like(it), it))
    conv.issue_k1([j[:4] for j in jobs])  # one stacked launch
    torch.cuda.synchronize()
    for j in jobs:
        assert torch.equal(j[3], j[4])
    print("K1: tc == int on", len(jobs), "layers, stacked launch ok")
    # NTT (row kernel n=2048, split kernel n=16384) round trips
    for n in (2048, 16384):
        q = P.q if n == 2048 else params.limb_primes(n, params.find_plaintext_modulus(n), 1)[0]
        x = torch.from_numpy(rng.integers(0, q, (3, n))).cuda()
        y, z = torch.empty_like(x), torch.empty_like(x)
        pl = device.plan_array(n, [q])
        _native.call("fhe_ntt_forward", pl, 1, 3, 1, x.data_ptr(), y.data_ptr(), device.stream())
        _native.call("fhe_ntt_inverse", pl, 1, 3, 1, y.data_ptr(), z.data_ptr(), device.stream())
        assert torch.equal(x, z)
    print("NTT round trips ok")
    # key switch: hrot_many (multi-step kernel) vs per-step keyswitch_rows
    sk = bfv.keygen(P, rng)
    steps = [1, 2, 5]
    swk = bfv.gen_switching_keys(sk, steps, rng)
    t = torch.from_numpy(rng.integers(0, P.q, (3, 2, P.n))).cuda()
    dig = bfv.key_digits_rows(t[:, 1].contiguous(), P, swk.decomp_log, 4)
    multi = bfv.keyswitch_rows_multi(t, dig, steps, swk)
    for s, m in zip(steps, multi):
        assert torch.equal(m, bfv.keyswitch_rows(t, dig, s, swk))
    print("key switch multi == per-step")
    # act2pc layer exchange
    a = rng.integers(-20, 20, (2, 8, 8))
    x = conv.pack_input(a, P, 3, lambda pt: bfv.encrypt_private(pt, sk, rng))
    rp = act2pc.RepackPlan(x.layout, 2, conv.layout_direct(P, 8, 8, 3), P)
    out = act2pc.run_layer_activation(x, act2pc.offline_prepare_layer(rp, P, rng), sk,
                                      bfv.precompute_zero_rows(sk, rng, 3 * rp.k_dst), P, graph=False)
    assert np.array_equal(conv.unpack(out, sk), bfv.centered(a * a + a, P.p))
    print("act2pc layer ok")
    # pool
    lay8 = conv.replace(conv.layout_direct(P, 8, 8, 3), c_n=1)
    xs = conv.PackedTensor(bfv.cts_from_rows(torch.from_numpy(rng.integers(0, P.q, (4, 2, P.n))).cuda(), P.q,
                                             bfv.Encoding.DIRECT, bfv.Domain.COEFF), lay8, 4)
    conv.avg_pool(xs, 8, P)
    torch.cuda.synchronize()
    print("sanitize smoke ok")


if __name__ == "__main__":
    main()
