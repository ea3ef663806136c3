"""Configs 3, 4 and 5 end to end on the device (inference.py): conv -> x²+x
(shares, client repack, stride) -> ... [-> 2x2 pool -> masked repack round]
-> ... -> avg_pool -> FC, decrypted logits equal to the integer model mod p."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["config3", "config4", "config5"])
def test_chain_matches_integer_model(name):
    from paper_2401_16732_b200 import bfv, inference, params

    P = params.default_params()
    rng = np.random.default_rng(2024 + len(name))
    layers = inference.config_layers(name)
    seq, pool, fc = inference.main_path(layers)
    weights = inference.random_weights(layers, rng)
    sk = bfv.keygen(P, rng)
    x = rng.integers(0, 8, (seq[0].c_i, seq[0].H, seq[0].W), dtype=np.int64)
    got = inference.he_forward(layers, x, weights, sk, rng, P)
    want = inference.plain_forward(layers, x, weights, P.p)
    assert got.shape == (fc.c_o,)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name,reqs", [("config3", 3), ("config5", 2)])
def test_chain_many_requests(name, reqs):
    """he_forward_many: the same conv layer of several requests in one stacked
    tensor-core launch per layer; every request's logits equal the integer model."""
    from paper_2401_16732_b200 import bfv, inference, params

    P = params.default_params()
    rng = np.random.default_rng(77 + reqs)
    layers = inference.config_layers(name)
    seq, pool, fc = inference.main_path(layers)
    weights = inference.random_weights(layers, rng)
    sk = bfv.keygen(P, rng)
    xs = [rng.integers(0, 8, (seq[0].c_i, seq[0].H, seq[0].W), dtype=np.int64) for _ in range(reqs)]
    got = inference.he_forward_many(layers, xs, weights, sk, rng, P)
    for x, g in zip(xs, got):
        assert np.array_equal(g, inference.plain_forward(layers, x, weights, P.p))
