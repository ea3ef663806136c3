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


@pytest.mark.parametrize("name", ["config3", "config5"])
def test_chain_online_phase_matches(name):
    """he_prepare (the offline phase up front) + he_forward_online (no host
    synchronisation until the logits; budget checks deferred) equals the
    integer model; a second inference prepares fresh material."""
    from paper_2401_16732_b200 import bfv, conv, inference, params

    P = params.default_params()
    rng = np.random.default_rng(31 + len(name))
    layers = inference.config_layers(name)
    seq, pool, fc = inference.main_path(layers)
    weights = inference.random_weights(layers, rng)
    specs = inference.layer_specs(layers, weights)
    sk = bfv.keygen(P, rng)
    for _ in range(2):
        x = rng.integers(0, 8, (seq[0].c_i, seq[0].H, seq[0].W), dtype=np.int64)
        prepared = inference.he_prepare(layers, P, sk, rng)
        cur = conv.pack_input_private(x, P, seq[0].f_w, sk, rng)
        got = inference.he_forward_online(layers, cur, weights, sk, P, prepared, specs=specs)
        assert np.array_equal(got, inference.plain_forward(layers, x, weights, P.p))


def test_deferred_budget_check_raises():
    """A stored residual above the budget makes the deferred check raise the
    per-round check's ProtocolError."""
    import torch

    from paper_2401_16732_b200 import act2pc, params
    from paper_2401_16732_b200.errors import ProtocolError

    P = params.default_params()
    ok = torch.tensor([1, 5, 3], dtype=torch.int64, device="cuda")
    act2pc.check_deferred_budgets(P, ok)
    bad = torch.tensor([1, P.q // (2 * P.p) * 4, 3], dtype=torch.int64, device="cuda")
    with pytest.raises(ProtocolError):
        act2pc.check_deferred_budgets(P, bad)


def test_pack_input_private_matches_per_ciphertext_encryption():
    """conv.pack_input_private (batched encryptions) equals pack_input with
    encrypt_private per ciphertext on the same rng: identical ciphertexts and
    the same rng state afterwards."""
    from paper_2401_16732_b200 import bfv, conv, params

    P = params.default_params()
    sk = bfv.keygen(P, np.random.default_rng(5))
    x = np.random.default_rng(6).integers(0, 8, (3, 56, 56), dtype=np.int64)
    r1, r2 = np.random.default_rng(9), np.random.default_rng(9)
    a = conv.pack_input(x, P, 7, lambda pt: bfv.encrypt_private(pt, sk, r1))
    b = conv.pack_input_private(x, P, 7, sk, r2)
    assert a.layout == b.layout and a.channels == b.channels
    assert np.array_equal(bfv.cts_rows(a.cts).cpu().numpy(), bfv.cts_rows(b.cts).cpu().numpy())
    assert r1.integers(0, 1 << 62) == r2.integers(0, 1 << 62)


def test_chain_main_path_only_matches():
    """residual=False keeps the main-path-only chain (no shortcut additions)
    and equals the integer model without them."""
    from paper_2401_16732_b200 import bfv, inference, params

    P = params.default_params()
    rng = np.random.default_rng(4040)
    layers = inference.config_layers("config3")
    seq, pool, fc = inference.main_path(layers)
    weights = inference.random_weights(layers, rng)
    sk = bfv.keygen(P, rng)
    x = rng.integers(0, 8, (seq[0].c_i, seq[0].H, seq[0].W), dtype=np.int64)
    got = inference.he_forward(layers, x, weights, sk, rng, P, residual=False)
    assert np.array_equal(got, inference.plain_forward(layers, x, weights, P.p, residual=False))
    assert not np.array_equal(got, inference.plain_forward(layers, x, weights, P.p))
