"""Per-request timing of inference.he_forward_many for 1 and R requests (development probe)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2401_16732_b200 import bfv, inference, params  # noqa: E402

P = params.default_params()
name = sys.argv[1] if len(sys.argv) > 1 else "config5"
layers = inference.config_layers(name)
convs = inference._convs(layers)
rng = np.random.default_rng(77)
weights = inference.random_weights(layers, rng)
specs = inference.layer_specs(layers, weights)
sk = bfv.keygen(P, np.random.default_rng(78))
for reqs in [1, 1, 4, 8]:
    rng = np.random.default_rng(90)
    xs = [rng.integers(0, 8, (convs[0].c_i, convs[0].H, convs[0].W), dtype=np.int64) for _ in range(reqs)]
    t = {}
    inference.he_forward_many(layers, xs, weights, sk, rng, P, timings=t, specs=specs)
    print(reqs, {k: round(v * 1e3 / reqs, 2) for k, v in t.items() if k.endswith("_s") and not isinstance(v, list)})
t = {}
x = xs[0]
inference.he_forward(layers, x, weights, sk, rng, P, timings=t, specs=specs)
print("single", {k: round(v * 1e3, 2) for k, v in t.items() if k.endswith("_s") and not isinstance(v, list)})
