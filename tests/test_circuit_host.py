"""Host-side pieces of the circuit workload (CPU): the executor's generator
hash (torch int64) equals the oracle's (numpy), and the float64 oracle
behaves like the model it restates."""

import numpy as np
import torch

from oracle import circuit as OC
from paper_2507_17087_b200.executors import circuit as C


def test_hash_matches_oracle():
    idx = torch.arange(0, 3_000_000, 7, dtype=torch.int64)
    for salt in (0, 5, 64 * 3 + 9):
        assert np.array_equal(C.hash31(idx, salt).numpy(), OC.hash31(idx.numpy(), salt))


def test_oracle_model_properties():
    # no wires' steps -> currents stay zero, voltages just leak
    v, i = OC.simulate(4, 8, 16, 100, 0, 1e-4, 0, 2)
    gen = OC.generate(4, 8, 16, 100, 0)
    assert np.all(i == 0)
    assert np.allclose(v, gen["v0"] * (1 - gen["leak"]) ** 2)
    # pct_in = 100: every wire stays inside its piece
    g = OC.generate(6, 10, 40, 100, 1)
    assert np.array_equal(g["in_node"] // 10, g["out_node"] // 10)
    # pct_in = 0: every wire crosses to a neighbouring piece
    g = OC.generate(6, 10, 40, 0, 1)
    d = (g["out_node"] // 10 - g["in_node"] // 10) % 6
    assert set(d.tolist()) <= {1, 5}
    v, i = OC.simulate(3, 5, 20, 50, 5, 1e-4, 2, 1)
    assert np.isfinite(v).all() and np.abs(i).max() > 0
