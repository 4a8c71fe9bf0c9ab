"""The shared input generators: determinism, shard reproducibility, calibration."""
import numpy as np
import pytest

import synth
from scripts.calibrate import path_lengths
from synth.configs import WORKLOADS


def test_ensemble_deterministic_and_valid():
    a = synth.make_ensemble(20, 6, 6, 30, n_groups=2, zipf_s=1.0, seed=7)
    b = synth.make_ensemble(20, 6, 6, 30, n_groups=2, zipf_s=1.0, seed=7)
    for name in ("node_offset", "left", "right", "feature", "threshold", "cover", "leaf_value", "tree_group"):
        assert np.array_equal(getattr(a, name), getattr(b, name))
    internal = a.left >= 0
    for t in range(a.n_trees):
        lo, hi = a.node_offset[t], a.node_offset[t + 1]
        for j in range(hi - lo):
            g = lo + j
            if a.left[g] >= 0:
                assert a.cover[lo + a.left[g]] + a.cover[lo + a.right[g]] == a.cover[g]
    assert np.all(a.cover > 0)
    assert np.all((a.feature[internal] >= 0) & (a.feature[internal] < 6))
    assert a.tree_group.tolist() == [t % 2 for t in range(20)]


def test_x_shards_reproducible():
    full = synth.make_x(3, 100, 7)
    part = synth.make_x(3, 30, 7, row0=40)
    assert np.array_equal(full[40:70], part)
    assert full.dtype == np.float32 and full.min() >= 0 and full.max() < 1


@pytest.mark.parametrize("name", ["cal_housing-small", "cal_housing-med", "adult-large", "fashion_mnist-med"])
def test_calibration_within_3_percent(name):
    """Mean merged path length within +-3% of Table 5's 'none' utilisation x 32
    (PAPER.md:466-520); leaves within 1% of Table 3."""
    w = WORKLOADS[name]
    ens = w.ensemble()
    lens = path_lengths(ens)
    assert abs(lens.mean() / w.paper_mean_len - 1) < 0.03
    assert abs(len(lens) / w.paper_leaves - 1) < 0.01
