"""The five BASELINE.json workloads (configs[0..4]) as synthetic-input recipes.

Shapes follow the paper's models (Table 3: trees, leaves,
max depth) and datasets (Table 2: features, classes).  The
two growth knobs (Zipf skew ``zipf_s`` of the split-feature choice and depth
bias ``beta``) are calibrated so the mean merged path length (root included)
lands within +-3% of the Table 5 "none" utilisation x 32;
scripts/calibrate.py reports the achieved values.
"""
from __future__ import annotations

from dataclasses import dataclass

from . import Ensemble, inject_ties, make_ensemble, make_x


@dataclass(frozen=True)
class Workload:
    name: str
    n_trees: int
    n_groups: int
    n_features: int
    max_depth: int
    leaves_per_tree: float
    zipf_s: float
    beta: float
    seed: int
    rows: int  # rows used by the parity tests / SURVEY §8(d)
    paper_mean_len: float | None  # Table 5 "none" util x 32 (root included)
    paper_leaves: int | None  # Table 3
    paper_bfd_bins: int | None  # Table 5
    tie_frac: float = 0.0
    note: str = ""

    def ensemble(self) -> Ensemble:
        return make_ensemble(self.n_trees, self.n_features, self.max_depth, self.leaves_per_tree,
                             n_groups=self.n_groups, zipf_s=self.zipf_s, beta=self.beta, seed=self.seed)

    def x(self, n_rows: int | None = None, row0: int = 0, ens: Ensemble | None = None):
        n = self.rows if n_rows is None else n_rows
        x = make_x(self.seed * 7919 + 17, n, self.n_features, row0)
        if self.tie_frac > 0.0:
            if ens is None:
                ens = self.ensemble()
            x = inject_ties(x, ens, self.tie_frac, self.seed * 104729 + row0)
        return x


WORKLOADS = {
    # configs[0]: single depth-3 tree, 8 features, 100 rows, vs brute force
    "depth3-single": Workload("depth3-single", 1, 1, 8, 3, 8, zipf_s=1.5, beta=0.0, seed=1, rows=100,
                              paper_mean_len=None, paper_leaves=None, paper_bfd_bins=None, tie_frac=0.1,
                              note="complete depth-3 tree; >=10% of X entries equal a split threshold"),
    # configs[1]: cal_housing-shaped small / med
    "cal_housing-small": Workload("cal_housing-small", 10, 1, 8, 3, 8, zipf_s=2.6, beta=0.0, seed=2,
                                  rows=10_000, paper_mean_len=0.085938 * 32, paper_leaves=80,
                                  paper_bfd_bins=7),
    "cal_housing-med": Workload("cal_housing-med", 100, 1, 8, 8, 216.43, zipf_s=0.75, beta=0.0, seed=3,
                                rows=10_000, paper_mean_len=0.181457 * 32, paper_leaves=21_643,
                                paper_bfd_bins=4_170),
    # configs[2]
    "adult-large": Workload("adult-large", 1000, 1, 14, 16, 642.035, zipf_s=0.0, beta=0.1, seed=4,
                            rows=10_000, paper_mean_len=0.297131 * 32, paper_leaves=642_035,
                            paper_bfd_bins=200_152),
    # configs[3]
    "fashion_mnist-med": Workload("fashion_mnist-med", 1000, 10, 784, 8, 144.154, zipf_s=0.5, beta=0.0,
                                  seed=5, rows=10_000, paper_mean_len=0.264387 * 32, paper_leaves=144_154,
                                  paper_bfd_bins=43_313),
    # configs[4]
    "covtype-large": Workload("covtype-large", 8000, 8, 54, 16, 829.555, zipf_s=1.0, beta=0.0, seed=6,
                              rows=1_048_576, paper_mean_len=0.299913 * 32, paper_leaves=6_636_440,
                              paper_bfd_bins=2_109_830),
}
