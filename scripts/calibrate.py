"""Report structural statistics of the synthetic workloads beside the paper's
Table 3 / Table 5 targets.

Mean merged length = 1 (root lane) + number of distinct features on each
root-to-leaf path, averaged over leaves: a property of the generated input,
counted here directly (no code from oracle/ or the product library).
"""
from __future__ import annotations

import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/scripts/", 1)[0])
from synth.configs import WORKLOADS  # noqa: E402


def path_lengths(ens):
    lens = []
    for t in range(ens.n_trees):
        left, right, feat, _, _, _ = ens.tree(t)
        stack = [(0, ())]
        while stack:
            n, fs = stack.pop()
            if left[n] < 0:
                lens.append(1 + len(set(fs)))
            else:
                f = int(feat[n])
                stack.append((int(right[n]), fs + (f,)))
                stack.append((int(left[n]), fs + (f,)))
    return np.array(lens)


def main(names):
    for name in names:
        w = WORKLOADS[name]
        t0 = time.time()
        ens = w.ensemble()
        dt = time.time() - t0
        lens = path_lengths(ens)
        k = lens - 1
        print(f"{name:20s} gen {dt:6.2f}s trees {ens.n_trees} leaves {len(lens)} (paper {w.paper_leaves}) "
              f"mean_len {lens.mean():.3f} (paper {w.paper_mean_len}) max_len {lens.max()} "
              f"E[k^2]/k^2 {np.mean(k.astype(float)**2) / max(k.mean(), 1e-9)**2:.3f} "
              f"LB bins {int(np.ceil(lens.sum() / 32))} (paper BFD {w.paper_bfd_bins})")


if __name__ == "__main__":
    main(sys.argv[1:] or list(WORKLOADS))
