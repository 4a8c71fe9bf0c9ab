"""Small invocations of every kernel for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): configs[0] (single depth-3 tree) and cal_housing-small,
both layouts, fp32 / fp64, SHAP, interactions and the fused call, plus a
ragged row count and the wide-slot (covtype-shaped, 54 features) SHAP kernel
on a 40-tree subset.  Exits non-zero if any result is not finite.

usage: compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2010_13972_b200 import TreeShapExplainer  # noqa: E402
from synth.configs import WORKLOADS  # noqa: E402


def main():
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cases = [("depth3-single", None, 100), ("cal_housing-small", None, 77)]
    n_calls = 0
    for name, _, n in cases:
        w = WORKLOADS[name]
        ens = w.ensemble()
        x = w.x(n, ens=ens)
        for layout in ("nodal", "warp_bins"):
            for dtype in ("f32", "f64"):
                ex = TreeShapExplainer(ens, dtype=dtype, layout=layout, device=dev)
                xd = torch.from_numpy(x).to(dev, ex.torch_dtype)
                outs = [ex.shap_device(xd), ex.interactions_device(xd), *ex.shap_and_interactions_device(xd)]
                torch.cuda.synchronize()
                n_calls += 3
                for o in outs:
                    assert torch.isfinite(o).all(), (name, layout, dtype)
    # wide identity map (54 features, 64-slot SHAP kernel) and per-chunk maps (fashion, 32 slots)
    for name, trees in (("covtype-large", 40), ("fashion_mnist-med", 40)):
        w = WORKLOADS[name]
        ens = w.ensemble().subset(range(trees))
        x = w.x(65, ens=ens)
        ex = TreeShapExplainer(ens, dtype="f32", device=dev, interactions=False)
        phi = ex.shap_device(torch.from_numpy(x).to(dev))
        pij = ex.interactions_device(torch.from_numpy(x[:33]).to(dev))
        torch.cuda.synchronize()
        n_calls += 2
        assert torch.isfinite(phi).all() and torch.isfinite(pij).all(), name
    print(f"sanitize cases ok: {n_calls} calls")


if __name__ == "__main__":
    main()
