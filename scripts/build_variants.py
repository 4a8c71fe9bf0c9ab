"""Build kernel variants of the current sources (in parallel) for on-GPU A/B:
python scripts/build_variants.py name=DEF1,DEF2 name2=DEF3 ...  ->  _lib/var_<name>.so"""
import concurrent.futures as cf
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_13972_b200 import _build  # noqa: E402


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(_build.LIB_DIR, f"var_{name}.so")
    _build.build(force=True, out=out, defines=[d for d in defs.split(",") if d])
    return out


if __name__ == "__main__":
    with cf.ThreadPoolExecutor(2) as ex:
        for o in ex.map(one, sys.argv[1:]):
            print(o)
