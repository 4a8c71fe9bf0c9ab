"""B200-native exact path-wise TreeShap (GPUTreeShap, arXiv 2010.13972).

The hot path sits behind the C ABI of include/gts.h (libgts.so, built in-tree
by ``_build.build()``); ``gts`` is its thin ctypes binding with the same names,
``TreeShapExplainer`` the model-bound convenience API.
"""
from . import gts  # noqa: F401
from .gts import (gts_binpack, gts_blob_plan, gts_blob_write, gts_extract_paths,  # noqa: F401
                  gts_shap, gts_shap_and_interactions, gts_shap_interactions)

__all__ = ["gts", "gts_extract_paths", "gts_binpack", "gts_blob_plan", "gts_blob_write", "gts_shap",
           "gts_shap_interactions", "gts_shap_and_interactions", "TreeShapExplainer"]


def __getattr__(name):
    if name == "TreeShapExplainer":
        from .explainer import TreeShapExplainer
        return TreeShapExplainer
    raise AttributeError(name)
