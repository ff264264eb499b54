"""B200-native (sm_100a) NIRVANA cache lookup -- arXiv 2312.04429, "Approximate Caching for
Efficiently Serving Diffusion Models".

The product is ``libnirvana_cache.so`` (C ABI in ``include/nirvana_cache.h``); this package
holds its CUDA sources (``csrc/``), the nvcc build script (``build.py``) and a thin ctypes
binding (``binding.py``).  ``import paper_2312_04429_b200.binding`` requires the built
library: there is no CPU fallback.
"""
import importlib

__all__ = ["binding", "NirvanaCache", "CacheError"]


def __getattr__(name):
    if name in ("binding", "NirvanaCache", "CacheError"):
        mod = importlib.import_module(__name__ + ".binding")
        return mod if name == "binding" else getattr(mod, name)
    raise AttributeError(name)
