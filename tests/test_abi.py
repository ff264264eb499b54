"""The C-ABI library builds, loads and exports every function include/nirvana_cache.h declares
(no GPU: no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nirvana_cache.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cache_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2312_04429_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = _declared()
    for fn in ("cache_create", "cache_insert", "cache_query_batch", "cache_evict", "cache_destroy"):
        assert fn in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for fn in _declared():
        assert hasattr(lib, fn), fn
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (cache_\w+)", out))
    assert set(_declared()) <= exported


def test_binding_loads_and_default_config(libpath):
    from paper_2312_04429_b200 import binding
    cfg = binding.default_config()
    assert cfg.dim == 768 and cfg.num_k == 5 and list(cfg.k_values)[:5] == [5, 10, 15, 20, 25]
    assert list(cfg.thresholds)[:5] == [0.65, 0.75, 0.85, 0.90, 0.95]
    assert cfg.latent_bytes == 32768
    assert binding.lib().cache_last_error() is not None


def test_library_is_sm100a_code(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_rejects_bad_config_without_gpu(libpath):
    from paper_2312_04429_b200 import binding
    cfg = binding.default_config(dim=100, entry_capacity=10, latent_capacity=10)
    h = ctypes.c_void_p()
    rc = binding.lib().cache_create(ctypes.byref(cfg), 0, ctypes.byref(h))
    assert rc == binding.E_DIM and not h.value
