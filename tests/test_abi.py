"""The C-ABI library builds, loads and exports every function include/nirvana_cache.h declares
(no GPU: no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nirvana_cache.h")
HEADERS = sorted(os.path.join(ROOT, "include", f) for f in os.listdir(os.path.join(ROOT, "include"))
                 if f.endswith(".h"))


def _declared():
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        src = re.sub(r"#define[^\n]*", "", src)
        names |= set(re.findall(r"\b(cache_\w+)\s*\(", src))
    return sorted(names)


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


def test_struct_layouts_match_the_binding(tmp_path):
    """sizeof / offsetof of every ABI struct, printed by a C program compiled against the
    header, equal the ctypes mirrors in the binding."""
    from paper_2312_04429_b200 import binding as B
    structs = {"cache_config": B.CacheConfig, "cache_stats_t": B.CacheStats, "cache_peer_desc": B.PeerDesc}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "nirvana_cache.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    lines += ['printf("cache_shard_rec size %zu\\n", sizeof(cache_shard_rec));',
              'printf("cache_evict_state size %zu\\n", sizeof(cache_evict_state));', "return 0; }"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           str(src), "-o", str(exe)])
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        *k, v = ln.split()
        got[tuple(k)] = int(v)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f, _ in py._fields_:
            assert got[(cname, f)] == getattr(py, f).offset, (cname, f)
    assert got[("cache_shard_rec", "size")] == B.SHARD_REC_BYTES == 16
    assert got[("cache_evict_state", "size")] == B.EVICT_STATE_BYTES
