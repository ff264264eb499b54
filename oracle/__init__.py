"""fp64 CPU oracle of the NIRVANA cache lookup (arXiv 2312.04429) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_2312_04429_b200`` never imports it and shares no code with it.

The arithmetic lives in ``nirvana_oracle.c`` (plain C, fp64, index-order sums, no FMA
contraction); this module is only a ctypes marshaller around it.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "nirvana_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, E_INVALID_ARG, E_FULL, E_EVICT_RANGE, E_BAD_ROWS, E_OOM = 0, 1, 3, 4, 5, 8
LCBFU, LRU, LFU, FIFO = 0, 1, 2, 3   # eviction policies
ROW_OK, ROW_NONFINITE, ROW_ZERO_NORM, ROW_NO_ITEMS = 0, 1, 2, 3
NO_ID = np.uint64(0xFFFFFFFFFFFFFFFF)

PAPER_K_VALUES = (5, 10, 15, 20, 25)
PAPER_THRESHOLDS = (0.65, 0.75, 0.85, 0.90, 0.95)  # Fig. 11


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2 -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P, I64, I32, U64, D = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_uint64, ctypes.c_double
        L.oracle_create.restype = P
        L.oracle_create.argtypes = [I32, I64, I64, I64, I32, P, P, I32]
        L.oracle_destroy.argtypes = [P]
        L.oracle_insert.argtypes = [P, I64, P, I32, P, P, P, P]
        L.oracle_query.argtypes = [P, I64, P, I32, I32, P, P, P, P, P, P, P, I32]
        L.oracle_record_access.argtypes = [P, I64, P, P]
        L.oracle_set_count.argtypes = [P, U64, ctypes.c_int32, U64]
        L.oracle_score_id.argtypes = [P, P, I32, U64]
        L.oracle_score_id.restype = D
        L.oracle_evict.argtypes = [P, I64, P, P, P]
        L.oracle_evict_policy.argtypes = [P, I64, I32, P, P, P]
        L.oracle_evict_entries.argtypes = [P, I64, I32, P]
        L.oracle_tick.argtypes = [P]
        L.oracle_tick.restype = None
        L.oracle_clock.argtypes = [P]
        L.oracle_clock.restype = U64
        L.oracle_get_last.argtypes = [P, U64, P]
        L.oracle_live_entries.argtypes = [P]
        L.oracle_live_entries.restype = I64
        L.oracle_live_items.argtypes = [P]
        L.oracle_live_items.restype = I64
        L.oracle_next_id.argtypes = [P]
        L.oracle_next_id.restype = U64
        L.oracle_get_row.argtypes = [P, U64, P]
        L.oracle_get_meta.argtypes = [P, U64, P, P]
        L.oracle_bf16_round.argtypes = [D]
        L.oracle_bf16_round.restype = D
        L.oracle_normalise.argtypes = [I32, P, P]
        L.oracle_select_k.argtypes = [P, D]
        L.oracle_select_k.restype = I32
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def bf16_round(v: float) -> float:
    return lib().oracle_bf16_round(float(v))


def normalise(x) -> tuple[int, np.ndarray]:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros_like(x)
    st = lib().oracle_normalise(x.shape[0], _p(x), _p(y))
    return st, y


class OracleCache:
    """ctypes handle around ``oracle_cache`` (host memory, synchronous)."""

    def __init__(self, dim=768, entry_capacity=1024, latent_capacity=None, latent_bytes=0,
                 k_values=PAPER_K_VALUES, thresholds=PAPER_THRESHOLDS, k_bias=0):
        self.dim = dim
        self.num_k = len(k_values)
        self.k_values = tuple(int(k) for k in k_values)
        self.latent_bytes = int(latent_bytes)
        if latent_capacity is None:
            latent_capacity = entry_capacity * self.num_k
        kv = np.asarray(k_values, dtype=np.int32)
        th = np.asarray(thresholds, dtype=np.float64)
        self._h = lib().oracle_create(dim, entry_capacity, latent_capacity, latent_bytes,
                                      self.num_k, _p(kv), _p(th), k_bias)
        if not self._h:
            raise ValueError("oracle_create rejected the configuration")

    def close(self):
        if self._h:
            lib().oracle_destroy(self._h)
            self._h = None

    __del__ = close

    def insert(self, emb, latents=None, present=None, emb_is_bf16=False):
        emb = np.ascontiguousarray(emb, dtype=np.uint16 if emb_is_bf16 else np.float32)
        n = emb.shape[0]
        lat = None if latents is None else np.ascontiguousarray(latents, dtype=np.uint8)
        pr = None if present is None else np.ascontiguousarray(present, dtype=np.uint8)
        ids = np.empty(n, dtype=np.uint64)
        st = np.empty(n, dtype=np.int32)
        rc = lib().oracle_insert(self._h, n, _p(emb), int(emb_is_bf16), _p(lat), _p(pr), _p(ids), _p(st))
        return rc, ids, st

    def query(self, q, topk=1, want_latents=True, apply_counters=True, q_is_bf16=False):
        q = np.ascontiguousarray(q, dtype=np.uint16 if q_is_bf16 else np.float32)
        b = q.shape[0]
        ids = np.empty((b, topk), dtype=np.uint64)
        sc = np.empty((b, topk), dtype=np.float64)
        raw = np.empty((b, topk), dtype=np.float64)
        k = np.empty(b, dtype=np.int32)
        kstar = np.empty(b, dtype=np.int32)
        st = np.empty(b, dtype=np.int32)
        lat = np.zeros((b, self.latent_bytes), dtype=np.uint8) if (want_latents and self.latent_bytes) else None
        rc = lib().oracle_query(self._h, b, _p(q), int(q_is_bf16), topk, _p(ids), _p(sc), _p(raw),
                                _p(k), _p(kstar), _p(lat), _p(st), int(apply_counters))
        return dict(rc=rc, ids=ids, scores=sc, raw=raw, k=k, kstar=kstar, status=st, latents=lat)

    def record_access(self, ids, ks):
        ids = np.ascontiguousarray(ids, dtype=np.uint64)
        ks = np.ascontiguousarray(ks, dtype=np.int32)
        return lib().oracle_record_access(self._h, ids.shape[0], _p(ids), _p(ks))

    def score_id(self, qrow, id_, q_is_bf16=False):
        q = np.ascontiguousarray(qrow, dtype=np.uint16 if q_is_bf16 else np.float32)
        return lib().oracle_score_id(self._h, _p(q), int(q_is_bf16), int(id_))

    def evict(self, n, policy=0):
        """policy: 0 LCBFU, 1 LRU, 2 LFU, 3 FIFO."""
        ev = np.empty(max(n, 1), dtype=np.uint64)
        dirty = np.empty(max(n, 1), dtype=np.uint64)
        nd = np.zeros(1, dtype=np.int64)
        rc = lib().oracle_evict_policy(self._h, n, policy, _p(ev), _p(dirty), _p(nd))
        return rc, ev[:n].copy(), dirty[: int(nd[0])].copy()

    def evict_entries(self, n, policy=0):
        """Entry granularity (R24): remove the n entries with the smallest aggregated policy
        score (LCBFU sum f*K, LRU max last, LFU sum f, FIFO 0), ties by id.  Returns (rc, ids)."""
        ids = np.empty(max(n, 1), dtype=np.uint64)
        rc = lib().oracle_evict_entries(self._h, n, policy, _p(ids))
        return rc, ids[:n].copy()

    def set_count(self, id_, j, f):
        """Test hook: access count f of item (id, K_j)."""
        return lib().oracle_set_count(self._h, int(id_), int(j), int(f))

    def tick(self):
        lib().oracle_tick(self._h)

    @property
    def clock(self):
        return lib().oracle_clock(self._h)

    def last(self, id_):
        out = np.empty(self.num_k, dtype=np.uint64)
        if lib().oracle_get_last(self._h, int(id_), _p(out)) != 0:
            raise KeyError(id_)
        return out

    def select_k(self, s):
        return lib().oracle_select_k(self._h, float(s))

    @property
    def live_entries(self):
        return lib().oracle_live_entries(self._h)

    @property
    def live_items(self):
        return lib().oracle_live_items(self._h)

    @property
    def next_id(self):
        return lib().oracle_next_id(self._h)

    def row(self, id_):
        out = np.empty(self.dim, dtype=np.float64)
        if lib().oracle_get_row(self._h, int(id_), _p(out)) != 0:
            raise KeyError(id_)
        return out

    def meta(self, id_):
        f = np.empty(self.num_k, dtype=np.uint64)
        m = np.zeros(1, dtype=np.uint32)
        if lib().oracle_get_meta(self._h, int(id_), _p(f), _p(m)) != 0:
            raise KeyError(id_)
        return f, int(m[0])
