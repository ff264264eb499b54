"""Thin ctypes binding of ``libnirvana_cache.so`` (include/nirvana_cache.h).

Argument marshalling only: every step of the lookup runs in the library's CUDA kernels.
PyTorch provides device memory and streams.  There is no CPU fallback: if the built library
is missing this module raises on import.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnirvana_cache.so")

OK, E_INVALID_ARG, E_DIM, E_FULL, E_EVICT_RANGE, E_BAD_ROWS, E_CUDA, E_NCCL, E_OOM, E_STATE, E_UNSUPPORTED = range(11)
ROW_OK, ROW_NONFINITE, ROW_ZERO_NORM, ROW_NO_ITEMS = range(4)
DTYPE_F32, DTYPE_BF16 = 0, 1
SCORER_AUTO, SCORER_TC, SCORER_STREAM, SCORER_TC_SINGLE = 0, 1, 2, 3
MAX_K, MAX_TOPK = 8, 16
NO_ID = 0xFFFFFFFFFFFFFFFF

_STATUS = {OK: "OK", E_INVALID_ARG: "INVALID_ARG", E_DIM: "DIM", E_FULL: "FULL", E_EVICT_RANGE: "EVICT_RANGE",
           E_BAD_ROWS: "BAD_ROWS", E_CUDA: "CUDA", E_NCCL: "NCCL", E_OOM: "OOM", E_STATE: "STATE",
           E_UNSUPPORTED: "UNSUPPORTED"}


class CacheError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


class CacheConfig(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("entry_capacity", ctypes.c_int64),
                ("latent_capacity", ctypes.c_int64), ("latent_bytes", ctypes.c_int64),
                ("num_k", ctypes.c_int32), ("k_values", ctypes.c_int32 * MAX_K),
                ("thresholds", ctypes.c_double * MAX_K), ("k_bias", ctypes.c_int32),
                ("max_topk", ctypes.c_int32), ("shard_rank", ctypes.c_int32), ("shard_world", ctypes.c_int32),
                ("latent_alias", ctypes.c_int32), ("evict_policy", ctypes.c_int32),
                ("evict_granularity", ctypes.c_int32)]


POLICY_LCBFU, POLICY_LRU, POLICY_LFU, POLICY_FIFO = 0, 1, 2, 3
EVICT_ITEM, EVICT_ENTRY = 0, 1   # eviction granularity (CACHE_EVICT_*)


def alias_slot(id_: int, j: int, cap: int) -> int:
    """CACHE_ALIAS_SLOT of include/nirvana_cache.h (the declared aliasing map)."""
    return ((((int(id_) & 0xFFFFFFFF) * 8 + j) * 2654435761) & 0xFFFFFFFF) % cap


class CacheStats(ctypes.Structure):
    _fields_ = [("live_entries", ctypes.c_int64), ("live_items", ctypes.c_int64), ("holes", ctypes.c_int64),
                ("entry_hwm", ctypes.c_int64), ("next_id", ctypes.c_uint64), ("queries", ctypes.c_int64),
                ("free_entries", ctypes.c_int64), ("free_items", ctypes.c_int64)]


class PeerDesc(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("pid", ctypes.c_int32), ("num_k", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("latent_bytes", ctypes.c_int64), ("lslot", ctypes.c_void_p),
                ("fcnt", ctypes.c_void_p), ("pool", ctypes.c_void_p), ("lastacc", ctypes.c_void_p),
                ("ipc_lslot", ctypes.c_ubyte * 64), ("ipc_fcnt", ctypes.c_ubyte * 64),
                ("ipc_pool", ctypes.c_ubyte * 64), ("ipc_lastacc", ctypes.c_ubyte * 64),
                ("arena", ctypes.c_void_p), ("arena_nb", ctypes.c_int64), ("arena_topk", ctypes.c_int32),
                ("reserved2", ctypes.c_int32), ("ipc_arena", ctypes.c_ubyte * 64),
                ("process_token", ctypes.c_uint64)]


SHARD_REC_BYTES = 16   # cache_shard_rec
EVICT_STATE_BYTES = 24  # cache_evict_state


EXPORTS = ("cache_default_config", "cache_create", "cache_destroy", "cache_insert", "cache_query_batch",
           "cache_query_batch_host", "cache_evict", "cache_get_meta", "cache_get_row", "cache_stats",
           "cache_set_scorer", "cache_set_query_slices", "cache_set_profile_events", "cache_kernel_launches",
           "cache_last_error",
           "cache_evict_hist", "cache_evict_pick", "cache_evict_apply", "cache_live_items", "cache_query_local",
           "cache_query_merge", "cache_export_peer", "cache_attach_peers", "cache_pool_write",
           "cache_set_evict_policy", "cache_predictor_train", "cache_predict", "cache_predictor_get",
           "cache_set_evict_granularity", "cache_live_entries", "cache_push_reserve", "cache_push_queries",
           "cache_push_scan", "cache_push_merge", "cache_push_evict_hist", "cache_push_evict_pick",
           "cache_push_evict_apply", "cache_profile_thresholds", "cache_set_thresholds", "cache_query_peek",
           "cache_push_status", "cache_set_peer_timeout", "cache_last_evicted_keys",
           "cache_evict_view", "cache_query_submit", "cache_query_complete", "cache_evict_sel_begin",
           "cache_evict_sel_level", "cache_evict_sel_pick", "cache_evict_sel_apply", "cache_push_evict_sel_level",
           "cache_push_evict_sel_pick", "cache_get_config", "cache_save", "cache_load")


def load_library(path: str = LIB_PATH):
    if not os.path.exists(path):
        raise ImportError(f"CUDA library {path} is missing: run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P, I64, I32, U64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64
    L.cache_default_config.argtypes = [ctypes.POINTER(CacheConfig)]
    L.cache_create.argtypes = [ctypes.POINTER(CacheConfig), ctypes.c_int, ctypes.POINTER(P)]
    L.cache_destroy.argtypes = [P]
    L.cache_get_config.argtypes = [P, ctypes.POINTER(CacheConfig)]
    L.cache_get_config.restype = ctypes.c_int
    L.cache_save.argtypes = [P, ctypes.c_char_p, I32]
    L.cache_save.restype = ctypes.c_int
    L.cache_load.argtypes = [ctypes.c_char_p, I32, ctypes.POINTER(P)]
    L.cache_load.restype = ctypes.c_int
    L.cache_insert.argtypes = [P, I64, P, I32, P, P, P, P, P]
    L.cache_query_batch.argtypes = [P, I64, P, I32, I32, P, P, P, P, P, P, P]
    L.cache_query_batch_host.argtypes = [P, I64, P, I32, I32, P, P, P, P, P, P]
    L.cache_query_peek.argtypes = [P, I64, P, I32, I32, P, P, P, P, P]
    L.cache_query_peek.restype = ctypes.c_int
    L.cache_evict_sel_begin.argtypes = [P, I64, P]
    L.cache_evict_sel_level.argtypes = [P, I32, P, P]
    L.cache_evict_sel_pick.argtypes = [P, I32, P, P, P]
    L.cache_evict_sel_apply.argtypes = [P, I64, P, P, P, P, P]
    L.cache_push_evict_sel_level.argtypes = [P, I32, P]
    L.cache_push_evict_sel_pick.argtypes = [P, I32, P, P]
    for fn in ("cache_evict_sel_begin", "cache_evict_sel_level", "cache_evict_sel_pick", "cache_evict_sel_apply",
               "cache_push_evict_sel_level", "cache_push_evict_sel_pick"):
        getattr(L, fn).restype = ctypes.c_int
    L.cache_query_submit.argtypes = [P, I32, I64, P, I32, I32, P, P]
    L.cache_query_submit.restype = ctypes.c_int
    L.cache_query_complete.argtypes = [P, I32, P, P, P, P]
    L.cache_query_complete.restype = ctypes.c_int
    L.cache_evict_view.argtypes = [P, I64, P, P, P, P]
    L.cache_evict_view.restype = ctypes.c_int
    L.cache_last_evicted_keys.argtypes = [P, P, I64, P]
    L.cache_last_evicted_keys.restype = ctypes.c_int
    L.cache_push_status.argtypes = [P, P]
    L.cache_push_status.restype = ctypes.c_int
    L.cache_set_peer_timeout.argtypes = [P, I64]
    L.cache_set_peer_timeout.restype = ctypes.c_int
    L.cache_evict.argtypes = [P, I64, P, P, P, P]
    L.cache_get_meta.argtypes = [P, U64, P, P]
    L.cache_get_row.argtypes = [P, U64, P]
    L.cache_stats.argtypes = [P, ctypes.POINTER(CacheStats)]
    L.cache_set_scorer.argtypes = [P, I32]
    L.cache_set_query_slices.argtypes = [P, I32]
    L.cache_set_evict_policy.argtypes = [P, I32]
    L.cache_set_evict_policy.restype = ctypes.c_int
    L.cache_set_profile_events.argtypes = [P, P]
    L.cache_evict_hist.argtypes = [P, P, I32, P, P]
    L.cache_evict_pick.argtypes = [P, P, P, I32, P]
    L.cache_evict_apply.argtypes = [P, P, I64, P, P, P, P, P]
    L.cache_live_items.argtypes = [P]
    L.cache_live_items.restype = I64
    L.cache_live_entries.argtypes = [P]
    L.cache_live_entries.restype = I64
    L.cache_push_reserve.argtypes = [P, I64, I32]
    L.cache_push_queries.argtypes = [P, I64, P, I32, P]
    L.cache_push_scan.argtypes = [P, I64, I32, P]
    L.cache_push_merge.argtypes = [P, I64, I32, P, P, P, P, P, P, P]
    L.cache_profile_thresholds.argtypes = [P, I64, P, I32, P, ctypes.c_double, P, P, P]
    L.cache_set_thresholds.argtypes = [P, P]
    L.cache_push_evict_hist.argtypes = [P, I64, I32, P]
    L.cache_push_evict_pick.argtypes = [P, I32, P]
    L.cache_push_evict_apply.argtypes = [P, I64, P, P, P, P, P]
    L.cache_set_evict_granularity.argtypes = [P, I32]
    L.cache_set_evict_granularity.restype = ctypes.c_int
    L.cache_query_local.argtypes = [P, I64, P, I32, I32, P, P]
    L.cache_query_merge.argtypes = [P, I64, I64, I64, I32, P, P, P, P, P, P, P, P]
    L.cache_export_peer.argtypes = [P, ctypes.POINTER(PeerDesc)]
    L.cache_pool_write.argtypes = [P, I64, I64, P, P]
    L.cache_pool_write.restype = ctypes.c_int
    L.cache_predictor_train.argtypes = [P, ctypes.c_double, I32, ctypes.c_double, P]
    L.cache_predict.argtypes = [P, I64, P, I32, P, P, P]
    L.cache_predictor_get.argtypes = [P, P, P]
    for fn in ("cache_predictor_train", "cache_predict", "cache_predictor_get"):
        getattr(L, fn).restype = ctypes.c_int
    L.cache_attach_peers.argtypes = [P, I32, P]
    for fn in ("cache_evict_hist", "cache_evict_pick", "cache_evict_apply", "cache_query_local",
               "cache_query_merge", "cache_export_peer", "cache_attach_peers"):
        getattr(L, fn).restype = ctypes.c_int
    L.cache_kernel_launches.argtypes = [P]
    L.cache_kernel_launches.restype = I64
    L.cache_last_error.restype = ctypes.c_char_p
    for fn in ("cache_create", "cache_destroy", "cache_insert", "cache_query_batch", "cache_query_batch_host",
               "cache_evict", "cache_get_meta", "cache_get_row", "cache_stats", "cache_set_scorer",
               "cache_set_query_slices", "cache_set_profile_events"):
        getattr(L, fn).restype = ctypes.c_int
    return L


_lib = load_library()


def lib():
    return _lib


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return ctypes.c_void_p(t.data_ptr())
    return t.ctypes.data_as(ctypes.c_void_p)


def _stream(stream):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _check(rc, allow=()):
    if rc != OK and rc not in allow:
        raise CacheError(rc, _lib.cache_last_error().decode())
    return rc


def default_config(**kw) -> CacheConfig:
    cfg = CacheConfig()
    _lib.cache_default_config(ctypes.byref(cfg))
    for k, v in kw.items():
        if k in ("k_values", "thresholds"):
            arr = getattr(cfg, k)
            for i, x in enumerate(v):
                arr[i] = x
            if k == "k_values":
                cfg.num_k = len(v)
        else:
            setattr(cfg, k, v)
    return cfg


class _ArrIface:
    """A read-only numpy view of library memory through __array_interface__ (np.ctypeslib's
    as_array builds a new ctypes array type per length: tens of microseconds per call)."""
    __slots__ = ("__array_interface__",)

    def __init__(self, addr: int, k: int):
        self.__array_interface__ = {"data": (addr, True), "shape": (k,), "typestr": "<u8", "version": 3}


def _u64_view(addr, k: int) -> np.ndarray:
    if k == 0 or not addr:
        return np.zeros(0, np.uint64)
    return np.asarray(_ArrIface(addr, k))


class NirvanaCache:
    """One cache handle on one CUDA device (see include/nirvana_cache.h)."""

    def __init__(self, entry_capacity: int, latent_capacity: int | None = None, dim: int = 768,
                 latent_bytes: int = 32768, k_values=(5, 10, 15, 20, 25),
                 thresholds=(0.65, 0.75, 0.85, 0.90, 0.95), k_bias: int = 0, max_topk: int = MAX_TOPK,
                 device: int | None = None, shard_rank: int = 0, shard_world: int = 1, latent_alias: bool = False,
                 evict_granularity: int = EVICT_ITEM):
        if device is None:
            device = torch.cuda.current_device()
        self.device = device
        if latent_capacity is None:
            latent_capacity = entry_capacity * len(k_values)
        self.cfg = default_config(dim=dim, entry_capacity=entry_capacity, latent_capacity=latent_capacity,
                                  latent_bytes=latent_bytes, k_values=tuple(k_values),
                                  thresholds=tuple(thresholds), k_bias=k_bias, max_topk=max_topk,
                                  shard_rank=shard_rank, shard_world=shard_world, latent_alias=int(latent_alias),
                                  evict_granularity=evict_granularity)
        self.granularity = evict_granularity
        self.latent_capacity = latent_capacity
        self.shard_rank, self.shard_world = shard_rank, shard_world
        self.dim, self.latent_bytes, self.num_k = dim, latent_bytes, len(k_values)
        self.k_values = tuple(k_values)
        h = ctypes.c_void_p()
        _check(_lib.cache_create(ctypes.byref(self.cfg), device, ctypes.byref(h)))
        self._h = h

    def _adopt_config(self):
        """Attributes from the handle's live configuration (cache_get_config)."""
        c = CacheConfig()
        _check(_lib.cache_get_config(self._h, ctypes.byref(c)))
        self.cfg = c
        self.granularity = c.evict_granularity
        self.latent_capacity = c.latent_capacity
        self.shard_rank, self.shard_world = c.shard_rank, c.shard_world
        self.dim, self.latent_bytes, self.num_k = c.dim, c.latent_bytes, c.num_k
        self.k_values = tuple(c.k_values[: c.num_k])

    def save(self, path: str, with_latents: bool = True):
        """cache_save: the whole state to `path` (checkpoint)."""
        _check(_lib.cache_save(self._h, os.fsencode(path), int(bool(with_latents))))

    @classmethod
    def load(cls, path: str, device: int | None = None) -> "NirvanaCache":
        """cache_load: a new handle holding the state saved in `path` (resume)."""
        if device is None:
            device = torch.cuda.current_device()
        self = cls.__new__(cls)
        self.device = device
        h = ctypes.c_void_p()
        _check(_lib.cache_load(os.fsencode(path), device, ctypes.byref(h)))
        self._h = h
        self._adopt_config()
        return self

    def close(self):
        if getattr(self, "_h", None):
            _lib.cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------------------------
    def insert(self, emb: torch.Tensor, latents: torch.Tensor | None = None, present=None, stream=None,
               raise_on_bad_rows: bool = False):
        """emb: [n][dim] f32/bf16 cuda; latents: [n][num_k][latent_bytes] u8 cuda or None;
        present: [n] u8 masks (numpy or tensor) or None.  Returns (ids u64[n], row_status i32[n])."""
        assert emb.is_cuda and emb.is_contiguous() and emb.dim() == 2 and emb.shape[1] == self.dim
        n = emb.shape[0]
        dt = DTYPE_BF16 if emb.dtype == torch.bfloat16 else DTYPE_F32
        assert emb.dtype in (torch.float32, torch.bfloat16)
        if latents is not None:
            assert latents.is_cuda and latents.is_contiguous() and latents.dtype == torch.uint8
            assert latents.numel() == n * self.num_k * self.latent_bytes
        pr = None
        if present is not None:
            pr = present if isinstance(present, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(present, np.uint8))
            pr = pr.contiguous()
        ids = np.empty(n, dtype=np.uint64)
        st = np.empty(n, dtype=np.int32)
        rc = _lib.cache_insert(self._h, n, _ptr(emb), dt, _ptr(latents), _ptr(pr), _ptr(ids), _ptr(st),
                               _stream(stream))
        _check(rc, allow=() if raise_on_bad_rows else (E_BAD_ROWS,))
        return ids, st

    def alloc_outputs(self, b: int, topk: int = 1, latents: bool = True):
        dev = torch.device("cuda", self.device)
        return dict(ids=torch.empty((b, topk), dtype=torch.int64, device=dev),
                    scores=torch.empty((b, topk), dtype=torch.float32, device=dev),
                    k=torch.empty(b, dtype=torch.int32, device=dev),
                    latents=torch.empty((b, self.latent_bytes), dtype=torch.uint8, device=dev) if latents else None,
                    ptrs=torch.empty(b, dtype=torch.int64, device=dev),
                    status=torch.empty(b, dtype=torch.int32, device=dev))

    def query_into(self, q: torch.Tensor, out: dict, topk: int = 1, stream=None):
        """Asynchronous lookup into preallocated outputs (see alloc_outputs)."""
        b = q.shape[0]
        dt = DTYPE_BF16 if q.dtype == torch.bfloat16 else DTYPE_F32
        rc = _lib.cache_query_batch(self._h, b, _ptr(q), dt, topk, _ptr(out["ids"]), _ptr(out["scores"]),
                                    _ptr(out["k"]), _ptr(out["latents"]), _ptr(out["ptrs"]),
                                    _ptr(out["status"]), _stream(stream))
        _check(rc)
        return out

    def query(self, q: torch.Tensor, topk: int = 1, latents: bool = True, stream=None):
        assert q.is_cuda and q.is_contiguous() and q.dim() == 2 and q.shape[1] == self.dim
        out = self.alloc_outputs(q.shape[0], topk, latents)
        return self.query_into(q, out, topk, stream)

    def submit(self, slot: int, q_host: torch.Tensor, topk: int = 1, latent_out: torch.Tensor | None = None,
               stream=None):
        """Pipelined lookup (cache_query_submit): q_host = pinned CPU tensor, kept alive by the
        caller until complete(slot); latent_out = device buffer or None."""
        dt = DTYPE_BF16 if q_host.dtype == torch.bfloat16 else DTYPE_F32
        _check(_lib.cache_query_submit(self._h, slot, q_host.shape[0], _ptr(q_host), dt, topk, _ptr(latent_out),
                                       _stream(stream)))

    def complete(self, slot: int, out: dict):
        """Wait for slot; out: host tensors ids [b][topk] int64, scores f32, k i32, status i32."""
        _check(_lib.cache_query_complete(self._h, slot, _ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["k"]),
                                         _ptr(out.get("status"))))
        return out

    def peek(self, q: torch.Tensor, topk: int = 1, stream=None):
        """Read-only lookup (cache_query_peek): ids / scores / K as query() would report them,
        with no access counted, no LRU clock tick and no latent gather."""
        assert q.is_cuda and q.is_contiguous() and q.dim() == 2 and q.shape[1] == self.dim
        out = self.alloc_outputs(q.shape[0], topk, latents=False)
        dt = DTYPE_BF16 if q.dtype == torch.bfloat16 else DTYPE_F32
        _check(_lib.cache_query_peek(self._h, q.shape[0], _ptr(q), dt, topk, _ptr(out["ids"]), _ptr(out["scores"]),
                                     _ptr(out["k"]), _ptr(out["status"]), _stream(stream)))
        return out

    def query_host(self, q: np.ndarray, topk: int = 1, latents: bool = True, out: dict | None = None, stream=None):
        """End-to-end lookup with host buffers (pinned numpy-compatible tensors recommended)."""
        b = q.shape[0]
        if out is None:
            out = dict(ids=np.empty((b, topk), np.uint64), scores=np.empty((b, topk), np.float32),
                       k=np.empty(b, np.int32), status=np.empty(b, np.int32),
                       latents=np.empty((b, self.latent_bytes), np.uint8) if latents else None)
        dt = DTYPE_BF16 if (isinstance(q, torch.Tensor) and q.dtype == torch.bfloat16) else DTYPE_F32
        rc = _lib.cache_query_batch_host(self._h, b, _ptr(q), dt, topk, _ptr(out["ids"]), _ptr(out["scores"]),
                                         _ptr(out["k"]), _ptr(out["latents"]), _ptr(out["status"]), _stream(stream))
        _check(rc)
        return out

    def evict_count(self, n: int, stream=None):
        """Evict without producing the lists (cache_evict with NULL outputs): (evicted, dirty)."""
        nd = np.zeros(1, dtype=np.int64)
        _check(_lib.cache_evict(self._h, n, None, None, _ptr(nd), _stream(stream)))
        return n, int(nd[0])

    def evict(self, n: int, stream=None, out=None, view: bool = False):
        """Returns (evicted, dirty ids).  out: optional (evicted, dirty) uint64 arrays of capacity
        >= n, reused across calls.  view=True: read-only numpy views of the library's pinned lists
        (cache_evict_view; no copy), valid until this cache's next eviction."""
        if view:
            pe, pd = ctypes.c_void_p(), ctypes.c_void_p()
            nd = ctypes.c_int64()
            _check(_lib.cache_evict_view(self._h, n, ctypes.byref(pe), ctypes.byref(pd), ctypes.byref(nd),
                                         _stream(stream)))
            return _u64_view(pe.value, n), _u64_view(pd.value, nd.value)
        if out is not None and len(out[0]) >= max(n, 1) and len(out[1]) >= max(n, 1):
            ev, dirty = out
        else:
            ev = np.empty(max(n, 1), dtype=np.uint64)
            dirty = np.empty(max(n, 1), dtype=np.uint64)
        nd = np.zeros(1, dtype=np.int64)
        _check(_lib.cache_evict(self._h, n, _ptr(ev), _ptr(dirty), _ptr(nd), _stream(stream)))
        return ev[:n], dirty[: int(nd[0])]   # views (no copy of the lists)

    def meta(self, id_: int):
        f = np.empty(self.num_k, dtype=np.uint64)
        m = np.zeros(1, dtype=np.uint32)
        _check(_lib.cache_get_meta(self._h, int(id_), _ptr(f), _ptr(m)))
        return f, int(m[0])

    def row_bf16(self, id_: int) -> np.ndarray:
        out = np.empty(self.dim, dtype=np.uint16)
        _check(_lib.cache_get_row(self._h, int(id_), _ptr(out)))
        return out

    def stats(self) -> dict:
        s = CacheStats()
        _check(_lib.cache_stats(self._h, ctypes.byref(s)))
        return {k: getattr(s, k) for k, _ in CacheStats._fields_}

    def set_evict_policy(self, policy: int):
        """POLICY_LCBFU (paper), POLICY_LRU, POLICY_LFU, POLICY_FIFO (its baselines)."""
        _check(_lib.cache_set_evict_policy(self._h, policy))

    def set_scorer(self, scorer: int):
        _check(_lib.cache_set_scorer(self._h, scorer))

    def set_query_slices(self, slices: int):
        """0 = auto, 1 = one scan launch, n = n query slices (finalize overlapped with the next scan)."""
        _check(_lib.cache_set_query_slices(self._h, slices))

    # ------------------------- match predictor (NEXT-3) --------------------------------
    def train_predictor(self, nu: float = 0.001, epochs: int = 50, lr0: float = 0.5, stream=None):
        _check(_lib.cache_predictor_train(self._h, nu, epochs, lr0, _stream(stream)))

    def predict(self, q: torch.Tensor, stream=None):
        """-> (flags uint8 [b], margins float32 [b]) device tensors."""
        b = q.shape[0]
        flags = torch.empty(b, dtype=torch.uint8, device=q.device)
        margin = torch.empty(b, dtype=torch.float32, device=q.device)
        dt = DTYPE_BF16 if q.dtype == torch.bfloat16 else DTYPE_F32
        _check(_lib.cache_predict(self._h, b, _ptr(q), dt, _ptr(flags), _ptr(margin), _stream(stream)))
        return flags, margin

    def predictor(self):
        w = np.empty(self.dim, dtype=np.float32)
        rho = np.empty(1, dtype=np.float32)
        _check(_lib.cache_predictor_get(self._h, _ptr(w), _ptr(rho)))
        return w, float(rho[0])

    def pool_write(self, slot0: int, src: torch.Tensor, stream=None):
        """Fill pool slots [slot0, slot0 + n) from a [n][latent_bytes] uint8 device tensor."""
        n = src.numel() // self.latent_bytes
        _check(_lib.cache_pool_write(self._h, slot0, n, _ptr(src), _stream(stream)))

    # ------------------------- sharded-path building blocks --------------------------
    def query_local(self, q: torch.Tensor, topk: int, out_recs: torch.Tensor, stream=None):
        """Ingest + scan of this shard for the global batch q -> out_recs [b][topk] records
        (a uint8 tensor of b*topk*16 bytes)."""
        dt = DTYPE_BF16 if q.dtype == torch.bfloat16 else DTYPE_F32
        _check(_lib.cache_query_local(self._h, q.shape[0], _ptr(q), dt, topk, _ptr(out_recs), _stream(stream)))
        return out_recs

    def query_merge(self, b: int, row0: int, nb: int, topk: int, recs_all: torch.Tensor, out: dict, stream=None):
        """Merge the world x b x topk records for global rows [row0, row0+nb) into out."""
        _check(_lib.cache_query_merge(self._h, b, row0, nb, topk, _ptr(recs_all), _ptr(out["ids"]),
                                      _ptr(out["scores"]), _ptr(out["k"]), _ptr(out.get("latents")),
                                      _ptr(out.get("ptrs")), _ptr(out.get("status")), _stream(stream)))
        return out

    # ---- push exchange (include/nirvana_cache.h, cache_push_*) ----
    def push_reserve(self, max_nb: int, max_topk: int):
        """Allocate this rank's exchange arena; before export_peer."""
        _check(_lib.cache_push_reserve(self._h, max_nb, max_topk))

    def push_queries(self, q_local: torch.Tensor, stream=None):
        """Phase 1: ingest this rank's rows and store them into every rank's arena."""
        dt = DTYPE_BF16 if q_local.dtype == torch.bfloat16 else DTYPE_F32
        _check(_lib.cache_push_queries(self._h, q_local.shape[0], _ptr(q_local), dt, _stream(stream)))

    def push_scan(self, nb: int, topk: int, stream=None):
        """Phase 2: wait for every rank's rows, scan this shard, push records to their owners."""
        _check(_lib.cache_push_scan(self._h, nb, topk, _stream(stream)))

    def push_merge(self, nb: int, topk: int, out: dict, stream=None):
        """Phase 3: wait for every rank's records, merge this rank's own nb rows into out."""
        _check(_lib.cache_push_merge(self._h, nb, topk, _ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["k"]),
                                     _ptr(out.get("latents")), _ptr(out.get("ptrs")), _ptr(out.get("status")),
                                     _stream(stream)))
        return out

    def last_evicted_keys(self) -> np.ndarray:
        """64-bit unit keys of the last eviction that returned its list, in eviction order."""
        n = np.zeros(1, dtype=np.int64)
        _check(_lib.cache_last_evicted_keys(self._h, None, 0, _ptr(n)))
        out = np.empty(max(int(n[0]), 1), dtype=np.uint64)
        _check(_lib.cache_last_evicted_keys(self._h, _ptr(out), int(n[0]), _ptr(n)))
        return out[: int(n[0])]

    # ---- distributed fused eviction (cache_evict_sel_*) ----
    def evict_sel_begin(self, n: int, stream=None):
        _check(_lib.cache_evict_sel_begin(self._h, n, _stream(stream)))

    def evict_sel_level(self, level: int, hist: torch.Tensor, stream=None):
        """This rank's 4,096-bin histogram of the level into hist (cuda int32[4096])."""
        _check(_lib.cache_evict_sel_level(self._h, level, _ptr(hist), _stream(stream)))

    def evict_sel_pick(self, level: int, hist_sum: torch.Tensor, stream=None) -> bool:
        done = np.zeros(1, dtype=np.int32)
        _check(_lib.cache_evict_sel_pick(self._h, level, _ptr(hist_sum), _ptr(done), _stream(stream)))
        return bool(done[0])

    def evict_sel_apply(self, cap: int, stream=None, lists: bool = True):
        """This rank's share: (evicted, dirty) lists, or (n evicted, n dirty) with lists=False."""
        ev = np.empty(max(cap, 1), dtype=np.uint64) if lists else None
        dirty = np.empty(max(cap, 1), dtype=np.uint64) if lists else None
        n = np.zeros(1, dtype=np.int64)
        nd = np.zeros(1, dtype=np.int64)
        _check(_lib.cache_evict_sel_apply(self._h, cap, _ptr(ev), _ptr(n), _ptr(dirty), _ptr(nd), _stream(stream)))
        if not lists:
            return int(n[0]), int(nd[0])
        return ev[: int(n[0])], dirty[: int(nd[0])]

    def push_evict_sel_level(self, level: int, stream=None):
        _check(_lib.cache_push_evict_sel_level(self._h, level, _stream(stream)))

    def push_evict_sel_pick(self, level: int, stream=None) -> bool:
        done = np.zeros(1, dtype=np.int32)
        _check(_lib.cache_push_evict_sel_pick(self._h, level, _ptr(done), _stream(stream)))
        return bool(done[0])

    def push_status(self, stream=None):
        """Synchronise the stream; CacheError(E_NCCL) if a peer wait of this handle timed out."""
        _check(_lib.cache_push_status(self._h, _stream(stream)))

    def set_peer_timeout(self, ms: int):
        _check(_lib.cache_set_peer_timeout(self._h, int(ms)))

    # ---- cache-selector profiling (Alg. 2) ----
    def profile_thresholds(self, q: torch.Tensor, quality: torch.Tensor, alpha: float = 0.9, stream=None):
        """q: [b][dim] cuda profiling prompts; quality: [num_k][b] float32 cuda (the model's image
        quality per prompt and K).  Returns (thresholds float64[num_k], failed bool[num_k])."""
        dt = DTYPE_BF16 if q.dtype == torch.bfloat16 else DTYPE_F32
        quality = quality.contiguous().to(torch.float32)
        thr = np.empty(self.num_k, dtype=np.float64)
        failed = np.zeros(self.num_k, dtype=np.int64)
        _check(_lib.cache_profile_thresholds(self._h, q.shape[0], _ptr(q), dt, _ptr(quality), float(alpha),
                                             _ptr(thr), _ptr(failed), _stream(stream)))
        return thr, failed.astype(bool)

    def set_thresholds(self, thresholds):
        t = np.ascontiguousarray(thresholds, dtype=np.float64)
        _check(_lib.cache_set_thresholds(self._h, _ptr(t)))

    def push_evict_hist(self, n: int, pass_: int, stream=None):
        _check(_lib.cache_push_evict_hist(self._h, n, pass_, _stream(stream)))

    def push_evict_pick(self, pass_: int, stream=None):
        _check(_lib.cache_push_evict_pick(self._h, pass_, _stream(stream)))

    def push_evict_apply(self, n: int, stream=None, lists: bool = True):
        """lists=False: only the counts come back (returns (n_evicted, n_dirty))."""
        ev = np.empty(max(n, 1), dtype=np.uint64) if lists else None
        dirty = np.empty(max(n, 1), dtype=np.uint64) if lists else None
        cnt = np.zeros(1, dtype=np.int64)
        nd = np.zeros(1, dtype=np.int64)
        _check(_lib.cache_push_evict_apply(self._h, n, _ptr(ev), _ptr(cnt), _ptr(dirty), _ptr(nd), _stream(stream)))
        if not lists:
            return int(cnt[0]), int(nd[0])
        return ev[: int(cnt[0])].copy(), dirty[: int(nd[0])].copy()

    def export_peer(self) -> PeerDesc:
        d = PeerDesc()
        _check(_lib.cache_export_peer(self._h, ctypes.byref(d)))
        return d

    def attach_peers(self, descs):
        arr = (PeerDesc * len(descs))(*descs)
        _check(_lib.cache_attach_peers(self._h, len(descs), arr))

    def evict_hist(self, state: torch.Tensor, pass_: int, hist: torch.Tensor, stream=None):
        _check(_lib.cache_evict_hist(self._h, _ptr(state), pass_, _ptr(hist), _stream(stream)))

    def evict_pick(self, hist: torch.Tensor, state: torch.Tensor, pass_: int, stream=None):
        _check(_lib.cache_evict_pick(self._h, _ptr(hist), _ptr(state), pass_, _stream(stream)))

    def evict_apply(self, state: torch.Tensor, cap: int, stream=None, lists: bool = True):
        """lists=False: only the counts come back (returns (n_evicted, n_dirty))."""
        ev = np.empty(max(cap, 1), dtype=np.uint64) if lists else None
        dirty = np.empty(max(cap, 1), dtype=np.uint64) if lists else None
        n = np.zeros(1, dtype=np.int64)
        nd = np.zeros(1, dtype=np.int64)
        _check(_lib.cache_evict_apply(self._h, _ptr(state), cap, _ptr(ev), _ptr(n), _ptr(dirty), _ptr(nd),
                                      _stream(stream)))
        if not lists:
            return int(n[0]), int(nd[0])
        return ev[: int(n[0])].copy(), dirty[: int(nd[0])].copy()

    @property
    def live_items(self) -> int:
        return _lib.cache_live_items(self._h)

    @property
    def live_entries(self) -> int:
        return _lib.cache_live_entries(self._h)

    def set_evict_granularity(self, granularity: int):
        """EVICT_ITEM (the paper's item granularity) or EVICT_ENTRY: evict(n) then removes n
        whole entries by the aggregated policy score (include/nirvana_cache.h, R24)."""
        _check(_lib.cache_set_evict_granularity(self._h, granularity))
        self.granularity = granularity

    @property
    def evict_units(self) -> int:
        """What evict(n) counts on this rank: live items, or live entries in entry mode."""
        return self.live_entries if getattr(self, "granularity", EVICT_ITEM) == EVICT_ENTRY else self.live_items

    def set_profile_events(self, events):
        """events: 4 torch.cuda.Event(enable_timing=True) (recorded around ingest / score /
        finalize of every query), or None to disable."""
        if events is None:
            _check(_lib.cache_set_profile_events(self._h, None))
            self._prof = None
            return
        for e in events:
            e.record()          # materialise the underlying cudaEvent_t
        arr = (ctypes.c_void_p * 4)(*[e.cuda_event for e in events])
        self._prof = (events, arr)
        _check(_lib.cache_set_profile_events(self._h, arr))

    @property
    def kernel_launches(self) -> int:
        return _lib.cache_kernel_launches(self._h)


# ------------------------------- test-only entry points -------------------------------
_lib.cache_debug_tc_scores.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                       ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
_lib.cache_debug_tc_scores.restype = ctypes.c_int
_lib.cache_debug_slot_of.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
_lib.cache_debug_slot_of.restype = ctypes.c_int64


def debug_tc_scores(cache: NirvanaCache, q: torch.Tensor, stream=None) -> torch.Tensor:
    """Dense fl(<q~,x~> * inv_norm(x~)) from the tcgen05 main loop, [b][round_up(hwm, 256)]."""
    hwm = cache.stats()["entry_hwm"]
    ld = max(256, (hwm + 255) // 256 * 256)
    out = torch.full((q.shape[0], ld), float("nan"), dtype=torch.float32, device=q.device)
    dt = DTYPE_BF16 if q.dtype == torch.bfloat16 else DTYPE_F32
    _check(_lib.cache_debug_tc_scores(cache._h, q.shape[0], _ptr(q), dt, _ptr(out), ld, _stream(stream)))
    return out


_lib.cache_debug_sort_u64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
_lib.cache_debug_sort_u64.restype = ctypes.c_int


def debug_sort_u64(keys: torch.Tensor, stream=None) -> torch.Tensor:
    """Sort a cuda int64 tensor (as u64 bit patterns) in place with the eviction path's sort."""
    _check(_lib.cache_debug_sort_u64(_ptr(keys), keys.numel(), _stream(stream)))
    return keys


def debug_slot_of(cache: NirvanaCache, id_: int) -> int:
    return _lib.cache_debug_slot_of(cache._h, int(id_))


_lib.cache_debug_sort_u64_ex.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint64,
                                         ctypes.c_int32, ctypes.c_void_p]
_lib.cache_debug_sort_u64_ex.restype = ctypes.c_int
_lib.cache_debug_evict_stats.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
_lib.cache_debug_evict_stats.restype = ctypes.c_int
_lib.cache_debug_set_evict_cand_cap.argtypes = [ctypes.c_void_p, ctypes.c_int64]
_lib.cache_debug_set_evict_cand_cap.restype = ctypes.c_int


def debug_sort_u64_ex(keys: torch.Tensor, bits: int = 64, base: int = 0, small=False, stream=None):
    """The eviction sorts with their options: keys in [base, base + 2^bits); small = 1 / True:
    the one-CTA sort, 2: the cooperative one-launch LSD sort."""
    _check(_lib.cache_debug_sort_u64_ex(_ptr(keys), keys.numel(), bits, base, int(small), _stream(stream)))
    return keys


def debug_evict_stats(cache: NirvanaCache) -> dict:
    """Last cache_evict: levels, full sweeps, compaction level (0 = none), candidates."""
    a = (ctypes.c_int64 * 4)()
    _check(_lib.cache_debug_evict_stats(cache._h, a))
    return dict(levels=a[0], full_sweeps=a[1], compact_level=a[2], candidates=a[3])


def debug_set_evict_cand_cap(cache: NirvanaCache, cap: int):
    _check(_lib.cache_debug_set_evict_cand_cap(cache._h, int(cap)))


_lib.cache_debug_evict_window.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p]
_lib.cache_debug_evict_window.restype = ctypes.c_int


def debug_evict_window(cache: NirvanaCache, stride=None) -> int:
    """Set the single-sweep window's sample stride (-1 auto, 0 off, S fixed; None: leave it) and
    return the last eviction's window outcome (0 off, 1 used, 2 estimate missed)."""
    last = ctypes.c_int32(0)
    _check(_lib.cache_debug_evict_window(cache._h, -1 if stride is None else int(stride), int(stride is not None),
                                         ctypes.byref(last)))
    return last.value


_lib.cache_debug_set_count.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_uint32]
_lib.cache_debug_set_count.restype = ctypes.c_int


def debug_set_count(cache: NirvanaCache, id_: int, j: int, f: int):
    _check(_lib.cache_debug_set_count(cache._h, int(id_), int(j), int(f)))
