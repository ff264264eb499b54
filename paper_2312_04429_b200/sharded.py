"""Entry-sharded NIRVANA cache over several GPUs.

Every step runs in the library's kernels; this module only moves buffers between ranks with
collectives (torch.distributed / NCCL over NVLink, or in-process copies for virtual ranks):

  insert  every rank receives the same batch; accepted rows get global ids 0,1,2,...
          and rank r stores the rows with id % world == r (cache_insert, shard config)
  query   all-gather the ranks' local query batches -> global batch Q (b rows)
          -> cache_query_local on every rank (tcgen05 scan of its shard + local top-k)
          -> all-gather the 16-byte shard records (world x b x topk)
          -> cache_query_merge for the rank's own rows: merge under (score desc, id asc),
             Fig. 11 + holes, and the winning state copied straight out of the OWNER's latent
             pool over NVLink (peer pointers from CUDA IPC), access counted on the owner's f
  evict   the fused eviction's levels (cache_evict_sel_*): per rank a sweep of its shard into a
          4,096-bin histogram (level 0: log bins; later levels: 12-bit digits, applying the units
          certain to go and compacting the candidates), the histograms summed over ranks (an
          all-reduce, or P2P atomics into every rank's arena), the same pick on every rank; then
          each rank applies the global threshold to its own units.  Round 1's 8-pass radix
          protocol (cache_evict_hist / _pick / _apply) stays selectable (evict_protocol).

Because a query's answer is a max over shards under a total order and ids are global, the
results are identical to one unsharded cache (tested with virtual ranks on one GPU).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import binding as B


def _comm_errors(fn):
    """A failed collective (NCCL error, or the process group's timeout / watchdog when a rank
    died or stalled) surfaces as CacheError(E_NCCL), the status the C ABI reports when a
    push-exchange wait times out (failure detection)."""
    import functools

    @functools.wraps(fn)
    def wrap(*a, **kw):
        try:
            return fn(*a, **kw)
        except B.CacheError:
            raise
        except (RuntimeError, ValueError) as e:   # torch.distributed raises DistBackendError etc.
            raise B.CacheError(B.E_NCCL, f"collective {fn.__name__} failed: {e}") from e
    return wrap


class TorchComm:
    """Collectives of one process group (one rank per GPU).  Create the group with a timeout
    (init_process_group(timeout=...)) so that a dead rank fails the collectives instead of
    hanging them; the failure is reported as CacheError(E_NCCL)."""

    def __init__(self, group=None, device: str = "cuda"):
        import torch.distributed as dist
        self.dist, self.group, self.device = dist, group, device
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    @_comm_errors
    def all_gather(self, t: torch.Tensor) -> torch.Tensor:
        out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out.view(-1), t.contiguous().view(-1), group=self.group)
        return out

    @_comm_errors
    def all_reduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        self.dist.all_reduce(t, group=self.group)
        return t

    @_comm_errors
    def all_reduce_min_int(self, v: int) -> int:
        t = torch.tensor([v], dtype=torch.int64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    @_comm_errors
    def all_gather_object(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


def query_protocol(comm, q_local: torch.Tensor, topk: int, local_fn, merge_fn):
    """The sharded lookup's data movement: all-gather queries -> local scan (local_fn(qg) ->
    this rank's record tensor) -> all-gather records -> merge of this rank's own rows
    (merge_fn(b, row0, nb, recs_all)).  Rank r owns global rows [r*nb, (r+1)*nb)."""
    qg = comm.all_gather(q_local).reshape(-1, q_local.shape[1])
    recs = local_fn(qg)
    recs_all = comm.all_gather(recs)
    nb = q_local.shape[0]
    return merge_fn(qg.shape[0], comm.rank * nb, nb, recs_all)


def evict_protocol(comm, n: int, state, hist, hist_fn, pick_fn):
    """Distributed exact selection of the n lowest item keys: 8 MSB-first radix passes, each
    a per-rank histogram summed over ranks, then the same digit pick on every rank."""
    for p in range(8):
        hist_fn(state, p, hist)
        comm.all_reduce_sum(hist)
        pick_fn(hist, state, p)
    return state


def _dev() -> str:
    """Device of the small protocol tensors: the GPU's (the kernels write them); CPU only for the
    gloo protocol tests, whose ranks are played by numpy stand-ins."""
    return "cuda" if torch.cuda.is_available() else "cpu"


def _desc_bytes(d: B.PeerDesc) -> bytes:
    return ctypes.string_at(ctypes.addressof(d), ctypes.sizeof(d))


def _desc_from_bytes(b: bytes) -> B.PeerDesc:
    d = B.PeerDesc()
    ctypes.memmove(ctypes.addressof(d), b, ctypes.sizeof(d))
    return d


class ShardedCache:
    """One rank's handle of an entry-sharded cache (one process per GPU)."""

    evict_protocol = "levels"   # or "radix8": round 1's 8-pass radix-select protocol

    def __init__(self, comm: TorchComm, entry_capacity: int, latent_capacity: int | None = None,
                 push_max_nb: int = 0, push_max_topk: int = 1, **kw):
        """push_max_nb > 0: reserve the exchange arena for the fused push path (query_into
        then moves no data through the collective library); 0: all-gather path."""
        self.comm = comm
        self.cache = B.NirvanaCache(entry_capacity=entry_capacity, latent_capacity=latent_capacity,
                                    shard_rank=comm.rank, shard_world=comm.world, **kw)
        self.push = push_max_nb > 0
        if self.push:
            self.cache.push_reserve(push_max_nb, push_max_topk)
        descs = comm.all_gather_object(_desc_bytes(self.cache.export_peer()))
        self.cache.attach_peers([_desc_from_bytes(d) for d in descs])
        self.latent_bytes = self.cache.latent_bytes

    def insert(self, emb: torch.Tensor, latents=None, present=None):
        """Collective: every rank passes the SAME batch.  Conservative capacity agreement: the
        insert proceeds only if every rank can hold its worst-case share."""
        n = emb.shape[0]
        share = (n + self.comm.world - 1) // self.comm.world
        st = self.cache.stats()
        items_ok = bool(self.cache.cfg.latent_alias) or st["free_items"] >= share * self.cache.num_k
        ok = int(st["free_entries"] >= share and items_ok)
        if self.comm.all_reduce_min_int(ok) == 0:
            raise B.CacheError(B.E_FULL, "sharded insert: some rank lacks capacity for its share")
        return self.cache.insert(emb, latents, present)

    def set_evict_policy(self, policy: int):
        self.cache.set_evict_policy(policy)

    def set_evict_granularity(self, granularity: int):
        self.cache.set_evict_granularity(granularity)

    def alloc_outputs(self, b_local: int, topk: int = 1, latents: bool = True):
        return self.cache.alloc_outputs(b_local, topk, latents)

    def query_into(self, q_local: torch.Tensor, out: dict, topk: int = 1, stream=None):
        """Collective: every rank passes its own b_local queries (same b_local everywhere)."""
        if self.push:   # the three fused phases; the only cross-rank traffic is P2P stores
            nb = q_local.shape[0]
            self.cache.push_queries(q_local, stream)
            self.cache.push_scan(nb, topk, stream)
            return self.cache.push_merge(nb, topk, out, stream)

        def local_fn(qg):
            recs = torch.empty((qg.shape[0] * topk * B.SHARD_REC_BYTES,), dtype=torch.uint8, device=qg.device)
            return self.cache.query_local(qg, topk, recs, stream)

        def merge_fn(b, row0, nb, recs_all):
            return self.cache.query_merge(b, row0, nb, topk, recs_all, out, stream)

        return query_protocol(self.comm, q_local, topk, local_fn, merge_fn)

    def query_host(self, q_host: torch.Tensor, out_host: dict, out_dev: dict, topk: int = 1, stream=None):
        """End-to-end collective lookup from host memory: this rank's b_local fp32 (or bf16)
        query rows are copied from (pinned) host memory, looked up with query_into, and the
        ids / scores / K / status come back to out_host (pinned tensors); the latent states stay
        in out_dev["latents"], the denoiser's device input buffer.  Synchronises the stream."""
        s = stream if stream is not None else torch.cuda.current_stream()
        qd = getattr(self, "_q_stage", None)
        if qd is None or qd.shape != q_host.shape or qd.dtype != q_host.dtype:
            qd = self._q_stage = torch.empty(q_host.shape, dtype=q_host.dtype, device="cuda")
        with torch.cuda.stream(s):
            qd.copy_(q_host, non_blocking=True)
            self.query_into(qd, out_dev, topk, s)
            for k in ("ids", "scores", "k", "status"):
                out_host[k].copy_(out_dev[k], non_blocking=True)
        s.synchronize()
        if self.push:
            self.cache.push_status(s)   # E_NCCL if a peer wait of this batch timed out
        return out_host

    def status(self, stream=None):
        """Synchronise; CacheError(E_NCCL) if this rank's push exchange saw a peer time out."""
        if self.push:
            self.cache.push_status(stream)
        else:
            torch.cuda.synchronize()

    def evict(self, n: int, lists: bool = True):
        """Collective: evict the n globally lowest-keyed items (entries in entry mode; every
        rank passes the same n).  lists=False skips gathering the evicted / dirty id lists to
        every rank and returns this rank's (evicted count, dirty count) instead."""
        live = self.comm.all_reduce_sum(torch.tensor([self.cache.evict_units], dtype=torch.int64,
                                                     device=_dev())).item()
        if n > live:
            raise B.CacheError(B.E_EVICT_RANGE, "sharded evict: n exceeds live items / entries")
        if self.comm.world == 1:   # one shard: no exchange, the fused single-launch eviction
            if not lists:
                return self.cache.evict_count(n)
            ev, dirty = self.cache.evict(n, view=True)
            return ev.copy(), dirty.copy()
        if self.evict_protocol == "levels":   # the fused levels, histograms summed between them
            cap = max(1, min(n, self.cache.evict_units))
            self.cache.evict_sel_begin(n)
            for level in range(8):
                if self.push:   # summed over peer memory by the kernels themselves
                    self.cache.push_evict_sel_level(level)
                    done = self.cache.push_evict_sel_pick(level)
                else:
                    hist = torch.empty(4096, dtype=torch.int32, device=_dev())
                    self.cache.evict_sel_level(level, hist)
                    self.comm.all_reduce_sum(hist)
                    done = self.cache.evict_sel_pick(level, hist)
                if done:
                    break
            res = self.cache.evict_sel_apply(cap, lists=lists)
        elif self.push:   # round 1's 8-pass radix protocol, histograms over peer memory
            for p in range(8):
                self.cache.push_evict_hist(n, p)
                self.cache.push_evict_pick(p)
            res = self.cache.push_evict_apply(n, lists=lists)
        else:
            st = torch.tensor([0, 0, n], dtype=torch.int64, device="cuda")
            hist = torch.zeros(256, dtype=torch.int32, device="cuda")
            evict_protocol(self.comm, n, st, hist, self.cache.evict_hist, self.cache.evict_pick)
            res = self.cache.evict_apply(st, n, lists=lists)
        if not lists:
            return res   # this rank's (evicted count, dirty count)
        ev, dirty = res
        # numpy arrays (pickled as one buffer each), merged vectorised: Python lists of the 619K
        # keys of a 1% eviction at 12.5M entries per rank cost ~45 ms of host time
        evs = self.comm.all_gather_object(np.ascontiguousarray(self.cache.last_evicted_keys(), dtype=np.uint64))
        dts = self.comm.all_gather_object(np.ascontiguousarray(dirty, dtype=np.uint64))
        return _merge_evicted(evs, self.cache), _sorted_u64(dts)


class VirtualShards:
    """P shards of one cache held by ONE process on one GPU (virtual ranks): the same kernels
    and the same merge/P2P code path as ShardedCache, with collectives replaced by copies.
    Used to test sharding invariance on a single B200."""

    evict_protocol = "levels"   # or "radix8"

    def __init__(self, world: int, entry_capacity: int, latent_capacity: int | None = None,
                 push_max_nb: int = 0, push_max_topk: int = 1, **kw):
        self.world = world
        self.caches = [B.NirvanaCache(entry_capacity=entry_capacity, latent_capacity=latent_capacity,
                                      shard_rank=r, shard_world=world, **kw) for r in range(world)]
        self.push = push_max_nb > 0
        if self.push:
            for c in self.caches:
                c.push_reserve(push_max_nb, push_max_topk)
        descs = [c.export_peer() for c in self.caches]
        for c in self.caches:
            c.attach_peers(descs)
        self.latent_bytes = self.caches[0].latent_bytes

    def insert(self, emb, latents=None, present=None):
        res = [c.insert(emb, latents, present) for c in self.caches]
        return res[0]

    def query(self, q_global: torch.Tensor, topk: int = 1, latents: bool = True):
        """q_global = the concatenation of the ranks' local batches (b divisible by world)."""
        b = q_global.shape[0]
        assert b % self.world == 0
        bl = b // self.world
        if self.push:   # one stream: every rank's phase 1, then phase 2, then phase 3
            for r, c in enumerate(self.caches):
                c.push_queries(q_global[r * bl:(r + 1) * bl])
            for c in self.caches:
                c.push_scan(bl, topk)
            outs = [c.push_merge(bl, topk, c.alloc_outputs(bl, topk, latents)) for c in self.caches]
            return {k: (torch.cat([o[k] for o in outs]) if outs[0][k] is not None else None) for k in outs[0]}
        recs = []
        for c in self.caches:
            r = torch.empty((b * topk * B.SHARD_REC_BYTES,), dtype=torch.uint8, device=q_global.device)
            c.query_local(q_global, topk, r)
            recs.append(r)
        recs_all = torch.stack(recs)
        outs = []
        for r, c in enumerate(self.caches):
            o = c.alloc_outputs(bl, topk, latents)
            c.query_merge(b, r * bl, bl, topk, recs_all, o)
            outs.append(o)
        cat = {k: (torch.cat([o[k] for o in outs]) if outs[0][k] is not None else None) for k in outs[0]}
        return cat

    def evict(self, n: int):
        live = sum(c.evict_units for c in self.caches)
        if n > live:
            raise B.CacheError(B.E_EVICT_RANGE, "sharded evict: n exceeds live items / entries")
        if self.evict_protocol == "levels":   # the fused levels (one stream: level on every rank, then picks)
            caps = [max(1, min(n, c.evict_units)) for c in self.caches]
            for c in self.caches:
                c.evict_sel_begin(n)
            for level in range(8):
                if self.push:
                    for c in self.caches:
                        c.push_evict_sel_level(level)
                    dones = [c.push_evict_sel_pick(level) for c in self.caches]
                else:
                    hists = [torch.empty(4096, dtype=torch.int32, device="cuda") for _ in self.caches]
                    for c, h in zip(self.caches, hists):
                        c.evict_sel_level(level, h)
                    tot = torch.stack(hists).sum(0).to(torch.int32)
                    dones = [c.evict_sel_pick(level, tot) for c in self.caches]
                assert len(set(dones)) == 1, "ranks disagree on the selection (internal error)"
                if dones[0]:
                    break
            res = [c.evict_sel_apply(cap) for c, cap in zip(self.caches, caps)]
            keys = [c.last_evicted_keys() for c in self.caches]
            return _merge_evicted(keys, self.caches[0]), _sorted_u64([r[1] for r in res])
        if self.push:   # one stream: pass p's histogram on every rank, then every rank's pick
            for p in range(8):
                for c in self.caches:
                    c.push_evict_hist(n, p)
                for c in self.caches:
                    c.push_evict_pick(p)
            res = [c.push_evict_apply(n) for c in self.caches]
            keys = [c.last_evicted_keys() for c in self.caches]
            return _merge_evicted(keys, self.caches[0]), _sorted_u64([r[1] for r in res])
        sts = [torch.tensor([0, 0, n], dtype=torch.int64, device="cuda") for _ in self.caches]
        hists = [torch.zeros(256, dtype=torch.int32, device="cuda") for _ in self.caches]
        for p in range(8):
            for c, st, h in zip(self.caches, sts, hists):
                c.evict_hist(st, p, h)
            tot = torch.stack(hists).sum(0).to(torch.int32)
            for c, st, h in zip(self.caches, sts, hists):
                h.copy_(tot)
                c.evict_pick(h, st, p)
        res = [c.evict_apply(st, n) for c, st in zip(self.caches, sts)]
        keys = [c.last_evicted_keys() for c in self.caches]
        return _merge_evicted(keys, self.caches[0]), _sorted_u64([r[1] for r in res])

    def meta(self, id_: int):
        return self.caches[id_ % self.world].meta(id_)

    def set_evict_policy(self, policy: int):
        for c in self.caches:
            c.set_evict_policy(policy)

    def set_evict_granularity(self, granularity: int):
        for c in self.caches:
            c.set_evict_granularity(granularity)

    def stats(self):
        ss = [c.stats() for c in self.caches]
        return {k: sum(s[k] for s in ss) if k not in ("next_id",) else ss[0][k] for k in ss[0]}


def _sorted_u64(arrays) -> np.ndarray:
    """The union of the ranks' uint64 arrays (or lists), ascending.  Each rank's list is already
    ascending: the stable sort (timsort on integers wider than 16 bits) merges the runs in
    linear time."""
    parts = [np.asarray(a, dtype=np.uint64).ravel() for a in arrays]
    return np.sort(np.concatenate(parts), kind="stable") if parts else np.zeros(0, np.uint64)


def _merge_evicted(key_lists, cache):
    """The global eviction order (the API's: ascending unit key, R11 / R24) from the ranks'
    full 64-bit keys (cache_last_evicted_keys; keys are unique across ranks), mapped to what
    cache_evict reports: id << 3 | j per item, or the entry id in entry mode."""
    keys = _sorted_u64(key_lists)
    entry = getattr(cache, "granularity", B.EVICT_ITEM) == B.EVICT_ENTRY
    mask = np.uint64(0xFFFFFFFF) if entry else np.uint64((1 << 35) - 1)
    return keys & mask
