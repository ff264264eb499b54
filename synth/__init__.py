"""Seeded synthetic inputs shaped like the paper's workload (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no normalisation-for-storage, no scoring, no
K map, no eviction): it only draws inputs.  Both the CUDA path and the oracle consume what it
returns; neither is imported here.  Recipe:

* entries  -- 768-d CLIP-like text embeddings: n_c = max(1, n // 64) cluster centres
  ~ normalize(N(0, I)); entry = normalize(centre + sigma_e * g) with sigma_e chosen so that
  cos(entry, centre) ~= 0.85 (popular-prompt clusters).  0.1% of rows are exact
  duplicates of an earlier row (tie cases).  Returned as fp32; the library normalises and
  rounds to bf16 on insert.
* present  -- 5% of entries lose one random K (holes affect 4-5% of prompts).
* queries  -- anchor entry: cluster ~ Zipf(s) then uniform inside the cluster; target cosine t
  drawn from the paper's similarity buckets aligned with the Fig. 11 thresholds:
  <0.65 12% (88% overall hit-rate), (0.65,0.75] 20%, (0.75,0.85] 20%, (0.85,0.90] 20%,
  (0.90,0.95] 20%, >0.95 8% (K=25 hit-rate 8%); q = normalize(anchor + sigma * g),
  sigma = sqrt((1/t^2 - 1)/d).  1% of queries repeat a cached vector exactly (session
  repetition).
* latents  -- opaque latent_bytes-byte payloads (4x64x64 fp16 = 32 KiB in BASELINE configs);
  a counter-based 32-bit hash of (seed, row, j, word) with a 16-byte (row, j, magic) stamp so
  that a misrouted gather is detectable.  numpy and torch implementations of the same integer
  function (torch for filling device memory at benchmark scale).
"""
from __future__ import annotations

import numpy as np

D = 768
K_VALUES = (5, 10, 15, 20, 25)
BUCKETS = ((-1.0, 0.65, 0.12), (0.65, 0.75, 0.20), (0.75, 0.85, 0.20),
           (0.85, 0.90, 0.20), (0.90, 0.95, 0.20), (0.95, 1.0, 0.08))
MAGIC = 0x4E495256  # 'NIRV'


def _unit(x):
    n = np.sqrt(np.sum(x.astype(np.float64) ** 2, axis=-1, keepdims=True))
    return (x / n).astype(np.float32)


def entries(n: int, seed: int, dim: int = D, dup_frac: float = 0.001, cos_centre: float = 0.85,
            chunk: int = 65536):
    """Clustered unit-norm fp32 embeddings.  Returns (emb [n][dim] fp32, cluster [n] int64)."""
    rng = np.random.default_rng(seed)
    n_c = max(1, n // 64)
    centres = _unit(rng.standard_normal((n_c, dim), dtype=np.float32))
    cluster = rng.integers(0, n_c, size=n)
    sigma = np.sqrt((1.0 / cos_centre ** 2 - 1.0) / dim)
    out = np.empty((n, dim), dtype=np.float32)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        g = rng.standard_normal((e - s, dim), dtype=np.float32)
        out[s:e] = _unit(centres[cluster[s:e]] + np.float32(sigma) * g)
    n_dup = int(n * dup_frac)
    if n_dup and n > 1:
        dst = rng.choice(np.arange(1, n), size=min(n_dup, n - 1), replace=False)
        for d in np.sort(dst):
            src = int(rng.integers(0, d))
            out[d] = out[src]
            cluster[d] = cluster[src]
    return out, cluster


def present_masks(n: int, seed: int, num_k: int = 5, hole_frac: float = 0.05):
    """Per-entry K presence bitmasks (bit j = K_j stored); hole_frac of rows lose one K."""
    rng = np.random.default_rng(seed + 7777)
    m = np.full(n, (1 << num_k) - 1, dtype=np.uint8)
    sel = rng.random(n) < hole_frac
    drop = rng.integers(0, num_k, size=n)
    m[sel] &= ~(np.uint8(1) << drop[sel].astype(np.uint8))
    return m


def queries(emb: np.ndarray, cluster: np.ndarray, b: int, seed: int, zipf_s: float = 1.0,
            repeat_frac: float = 0.01, by_entry: bool = False):
    """Queries around Zipf-popular anchors with the bucket mixture above.

    Returns (q [b][dim] fp32, anchor_row [b] int64, target_cos [b] float64)."""
    rng = np.random.default_rng(seed + 1234567)
    n, dim = emb.shape
    if by_entry:
        ranks = np.arange(1, n + 1, dtype=np.float64)
        p = ranks ** -zipf_s
        p /= p.sum()
        perm = rng.permutation(n)
        anchor = perm[rng.choice(n, size=b, p=p)]
    else:
        uniq = np.unique(cluster)
        ranks = np.arange(1, len(uniq) + 1, dtype=np.float64)
        p = ranks ** -zipf_s
        p /= p.sum()
        perm = rng.permutation(uniq)
        cl = perm[rng.choice(len(uniq), size=b, p=p)]
        order = np.argsort(cluster, kind="stable")
        sorted_cl = cluster[order]
        lo = np.searchsorted(sorted_cl, cl, side="left")
        hi = np.searchsorted(sorted_cl, cl, side="right")
        anchor = order[lo + (rng.random(b) * (hi - lo)).astype(np.int64)]
    probs = np.array([w for _, _, w in BUCKETS])
    bk = rng.choice(len(BUCKETS), size=b, p=probs / probs.sum())
    lo_t = np.array([BUCKETS[i][0] for i in bk])
    hi_t = np.array([BUCKETS[i][1] for i in bk])
    lo_t = np.maximum(lo_t, 0.40)            # "miss" bucket drawn from (0.40, 0.65)
    t = lo_t + (hi_t - lo_t) * rng.random(b)
    t = np.clip(t, 0.40, 0.999)
    sigma = np.sqrt((1.0 / t ** 2 - 1.0) / dim)
    g = rng.standard_normal((b, dim), dtype=np.float32)
    q = _unit(emb[anchor] + (sigma[:, None] * g).astype(np.float32))
    rep = rng.random(b) < repeat_frac
    q[rep] = emb[anchor[rep]]
    t[rep] = 1.0
    return q, anchor, t


# ---------------- latent payloads: counter-based hash, numpy and torch -----------------
_M32 = 0xFFFFFFFF


def _mix_np(x):
    x = x.astype(np.uint32)
    x ^= x >> np.uint32(16)
    x *= np.uint32(0x21F0AAAD)
    x ^= x >> np.uint32(15)
    x *= np.uint32(0x735A2D97)
    x ^= x >> np.uint32(15)
    return x


def latent_np(rows, j: int, latent_bytes: int, seed: int) -> np.ndarray:
    """Payload bytes for (row, K-index j) of each row in ``rows``: [len(rows)][latent_bytes] u8."""
    rows = np.asarray(rows, dtype=np.uint64)
    nw = latent_bytes // 4
    w = np.arange(nw, dtype=np.uint32)[None, :]
    base = _mix_np((rows.astype(np.uint32) * np.uint32(8) + np.uint32(j)) ^ np.uint32(seed & _M32))
    h = _mix_np(base[:, None] ^ _mix_np(w + np.uint32(0x9E3779B9)))
    h[:, 0] = (rows & np.uint64(_M32)).astype(np.uint32)
    if nw > 1:
        h[:, 1] = (rows >> np.uint64(32)).astype(np.uint32)
    if nw > 2:
        h[:, 2] = np.uint32(j)
    if nw > 3:
        h[:, 3] = np.uint32(MAGIC)
    return h.view(np.uint8).reshape(len(rows), nw * 4)


def latents_np(rows, num_k: int, latent_bytes: int, seed: int) -> np.ndarray:
    """[len(rows)][num_k][latent_bytes] u8 (insert layout)."""
    return np.stack([latent_np(rows, j, latent_bytes, seed) for j in range(num_k)], axis=1)


def _mix_t(x):
    import torch  # noqa: F401  (local import: numpy users need not load torch)
    x = x ^ (x >> 16)
    x = (x * 0x21F0AAAD) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x735A2D97) & _M32
    x = x ^ (x >> 15)
    return x


def _normal_t(rows, cols, salt: int):
    """Counter-based standard normals N[row][col] (Box-Muller on two hashed uniforms): a pure
    function of (row, col, salt), so any subset of rows can be regenerated anywhere."""
    import torch
    r = (rows & _M32)[:, None]
    c = (cols & _M32)[None, :]
    h1 = _mix_t((_mix_t(r ^ (salt & _M32)) * 0x9E3779B1 + c) & _M32)
    h2 = _mix_t((h1 ^ 0x85EBCA6B) & _M32)
    u1 = (h1.to(torch.float64) + 0.5) / 4294967296.0
    u2 = (h2.to(torch.float64) + 0.5) / 4294967296.0
    return (torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(6.283185307179586 * u2)).to(torch.float32)


class TorchEntries:
    """On-device variant of ``entries`` for caches too large to draw on the host (C4/C5):
    the same recipe (cluster centres + noise at cos 0.85, Zipf-popular anchors, the Fig. 11
    similarity buckets for queries) but every number is a counter-based hash of (row, dim,
    seed), so row r is identical on every rank and in every call."""

    def __init__(self, n_total: int, seed: int, device, dim: int = D, cos_centre: float = 0.85):
        import torch
        self.n, self.seed, self.device, self.dim = n_total, seed, device, dim
        self.n_c = max(1, n_total // 64)
        cols = torch.arange(dim, dtype=torch.int64, device=device)
        self.cols = cols
        cen = []
        for s in range(0, self.n_c, 65536):
            rr = torch.arange(s, min(self.n_c, s + 65536), dtype=torch.int64, device=device)
            cen.append(_normal_t(rr, cols, seed * 7 + 1))
        c = torch.cat(cen)
        self.centres = c / c.norm(dim=1, keepdim=True)
        self.sigma = float(np.sqrt((1.0 / cos_centre ** 2 - 1.0) / dim))

    def cluster(self, rows):
        return _mix_t((rows & _M32) ^ (self.seed & _M32)) % self.n_c

    def rows(self, rows):
        """fp32 unit rows [len(rows)][dim] for an int64 tensor of row indices."""
        x = self.centres[self.cluster(rows)] + self.sigma * _normal_t(rows, self.cols, self.seed * 7 + 2)
        return x / x.norm(dim=1, keepdim=True)

    def queries(self, b: int, qseed: int, zipf_s: float = 1.0):
        """b queries around Zipf(zipf_s)-popular anchor rows with the bucket mixture of
        ``queries``.  Returns (q [b][dim] fp32, anchor rows, target cos)."""
        import torch
        rng = np.random.default_rng(qseed)
        # bounded Zipf(1) over the n rows by inverse CDF: P(rank <= k) ~ ln k / ln n
        ranks = np.floor(np.exp(rng.random(b) * np.log(self.n))).astype(np.int64) if zipf_s > 0 \
            else rng.integers(1, self.n, b)
        perm_a = np.uint64(rng.integers(1, 2 ** 31) | 1)
        anchor = ((ranks.astype(np.uint64) * perm_a) % np.uint64(self.n)).astype(np.int64)
        probs = np.array([w for _, _, w in BUCKETS])
        bk = rng.choice(len(BUCKETS), size=b, p=probs / probs.sum())
        lo = np.maximum(np.array([BUCKETS[i][0] for i in bk]), 0.40)
        hi = np.array([BUCKETS[i][1] for i in bk])
        t = np.clip(lo + (hi - lo) * rng.random(b), 0.40, 0.999)
        sig = torch.from_numpy(np.sqrt((1.0 / t ** 2 - 1.0) / self.dim)).to(self.device, torch.float32)
        a = torch.from_numpy(anchor).to(self.device)
        qrows = torch.arange(b, dtype=torch.int64, device=self.device) + (qseed * 1_000_003) % (1 << 30)
        q = self.rows(a) + sig[:, None] * _normal_t(qrows, self.cols, self.seed * 7 + 3)
        return q / q.norm(dim=1, keepdim=True), anchor, t


def latents_torch(row0: int, n: int, num_k: int, latent_bytes: int, seed: int, device):
    """Same bytes as ``latents_np(range(row0, row0+n), ...)`` generated with torch int64 ops
    on ``device``: returns a uint8 tensor [n][num_k][latent_bytes]."""
    import torch
    nw = latent_bytes // 4
    rows = torch.arange(row0, row0 + n, dtype=torch.int64, device=device)
    w = torch.arange(nw, dtype=torch.int64, device=device)
    mw = _mix_t((w + 0x9E3779B9) & _M32)
    out = torch.empty((n, num_k, nw), dtype=torch.int32, device=device)
    for j in range(num_k):
        base = _mix_t((((rows & _M32) * 8 + j) & _M32) ^ (seed & _M32))
        h = _mix_t(base[:, None] ^ mw[None, :])
        if nw > 0:
            h[:, 0] = rows & _M32
        if nw > 1:
            h[:, 1] = rows >> 32
        if nw > 2:
            h[:, 2] = j
        if nw > 3:
            h[:, 3] = MAGIC
        out[:, j, :] = (h - ((h >> 31) << 32)).to(torch.int32)  # reinterpret u32 -> i32 bits
    return out.view(torch.uint8).view(n, num_k, nw * 4)


# ---------------- the hand-worked exact cache H ------------------------------
def hand_vectors(dim: int = D):
    """u0..u4: unit vectors with dyadic components (||u||^2 = 1 exactly), zero padded."""
    comps = [
        [1.0, 0, 0, 0, 0],
        [0.75, 0.5, 0.25, 0.25, 0.25],
        [0.5, 0.5, 0.5, 0.5, 0],
        [0.875, 0.375, 0.25, 0.125, 0.125],
        [0.9375, 0.25, 0.125, 0.125, 0.125, 0.0625, 0.0625, 0.0625],
    ]
    out = np.zeros((5, dim), dtype=np.float32)
    for i, c in enumerate(comps):
        out[i, : len(c)] = c
    return out
