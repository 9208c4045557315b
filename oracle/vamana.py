"""ORACLE — test infrastructure only. Graph construction restated in numpy.

  * medoid: f64 mean, f64 einsum distances, lowest id         graph.py:159-171
  * robust_prune: (dist, id) order, alpha^2 * d* > d keeps    graph.py:174-228
  * pairwise distance, rows in the data role, pivot last      build.py:105-134
  * reverse-edge buffer sorted by (target, dist, source)      build.py:65-102
  * seed batch, 3-phase batch insert, group merge             build.py:246-348
  * connectivity repair (BFS + nearest-donor bridges)         build.py:137-224
  * two_pass refinement (search + prune at the final alpha)   build.py:351-386
  * quantized construction (RaBitQ estimates everywhere)      build.py:105-111, 124-129, 322-325
  * build schedule (R+1 doubling, entry -> medoid)            build.py:389-424
  * insert_stream chunking                                    build.py:427-447

The graph is a plain dict-free structure: adjacency int32[cap, R] padded -1,
degrees int32[cap], entry, active.
"""

from __future__ import annotations

import numpy as np

from . import rabitq as orq
from .search import ExactSource, beam_search


class Graph:
    def __init__(self, capacity: int, R: int):
        self.adj = np.full((capacity, R), -1, dtype=np.int32)
        self.deg = np.zeros(capacity, dtype=np.int32)
        self.R = R
        self.entry = 0
        self.active = 0

    def nbrs(self, u: int) -> np.ndarray:
        return self.adj[u, : self.deg[u]].copy()

    def put(self, u: int, ids) -> None:
        ids = np.asarray(ids, dtype=np.int32).ravel()
        assert ids.size <= self.R
        if ids.size:
            assert ids.min() >= 0 and ids.max() < self.active and not (ids == u).any()
            assert np.unique(ids).size == ids.size
        self.adj[u, : ids.size] = ids
        self.adj[u, ids.size:] = -1
        self.deg[u] = ids.size


class Pairwise:
    """build.py:105-134 (exact branch; u8 rows in exact int64, build.py:116-118, 132-133)."""

    def __init__(self, x: np.ndarray):
        self.integer = x.dtype == np.uint8
        self.x = x.astype(np.int64) if self.integer else x
        self.n = np.einsum("nd,nd->n", self.x, self.x)

    def __call__(self, pivot: int, ids) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        dots = np.einsum("md,d->m", self.x[ids], self.x[pivot])
        d = self.n[ids] - 2 * dots + self.n[pivot]
        if self.integer:
            return d.astype(np.float64)
        return np.maximum(d, np.float32(0)).astype(np.float64)


class Quant:
    """A fitted RaBitQ index (centroid, codes, meta, bits, seed) as a construction
    source: phase-1 searches bind the batch rows (build.py:322-325) and every
    pairwise distance binds the pivot row and estimates the ids (build.py:124-129)."""

    def __init__(self, centroid, codes, meta, bits: int, seed: int):
        self.centroid, self.codes, self.meta, self.bits, self.seed = centroid, codes, meta, bits, seed

    def source(self, queries: np.ndarray):
        return orq.QuantSource(self.codes, self.meta, self.bits, queries.shape[1],
                               *orq.bind(queries, self.centroid, self.bits, self.seed))

    def pairwise(self, x: np.ndarray):
        return QuantPairwise(self, x)


class QuantPairwise:
    def __init__(self, quant: Quant, x: np.ndarray):
        self.quant, self.x = quant, np.ascontiguousarray(x, dtype=np.float32)

    def __call__(self, pivot: int, ids) -> np.ndarray:
        ids = np.asarray(ids, dtype=np.int64)
        src = self.quant.source(self.x[pivot][None, :])
        return src(np.zeros(ids.size, dtype=np.int64), ids).astype(np.float64)


def medoid(x: np.ndarray) -> int:
    if x.shape[0] == 0:
        raise ValueError("medoid of an empty dataset")
    x64 = x.astype(np.float64)
    diff = x64 - x64.mean(axis=0)
    return int(np.argmin(np.einsum("nd,nd->n", diff, diff)))


def robust_prune(p: int, ids, dists, alpha: float, R: int, dist) -> tuple[np.ndarray, np.ndarray]:
    if alpha < 1.0:
        raise ValueError("alpha must be >= 1")
    if R < 1:
        raise ValueError("degree_cap must be >= 1")
    ids = np.asarray(ids, dtype=np.int64).ravel()
    ds = np.asarray(dists, dtype=np.float64).ravel()
    if ids.shape != ds.shape:
        raise ValueError("candidate ids and dists length mismatch")
    if (ids == p).any():
        raise ValueError("candidate set must not contain the pivot")
    if np.unique(ids).size != ids.size:
        raise ValueError("candidate set must be deduplicated")
    o = np.lexsort((ids, ds))
    ids, ds = ids[o], ds[o]
    a2 = float(alpha) * float(alpha)
    out_i, out_d = [], []
    while ids.size and len(out_i) < R:
        s = int(ids[0])
        out_i.append(s)
        out_d.append(float(ds[0]))
        ids, ds = ids[1:], ds[1:]
        if not ids.size:
            break
        survive = a2 * np.asarray(dist(s, ids), dtype=np.float64) > ds
        ids, ds = ids[survive], ds[survive]
    return np.asarray(out_i, dtype=np.int32), np.asarray(out_d, dtype=np.float64)


def reachable(g: Graph) -> np.ndarray:
    seen = np.zeros(g.active, dtype=bool)
    seen[g.entry] = True
    front = np.array([g.entry])
    while front.size:
        nxt = g.adj[front].ravel()
        nxt = nxt[nxt >= 0]
        nxt = np.unique(nxt[~seen[nxt]])
        seen[nxt] = True
        front = nxt
    return seen


def repair(g: Graph, dist: Pairwise) -> int:
    """build.py:154-224."""
    if g.active < 2:
        return 0
    R = g.R
    fan = min(R, 16)
    bridges = 0
    pins: dict[int, set] = {}
    while True:
        seen = reachable(g)
        lost = np.flatnonzero(~seen)
        if not lost.size:
            return bridges
        ok = np.flatnonzero(seen)
        donors = np.empty((lost.size, fan), dtype=np.int64)
        best = np.empty(lost.size)
        for i, x in enumerate(lost):
            d = dist(int(x), ok)
            top = np.argpartition(d, min(fan, d.size) - 1)[:fan]
            top = top[np.lexsort((ok[top], d[top]))]
            donors[i] = ok[top]
            best[i] = d[top[0]]
        for i in np.lexsort((lost, best)):
            x = int(lost[i])
            if seen[x]:
                continue
            placed = False
            for u in donors[i]:
                u = int(u)
                row = g.nbrs(u)
                pin = pins.setdefault(u, set())
                if row.size >= R:
                    ev = row[~np.isin(row, list(pin))] if pin else row
                    if not ev.size:
                        continue
                    drop = ev[np.argmax(dist(u, ev))]
                    row = row[row != drop]
                g.put(u, np.append(row, x))
                pin.add(x)
                bridges += 1
                placed = True
                break
            if not placed:
                raise RuntimeError(f"connectivity repair: no donor for vertex {x}")
            front = np.array([x])
            seen[x] = True
            while front.size:
                nxt = g.adj[front].ravel()
                nxt = nxt[nxt >= 0]
                nxt = np.unique(nxt[~seen[nxt]])
                seen[nxt] = True
                front = nxt


def batch_insert(g: Graph, x: np.ndarray, start: int, stop: int, R: int, L: int, alpha: float,
                 dist: Pairwise | None = None, always_prune=False, reverse_all=False, quant: Quant | None = None) -> int:
    """build.py:296-348. Returns the number of repair bridges."""
    if start == stop:
        return 0
    dist = dist or (quant.pairwise(x) if quant is not None else Pairwise(x))
    if g.active == 0:
        g.active = stop
        g.entry = medoid(x[:stop])
        if stop - start > 1:
            everyone = np.arange(start, stop)
            for v in range(start, stop):
                rest = everyone[everyone != v]
                kept, _ = robust_prune(v, rest, dist(v, rest), alpha, R, dist)
                g.put(v, kept)
        return repair(g, dist)
    src = quant.source(x[start:stop]) if quant is not None else ExactSource(x, x[start:stop])
    found = beam_search(g.adj, g.active, g.entry, src, stop - start, L)
    g.active = stop
    tgt, srcs, dd = [], [], []
    for v, res in zip(range(start, stop), found):
        kept, kd = robust_prune(v, res.visited_ids, res.visited_dists, alpha, R, dist)
        g.put(v, kept)
        e_ids, e_d = (res.visited_ids, res.visited_dists) if reverse_all else (kept, kd)
        tgt.append(np.asarray(e_ids, dtype=np.int64))
        srcs.append(np.full(len(e_ids), v, dtype=np.int64))
        dd.append(np.asarray(e_d, dtype=np.float64))
    merge_reverse(g, tgt, srcs, dd, R, alpha, dist, always_prune)
    return repair(g, dist)


def merge_reverse(g: Graph, tgt, srcs, dd, R: int, alpha: float, dist, always_prune=False) -> None:
    """build.py:269-293 over EdgeBuffer order (target, dist, source), build.py:65-102."""
    if tgt:
        t = np.concatenate(tgt)
        s = np.concatenate(srcs)
        d = np.concatenate(dd)
        o = np.lexsort((s, d, t))
        t, s, d = t[o], s[o], d[o]
        heads = np.flatnonzero(np.r_[True, t[1:] != t[:-1]])
        bounds = np.r_[heads, t.size]
        for a, b in zip(bounds[:-1], bounds[1:]):
            target = int(t[a])
            have = g.nbrs(target)
            keep = ~np.isin(s[a:b], have)
            fs, fd = s[a:b][keep], d[a:b][keep]
            if not fs.size:
                continue
            if not always_prune and have.size + fs.size <= R:
                g.put(target, np.concatenate([have, fs.astype(np.int32)]))
                continue
            hd = dist(target, have) if have.size else np.empty(0)
            kept, _ = robust_prune(target, np.concatenate([have.astype(np.int64), fs]),
                                   np.concatenate([np.asarray(hd, dtype=np.float64), fd]), alpha, R, dist)
            g.put(target, kept)


def refine_pass(g: Graph, x: np.ndarray, R: int, L: int, alpha: float, max_batch: int,
                dist: Pairwise | None = None, always_prune=False, quant: Quant | None = None) -> int:
    """build.py:351-386: per max_batch slice, search every active vertex on the
    current graph, prune it over (visited - itself) + (current neighbours missing
    from the trace) at the final alpha, then the grouped reverse merge; repair last."""
    dist = dist or (quant.pairwise(x) if quant is not None else Pairwise(x))
    n = g.active
    for lo in range(0, n, max_batch):
        hi = min(n, lo + max_batch)
        src = quant.source(x[lo:hi]) if quant is not None else ExactSource(x, x[lo:hi])
        found = beam_search(g.adj, g.active, g.entry, src, hi - lo, L)
        tgt, srcs, dd = [], [], []
        for v, res in zip(range(lo, hi), found):
            cur = g.nbrs(v)
            extra = cur[~np.isin(cur, res.visited_ids)]
            cand = np.concatenate([np.asarray(res.visited_ids, dtype=np.int64), extra.astype(np.int64)])
            cd = np.concatenate([np.asarray(res.visited_dists, dtype=np.float64),
                                 dist(v, extra) if extra.size else np.empty(0)])
            keep = cand != v
            kept, kd = robust_prune(v, cand[keep], cd[keep], alpha, R, dist)
            g.put(v, kept)
            tgt.append(np.asarray(kept, dtype=np.int64))
            srcs.append(np.full(len(kept), v, dtype=np.int64))
            dd.append(np.asarray(kd, dtype=np.float64))
        merge_reverse(g, tgt, srcs, dd, R, alpha, dist, always_prune)
    return repair(g, dist)


def build(x: np.ndarray, R: int, L: int, alpha: float, max_batch: int = 100_000, two_pass: bool = False,
          quant: Quant | None = None) -> Graph:
    """build.py:389-424 (two_pass: insertion passes at alpha=1, then refine_pass)."""
    x = np.ascontiguousarray(x) if np.asarray(x).dtype == np.uint8 else np.ascontiguousarray(x, dtype=np.float32)
    n = x.shape[0]
    if n == 0:
        raise ValueError("cannot build over an empty dataset")
    g = Graph(n, R)
    dist = quant.pairwise(x) if quant is not None else Pairwise(x)
    m = medoid(x)
    size, pos = R + 1, 0
    while pos < n:
        stop = min(n, pos + size)
        batch_insert(g, x, pos, stop, R, L, 1.0 if two_pass else alpha, dist, quant=quant)
        if m < g.active and g.entry != m:
            g.entry = m
            repair(g, dist)
        pos = stop
        size = min(size * 2, max_batch)
    if two_pass:
        refine_pass(g, x, R, L, alpha, max_batch, dist, quant=quant)
    return g


def insert_stream(g: Graph, x: np.ndarray, start: int, stop: int, R: int, L: int, alpha: float,
                  max_batch: int) -> None:
    dist = Pairwise(x)
    pos = start
    while pos < stop:
        nxt = min(stop, pos + max_batch)
        batch_insert(g, x, pos, nxt, R, L, alpha, dist)
        pos = nxt
