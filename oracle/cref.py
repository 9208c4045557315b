"""ORACLE — test infrastructure only. ctypes front of the C restatement (oracle/c/jbo.c).

The same algorithm as oracle/search.py and oracle/vamana.py (and so as the
reference, pkg/src/beamann), multi-threaded on the host cores. bench.py's CPU
legs use it to build and search the 1M-vector workload without a GPU and
without the product library; tests/test_oracle_c.py pins it to the reference
fixtures and to the numpy oracle.

  * build schedule (R+1 doubling, entry -> medoid, repair)   build.py:389-424
  * batch_insert (seed batch, 3 phases, repair)              build.py:246-348
  * run_beam_searches (lockstep), exact / RaBitQ sources     search.py:171-304, rabitq.py:225-244
  * search_knn_batch tail (rerank + top-k)                    search.py:351-383
  * exact_knn (f64 scores, stable order)                     oracle.py:20-62
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import rabitq as orq
from .search import UMAX, Result, unpack_dist, unpack_id

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libjbo.so")
SRC = os.path.join(HERE, "c", "jbo.c")

_lib = None


def build_library() -> str:
    """Compile oracle/c/jbo.c -> oracle/libjbo.so (make; gcc with OpenMP)."""
    if not os.path.exists(LIB) or (os.path.exists(SRC) and os.path.getmtime(LIB) < os.path.getmtime(SRC)):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "c")], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build_library()
        L = ctypes.CDLL(LIB)
        P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
        L.jbo_search.argtypes = [P, I, I64, I, P, P, P, P, I, I, P, P, P, I64, P, I, I, P, P, P]
        L.jbo_search.restype = I
        L.jbo_rerank_topk.argtypes = [P, I, P, I64, P, I, I, I, P, P]
        L.jbo_rerank_topk.restype = I
        L.jbo_row_norms.argtypes = [P, I64, I, P, I]
        L.jbo_row_norms.restype = None
        L.jbo_medoid.argtypes = [P, I64, I]
        L.jbo_medoid.restype = I64
        L.jbo_topk_rows.argtypes = [P, I64, I64, I, I, P, P]
        L.jbo_topk_rows.restype = I
        L.jbo_repair.argtypes = [P, P, I, I64, I64, P, P, I, I]
        L.jbo_repair.restype = I64
        L.jbo_batch_insert.argtypes = [P, P, I, P, P, P, P, I, I64, I64, I, D, I64, I, I, I]
        L.jbo_batch_insert.restype = I64
        L.jbo_num_threads.restype = I
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(lib().jbo_num_threads())


def row_norms(x: np.ndarray, threads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    out = np.empty(x.shape[0], dtype=np.float32)
    lib().jbo_row_norms(_p(x), x.shape[0], x.shape[1], _p(out), threads)
    return out


def medoid(x: np.ndarray) -> int:
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.shape[0] == 0:
        raise ValueError("medoid of an empty dataset")
    return int(lib().jbo_medoid(_p(x), x.shape[0], x.shape[1]))


class Graph:
    """The reference's GraphIndex slab: int32 [capacity, R] padded -1, degrees, entry, active."""

    def __init__(self, capacity: int, R: int):
        self.adj = np.full((capacity, R), -1, dtype=np.int32)
        self.deg = np.zeros(capacity, dtype=np.int32)
        self.R = R
        self.entry = 0
        self.active = 0


def _check_bridges(r: int) -> int:
    if r <= -1_000_000_000_000:
        raise RuntimeError(f"connectivity repair: no donor for vertex {-(r + 1_000_000_000_000) - 1}")
    if r < 0:
        raise ValueError(f"oracle batch_insert failed ({r})")
    return int(r)


class Rows:
    """f32 rows with their A1 norms (build.py:120)."""

    def __init__(self, x: np.ndarray, threads: int = 0):
        self.x = np.ascontiguousarray(x, dtype=np.float32)
        self.xn = row_norms(self.x, threads)


def batch_insert(g: Graph, rows: Rows, start: int, stop: int, L: int, alpha: float, always_prune=False,
                 reverse_all=False, threads: int = 0) -> int:
    """build.py:296-348. Returns the repair bridge count."""
    if start == stop:
        return 0
    a = np.array([g.active], dtype=np.int64)
    e = np.array([g.entry], dtype=np.int64)
    seed = medoid(rows.x[:stop]) if g.active == 0 else -1
    r = lib().jbo_batch_insert(_p(g.adj), _p(g.deg), g.R, _p(a), _p(e), _p(rows.x), _p(rows.xn), rows.x.shape[1],
                               start, stop, L, float(alpha), seed, int(always_prune), int(reverse_all), threads)
    g.active, g.entry = int(a[0]), int(e[0])
    return _check_bridges(r)


def repair(g: Graph, rows: Rows, threads: int = 0) -> int:
    return _check_bridges(lib().jbo_repair(_p(g.adj), _p(g.deg), g.R, g.active, g.entry, _p(rows.x),
                                           _p(rows.xn), rows.x.shape[1], threads))


def build(x: np.ndarray, R: int, L: int, alpha: float, max_batch: int = 100_000, threads: int = 0,
          rows: Rows | None = None) -> Graph:
    """build.py:389-424 (single pass)."""
    rows = rows or Rows(x, threads)
    n = rows.x.shape[0]
    if n == 0:
        raise ValueError("cannot build over an empty dataset")
    g = Graph(n, R)
    m = medoid(rows.x)
    size, pos = R + 1, 0
    while pos < n:
        stop = min(n, pos + size)
        batch_insert(g, rows, pos, stop, L, alpha, threads=threads)
        if m < g.active and g.entry != m:
            g.entry = m
            repair(g, rows, threads)
        pos = stop
        size = min(size * 2, max_batch)
    return g


def insert_stream(g: Graph, rows: Rows, start: int, stop: int, L: int, alpha: float, max_batch: int,
                  threads: int = 0) -> None:
    """build.py:427-447."""
    pos = start
    while pos < stop:
        nxt = min(stop, pos + max_batch)
        batch_insert(g, rows, pos, nxt, L, alpha, threads=threads)
        pos = nxt


def _search(adj, active, kind, args, nq, starts, L, threads):
    R = adj.shape[1]
    keys = np.empty((nq, L), dtype=np.uint64)
    hops = np.empty(nq, dtype=np.int64)
    evals = np.empty(nq, dtype=np.int64)
    st = np.ascontiguousarray(np.broadcast_to(np.asarray(starts, dtype=np.int64), (nq,)))
    adj = np.ascontiguousarray(adj, dtype=np.int32)
    x, xn, codes, meta, bits, D, q, qv, sumq = args
    rc = lib().jbo_search(_p(adj), R, active, kind, x, xn, codes, meta, bits, D, _p(q), _p(qv), sumq, nq, _p(st), L,
                          threads, _p(keys), _p(hops), _p(evals))
    if rc == -1:
        raise ValueError("search on an empty graph")
    if rc == -2:
        raise ValueError("beam_width must be in [1, 1024]")
    if rc == -4:
        raise ValueError("start vertex out of range")
    if rc:
        raise ValueError(f"oracle search failed ({rc})")
    return keys, hops, evals


def search_exact(adj, active: int, entry: int, rows: Rows, queries: np.ndarray, L: int, starts=None,
                 threads: int = 0):
    """run_beam_searches over ExactDistances: (frontier keys [nq, L] UMAX-padded, hops, evals)."""
    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
    qn = row_norms(q, threads)
    args = (_p(rows.x), _p(rows.xn), None, None, 0, q.shape[1], q, qn, None)
    return _search(adj, active, 0, args, q.shape[0], entry if starts is None else starts, L, threads)


class Quantized:
    """A fitted RaBitQ index (rabitq.py:113-168) as a C search source."""

    def __init__(self, centroid, codes, meta, bits: int, seed: int):
        self.centroid = np.ascontiguousarray(centroid, dtype=np.float32)
        self.codes = np.ascontiguousarray(codes, dtype=np.uint8)
        self.meta = np.ascontiguousarray(meta, dtype=np.float32)
        self.bits, self.seed = bits, seed

    @classmethod
    def fit(cls, x: np.ndarray, bits: int, seed: int) -> "Quantized":
        return cls(*orq.fit(x, bits, seed), bits, seed)


def search_rabitq(adj, active: int, entry: int, quant: Quantized, queries: np.ndarray, L: int, starts=None,
                  threads: int = 0):
    """run_beam_searches over the bound RaBitQ estimator (rabitq.py:170-181, 225-244)."""
    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
    rot, qadd, sumq = orq.bind(q, quant.centroid, quant.bits, quant.seed)
    rot, qadd, sumq = (np.ascontiguousarray(a, dtype=np.float32) for a in (rot, qadd, sumq))
    args = (None, None, _p(quant.codes), _p(quant.meta), quant.bits, q.shape[1], rot, qadd, _p(sumq))
    keys, hops, evals = _search(adj, active, 1, args, q.shape[0], entry if starts is None else starts, L, threads)
    return keys, hops, evals


def frontier_ids(keys: np.ndarray) -> np.ndarray:
    ids = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64).astype(np.int32)
    ids[keys == UMAX] = -1
    return ids


def results(keys: np.ndarray, hops, evals) -> list[Result]:
    """Frontier as oracle.search.Result objects (no trace)."""
    out = []
    for i in range(keys.shape[0]):
        k = keys[i][keys[i] != UMAX]
        out.append(Result(unpack_id(k).astype(np.int32), unpack_dist(k), None, None, int(hops[i]), int(evals[i])))
    return out


def rerank_topk(x: np.ndarray, queries: np.ndarray, fids: np.ndarray, k: int, threads: int = 0):
    """search.py:366-383 with exact rerank: (ids int32 [nq, k] -1 padded, dists f64 inf padded)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
    fids = np.ascontiguousarray(fids, dtype=np.int32)
    nq, L = fids.shape
    oi = np.empty((nq, k), dtype=np.int32)
    od = np.empty((nq, k), dtype=np.float64)
    lib().jbo_rerank_topk(_p(x), x.shape[1], _p(q), nq, _p(fids), L, k, threads, _p(oi), _p(od))
    return oi, od


def exact_knn(data: np.ndarray, queries: np.ndarray, k: int, block: int = 512, threads: int = 0):
    """oracle.py:20-62 (L2): f64 scores xn - 2 q.x + qn clamped at 0, first k of a stable order.
    The f64 GEMM is numpy's (BLAS); the selection is the C top-k."""
    x64 = np.asarray(data).astype(np.float64)
    xn = np.einsum("nd,nd->n", x64, x64)
    ids = np.empty((queries.shape[0], k), dtype=np.int32)
    ds = np.empty((queries.shape[0], k), dtype=np.float64)
    for lo in range(0, queries.shape[0], block):
        q = queries[lo:lo + block].astype(np.float64)
        s = q @ x64.T
        s *= -2.0
        s += xn[None, :]
        s += np.einsum("bd,bd->b", q, q)[:, None]
        np.maximum(s, 0.0, out=s)
        s = np.ascontiguousarray(s)
        lib().jbo_topk_rows(_p(s), s.shape[0], s.shape[1], k, threads, _p(ids[lo:lo + block]), _p(ds[lo:lo + block]))
    return ids, ds
