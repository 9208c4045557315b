"""Greedy beam search on B200 behind the reference's search API (mirror of search.py).

Public functions keep the reference's names, argument meaning, validation
messages and return types:
  run_beam_searches  search.py:272-304   -> list[SearchResult] (frontier + visited trace)
  beam_search        search.py:307-315
  search_knn         search.py:323-348
  search_knn_batch   search.py:351-383   -> (int32 ids [nq,k], f64 dists [nq,k])

Each call is ONE batched launch of the sm_100a kernel (one warp per query)
instead of the reference's per-hop numpy lockstep; frontier, trace, hops and
(when the visited table did not overflow) distance_evals are identical.
`search_knn_batch_device` is the HBM-resident variant used for throughput.
"""

from __future__ import annotations

import os

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import ElementKind, VectorDataset, as_dataset
from .graph import Candidate, GraphIndex, as_graph

__all__ = ["SearchParams", "SearchStats", "SearchResult", "beam_search", "search_knn", "search_knn_batch",
           "run_beam_searches", "search_knn_batch_device", "MAX_BEAM_WIDTH", "ExactDistances", "BoundDistances",
           "bind_distance_source", "MAX_DEGREE_CAP"]

MAX_BEAM_WIDTH = 1024
MAX_DEGREE_CAP = 128  # the search kernel's neighbour chunks: R <= 32 * 4
_UMAX = np.uint64(0xFFFFFFFFFFFFFFFF)
# Test/tuning hook: visited-table slots per query (0 = library default).
TUNING = {"hash_slots": 0}


ESTIMATORS = ("reference", "popcount")


@dataclass(frozen=True)
class SearchParams:
    """search.py:42-54, plus `estimator` for quantized sources:
    "reference" = the reference's float estimator, bit-exact (default);
    "popcount"  = 1-bit codes only, query quantized to 6-bit planes and <u,q>
                  computed with AND + popcount (faster; validated by recall)."""

    beam_width: int
    k: int = 10
    rerank: bool = False
    estimator: str = "reference"

    def __post_init__(self):
        if not 1 <= self.beam_width <= MAX_BEAM_WIDTH:
            raise ValueError(f"beam_width must be in [1, {MAX_BEAM_WIDTH}]")
        if not 1 <= self.k <= self.beam_width:
            raise ValueError("k must satisfy 1 <= k <= beam_width")
        if self.estimator not in ESTIMATORS:
            raise ValueError(f"estimator must be one of {ESTIMATORS}")


@dataclass
class SearchStats:
    hops: int = 0
    distance_evals: int = 0


@dataclass
class SearchResult:
    frontier_ids: np.ndarray
    frontier_dists: np.ndarray
    visited_ids: np.ndarray
    visited_dists: np.ndarray
    stats: SearchStats = field(default_factory=SearchStats)

    @property
    def frontier(self) -> list[Candidate]:
        return [Candidate(int(i), float(d)) for i, d in zip(self.frontier_ids, self.frontier_dists)]

    @property
    def visited(self) -> list[Candidate]:
        return [Candidate(int(i), float(d)) for i, d in zip(self.visited_ids, self.visited_dists)]


def _is_rabitq(source) -> bool:
    from .rabitq import RaBitQIndex

    return isinstance(source, RaBitQIndex) or (hasattr(source, "codes") and hasattr(source, "meta")
                                               and hasattr(source, "rotation_seed"))


class _Bound:
    """Device-side distance source bound to a query block (search.py:159-168)."""

    def __init__(self, source, q_dev, estimator: str = "reference"):
        torch = _lib.require_cuda()
        self.q_dev = q_dev
        nq, D = q_dev.shape
        if _is_rabitq(source):
            from .rabitq import as_rabitq

            idx = as_rabitq(source)
            if D != idx.dims:
                raise ValueError(f"query dims {D} != index dims {idx.dims}")
            dev = idx.device()
            self.kind = _lib.SRC_RABITQ
            self.dims = idx.dims
            self.records, self.record_bytes, self.bits = dev.records, dev.record_bytes, idx.bits
            if estimator == "popcount":
                self.kind = _lib.SRC_RABITQ_FAST
                self.records, self.record_bytes = idx.device_planes()
            self.rows = None
            self.rotated = torch.empty((nq, D), dtype=torch.float32, device=q_dev.device)
            self.qadd = torch.empty(nq, dtype=torch.float32, device=q_dev.device)
            self.qsumq = torch.empty(nq, dtype=torch.float32, device=q_dev.device)
            if nq:
                _lib.check(_lib.lib().jb_rabitq_bind(_lib.ptr(q_dev), nq, D, idx.bits, _lib.ptr(dev.centroid),
                                                     _lib.ptr(dev.rotation), _lib.ptr(self.rotated),
                                                     _lib.ptr(self.qadd), _lib.ptr(self.qsumq), _lib.stream_ptr()))
            self.count = idx.count
        else:
            ds = as_dataset(source)
            if D != ds.dims:
                raise ValueError(f"query dims {D} != dataset dims {ds.dims}")
            dev = ds.device()
            self.dims = ds.dims
            self.rows = dev
            self.records, self.record_bytes, self.bits = None, 0, 0
            self.rotated = q_dev
            self.qsumq = None
            if ds.element_kind is ElementKind.U8:  # integer distances (search.py:92-99)
                if q_dev.dtype != torch.uint8:
                    raise ValueError("u8 dataset requires u8 queries")
                self.kind = _lib.SRC_EXACT_U8
                self.qadd = torch.empty(nq, dtype=torch.int32, device=q_dev.device)
                if nq:
                    _lib.check(_lib.lib().jb_row_sq_norms_u8(_lib.ptr(q_dev), nq, D, _lib.ptr(self.qadd),
                                                            _lib.stream_ptr()))
            else:
                self.kind = _lib.SRC_EXACT
                self.screen = _screen(ds)
                self.qadd = torch.empty(nq, dtype=torch.float32, device=q_dev.device)
                if nq:
                    _lib.check(_lib.lib().jb_row_sq_norms(_lib.ptr(q_dev), nq, D, _lib.ptr(self.qadd),
                                                         _lib.stream_ptr()))
            self.count = ds.count


class _Pinned(threading.local):
    """Per-thread pinned staging buffers for host<->HBM copies (reused across calls,
    so the public host-array API pays one async copy each way, not a pin per call)."""

    def __init__(self):
        self.bufs = {}

    def get(self, name: str, nbytes: int):
        torch = _lib.require_cuda()
        b = self.bufs.get(name)
        if b is None or b.numel() < nbytes:
            b = torch.empty(max(nbytes, 1 << 16), dtype=torch.uint8, pin_memory=True)
            self.bufs[name] = b
        return b


_PINNED = _Pinned()


def _is_u8(source) -> bool:
    return not _is_rabitq(source) and as_dataset(source).element_kind is ElementKind.U8


def _queries_to_device(queries, u8: bool = False):
    """Query rows to HBM: f32, or (u8 source) uint8 — a u8 dataset requires u8
    queries (search.py:107-110)."""
    torch = _lib.require_cuda()
    if isinstance(queries, torch.Tensor):
        q = queries
        if q.dim() == 1:
            q = q[None, :]
        if u8:
            if q.dtype != torch.uint8:
                raise ValueError("u8 dataset requires u8 queries")
            return q.to(device="cuda").contiguous()
        return q.to(device="cuda", dtype=torch.float32).contiguous()
    q = np.atleast_2d(np.asarray(queries))
    if u8:
        if q.dtype != np.uint8:
            raise ValueError("u8 dataset requires u8 queries")
        return torch.from_numpy(np.ascontiguousarray(q)).to("cuda")
    q = np.ascontiguousarray(q, dtype=np.float32)
    if q.size == 0:
        return torch.empty(q.shape, dtype=torch.float32, device="cuda")
    buf = _PINNED.get("q", q.nbytes)
    host = buf[: q.nbytes].view(torch.float32).view(q.shape)
    host.numpy()[...] = q
    return host.to("cuda", non_blocking=True)


def _to_host(*tensors):
    """Async D2H of device tensors through pinned buffers, one stream sync, numpy copies out."""
    torch = _lib.require_cuda()
    outs = []
    for i, t in enumerate(tensors):
        nb = t.numel() * t.element_size()
        buf = _PINNED.get(f"out{i}", nb)
        h = buf[:nb].view(t.dtype).view(t.shape)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return [h.numpy().copy() for h in outs]


def _screen(ds):
    """Int8 screen records of an f32 dataset for the exact search (extension,
    jb_search_args.screen; identical results), or None. JB_SEARCH_SCREEN=0: off."""
    if os.environ.get("JB_SEARCH_SCREEN", "1") == "0":
        return None
    return ds.device_screen()


def _source_args(a, bound: _Bound) -> None:
    """Fill the distance-source + bound-query fields of a jb_search_args."""
    a.source = bound.kind
    a.dims = bound.dims
    if bound.kind == _lib.SRC_EXACT_U8:
        a.data_u8, a.norms_u32 = _lib.ptr(bound.rows.x), _lib.ptr(bound.rows.norms)
        a.queries_u8, a.query_norms_u32 = _lib.ptr(bound.rotated), _lib.ptr(bound.qadd)
    elif bound.kind == _lib.SRC_EXACT:
        a.data = _lib.ptr(bound.rows.x)
        a.data_norms = _lib.ptr(bound.rows.norms)
        scr = getattr(bound, "screen", None)
        if scr is not None:
            a.screen, a.screen_center = _lib.ptr(scr[0]), _lib.ptr(scr[1])
    else:
        a.records = _lib.ptr(bound.records)
        a.record_bytes = bound.record_bytes
        a.bits = bound.bits
    a.queries = _lib.ptr(bound.rotated)
    a.query_add = _lib.ptr(bound.qadd)
    a.query_sumq = _lib.ptr(bound.qsumq)


def _pack_keys(dists, ids, is_integer: bool) -> np.ndarray:
    """search.py:139-145: (f32 bits of max(d, 0) | integer distance) << 32 | id."""
    dists = np.asarray(dists)
    if is_integer:
        hi = dists.astype(np.uint64)
    else:
        hi = np.maximum(dists.astype(np.float32, copy=False), np.float32(0.0)).view(np.uint32).astype(np.uint64)
    return (hi << np.uint64(32)) | np.asarray(ids).astype(np.uint64)


def _decode_keys(keys, is_integer: bool) -> np.ndarray:
    """search.py:148-152."""
    hi = np.asarray(keys, dtype=np.uint64) >> np.uint64(32)
    if is_integer:
        return hi.astype(np.float64)
    return hi.astype(np.uint32).view(np.float32).astype(np.float64)


class BoundDistances:
    """A distance source bound to a query block (search.py:133-156 `_BoundExact`,
    rabitq.py:225-254 `_BoundQuantized`), held in HBM: `distances(qrows, ids)` is
    one jb_bound_distances launch in the search kernel's rounding (exact A1 f32,
    exact integers for u8 rows, the reference RaBitQ estimator)."""

    def __init__(self, source, queries, *, u8: bool | None = None):
        u8 = _is_u8(source) if u8 is None else u8
        q_dev = _queries_to_device(queries, u8)
        self._bound = _Bound(source, q_dev)
        self.source = source
        self.is_integer = self._bound.kind == _lib.SRC_EXACT_U8
        self.n_queries = int(q_dev.shape[0])
        self._padded = None

    def distances_device(self, qrows, ids):
        """Device tensors in, device tensor out (f32, or int64 for u8 rows)."""
        torch = _lib.require_cuda()
        qr = torch.as_tensor(qrows, dtype=torch.int64).reshape(-1).to("cuda")
        ii = torch.as_tensor(ids, dtype=torch.int64).reshape(-1).to("cuda")
        if qr.numel() != ii.numel():
            raise ValueError("qrows and ids length mismatch")
        n = int(ii.numel())
        if n:
            lo = torch.stack([qr.min(), ii.min()]).cpu()
            hi = torch.stack([qr.max(), ii.max()]).cpu()
            if lo.min() < 0 or int(hi[0]) >= self.n_queries or int(hi[1]) >= self._bound.count:
                raise IndexError("query row or vector id out of range")
        out = torch.empty(n, dtype=torch.int32 if self.is_integer else torch.float32, device="cuda")
        a = _lib.SearchArgs()
        _source_args(a, self._bound)
        stride = 0
        if self._bound.kind in (_lib.SRC_RABITQ, _lib.SRC_EXACT_U8):
            # the estimator / u8 dot read 16-byte words of the query row: pad the row stride
            D = self._bound.dims
            stride = (D + 15) // 16 * 16 if self.is_integer else (D + 3) // 4 * 4
            if stride != D:
                if self._padded is None:
                    src = self._bound.rotated
                    self._padded = torch.zeros((src.shape[0], stride), dtype=src.dtype, device=src.device)
                    self._padded[:, :D] = src
                if self.is_integer:
                    a.queries_u8 = _lib.ptr(self._padded)
                else:
                    a.queries = _lib.ptr(self._padded)
        _lib.check(_lib.lib().jb_bound_distances(_lib.C.byref(a), stride, _lib.ptr(qr), _lib.ptr(ii), n,
                                                 _lib.ptr(out), _lib.stream_ptr()))
        if self.is_integer:  # u32 distances (D * 255^2 < 2^32) -> int64 like the reference
            return out.to(torch.int64) & 0xFFFFFFFF
        return out

    def distances(self, qrows, ids) -> np.ndarray:
        """search.py:121-130 / rabitq.py:235-244: f32 (clamped at 0), or int64 for u8 rows."""
        qrows = np.asarray(qrows, dtype=np.int64)
        ids = np.asarray(ids, dtype=np.int64)
        shape = np.broadcast_shapes(qrows.shape, ids.shape)
        qrows, ids = np.broadcast_to(qrows, shape), np.broadcast_to(ids, shape)
        return self.distances_device(np.ascontiguousarray(qrows), np.ascontiguousarray(ids)).cpu().numpy().reshape(
            shape)

    def pack(self, dists, ids) -> np.ndarray:
        return _pack_keys(dists, ids, self.is_integer)

    def decode(self, keys) -> np.ndarray:
        return _decode_keys(keys, self.is_integer)


class ExactDistances:
    """search.py:82-116: squared distances over raw vectors; `bind(queries)` -> BoundDistances."""

    def __init__(self, dataset):
        self.dataset = as_dataset(dataset)
        self.is_integer = self.dataset.element_kind is ElementKind.U8
        if self.is_integer and self.dataset.dims * 255 ** 2 >= 1 << 32:
            raise ValueError("u8 dims too large for 32-bit packed distances")

    def bind(self, queries) -> BoundDistances:
        q = np.atleast_2d(np.asarray(queries)) if not _is_tensor(queries) else queries
        if q.shape[-1] != self.dataset.dims:
            raise ValueError(f"query dims {q.shape[-1]} != dataset dims {self.dataset.dims}")
        return BoundDistances(self.dataset, q, u8=self.is_integer)


def _is_tensor(x) -> bool:
    return type(x).__module__.startswith("torch")


def bind_distance_source(source, queries) -> BoundDistances:
    """search.py:159-168: bind a dataset or a quantized index to a query block."""
    if isinstance(source, VectorDataset) or (hasattr(source, "element_kind") and hasattr(source, "data")
                                             and not _is_rabitq(source)):
        return ExactDistances(source).bind(queries)
    if _is_rabitq(source):
        from .rabitq import as_rabitq

        return as_rabitq(source).bind(queries)
    raise TypeError(f"unsupported distance source {type(source).__name__}")


def _check_counts(graph: GraphIndex, source, exact_data=None, rerank: bool = False) -> None:
    """The kernels read records/rows by id: a source (or rerank rows) shorter than
    the graph's active vertices would be read out of bounds. The reference raises
    IndexError from codes[ids] / data[ids]; this raises before any launch."""
    n = as_rabitq_count(source)
    if n < graph.active_count:
        raise ValueError(f"distance source holds {n} vectors but the graph has {graph.active_count} active")
    if rerank and exact_data is not None and as_dataset(exact_data).count < graph.active_count:
        raise ValueError(f"exact_data holds {as_dataset(exact_data).count} rows but the graph has "
                         f"{graph.active_count} active")


def as_rabitq_count(source) -> int:
    if _is_rabitq(source):
        return int(np.asarray(source.codes).shape[0])
    return as_dataset(source).count


def _rerank_rows(exact_data):
    """f32 rows for the exact rerank: u8 rows are widened exactly (the reference's
    data[ids].astype(f32), search.py:318-320)."""
    ds = as_dataset(exact_data)
    return ds.device_f32(), ds.dims


def _launch(graph: GraphIndex, bound: _Bound, L: int, starts_dev=None, trace_cap: int = 0, out=None):
    torch = _lib.require_cuda()
    nq = bound.q_dev.shape[0]
    adj, _ = graph.device()
    dev = bound.q_dev.device
    fk = torch.empty((nq, L), dtype=torch.int64, device=dev) if out is None else out
    hops = torch.empty(nq, dtype=torch.int32, device=dev)
    evals = torch.empty(nq, dtype=torch.int32, device=dev)
    flags = torch.empty(nq, dtype=torch.int32, device=dev)
    tids = tdst = None
    if trace_cap:  # slots past a query's hop count stay -1 / 0 (defined when copied out whole)
        tids = torch.full((nq, trace_cap), -1, dtype=torch.int32, device=dev)
        tdst = torch.zeros((nq, trace_cap), dtype=torch.float32, device=dev)
    a = _lib.SearchArgs()
    a.adjacency = _lib.ptr(adj)
    a.degree_cap = graph.degree_cap
    a.active_count = graph.active_count
    _source_args(a, bound)
    a.nq = nq
    a.starts = _lib.ptr(starts_dev)
    a.start_vertex = graph.entry_point
    a.beam_width = L
    a.hash_slots = int(TUNING["hash_slots"])
    a.trace_cap = trace_cap
    a.frontier_keys = _lib.ptr(fk)
    a.hops = _lib.ptr(hops)
    a.evals = _lib.ptr(evals)
    a.trace_ids = _lib.ptr(tids)
    a.trace_dists = _lib.ptr(tdst)
    a.flags = _lib.ptr(flags)
    _lib.check(_lib.lib().jb_beam_search(_lib.C.byref(a), _lib.stream_ptr()))
    return fk, hops, evals, flags, tids, tdst


def _validate(graph: GraphIndex, beam_width: int):
    if graph.active_count == 0:
        raise ValueError("search on an empty graph")
    if not 1 <= beam_width <= MAX_BEAM_WIDTH:
        raise ValueError(f"beam_width must be in [1, {MAX_BEAM_WIDTH}]")
    if graph.degree_cap > MAX_DEGREE_CAP:
        raise ValueError(f"degree_cap {graph.degree_cap} exceeds the search kernel's limit {MAX_DEGREE_CAP}")


def _starts(graph: GraphIndex, starts, nq: int):
    if starts is None:
        return None
    s = np.broadcast_to(np.asarray(starts, dtype=np.int64), (nq,)).copy()
    if s.size and (s.min() < 0 or s.max() >= graph.active_count):
        raise ValueError("start vertex out of range")
    torch = _lib.require_cuda()
    return torch.from_numpy(s.astype(np.int32)).cuda()


def run_beam_searches(graph, source, queries, beam_width: int, starts=None) -> list[SearchResult]:
    """search.py:272-304: one SearchResult (frontier + visited trace + stats) per query row."""
    graph = as_graph(graph)
    _validate(graph, beam_width)
    _check_counts(graph, source)
    u8 = _is_u8(source)
    q_dev = _queries_to_device(queries, u8)
    nq = q_dev.shape[0]
    starts_dev = _starts(graph, starts, nq)
    bound = _Bound(source, q_dev)
    cap = max(2 * beam_width, beam_width + 64)
    fk, hops, evals, flags, tids, tdst = _launch(graph, bound, beam_width, starts_dev, cap)
    hops_h = hops.cpu().numpy()
    over = np.nonzero(hops_h > cap)[0]
    if not over.size:
        # queries whose visited table evicted ids counted re-evaluations: recount them
        # on device as |{start} U N(expanded)| (the reference's count)
        adj, _ = graph.device()
        _lib.check(_lib.lib().jb_count_evals(_lib.ptr(adj), graph.degree_cap, _lib.ptr(tids), cap, _lib.ptr(hops),
                                             _lib.ptr(starts_dev), graph.entry_point, _lib.ptr(flags), nq,
                                             _lib.ptr(evals), _lib.stream_ptr()))
        flags.zero_()
    if over.size:  # trace buffer overflowed for a few queries: re-run exactly those with a larger cap
        torch = _lib.require_cuda()
        sel = torch.from_numpy(over).cuda()
        cap2 = int(hops_h[over].max())
        b2 = _Bound(source, q_dev[sel].contiguous())
        st2 = starts_dev[sel].contiguous() if starts_dev is not None else None
        _, _, _, _, t2i, t2d = _launch(graph, b2, beam_width, st2, cap2)
        tids_h = np.full((nq, cap2), -1, dtype=np.int32)
        tdst_h = np.zeros((nq, cap2), dtype=np.float32)
        tids_h[:, :cap] = tids.cpu().numpy()
        tdst_h[:, :cap] = tdst.cpu().numpy()
        tids_h[over] = t2i.cpu().numpy()
        tdst_h[over] = t2d.cpu().numpy()
    else:
        tids_h, tdst_h = tids.cpu().numpy(), tdst.cpu().numpy()
    keys = fk.cpu().numpy().view(np.uint64)
    evals_h = evals.cpu().numpy().astype(np.int64)
    lossy = np.nonzero(flags.cpu().numpy())[0]
    if lossy.size:  # only after a trace re-run (overflowed cap): the device recount needs whole traces
        # The visited table evicted ids for these queries, so the device counted some
        # re-evaluations. The reference's count is |{start} U N(u) over expanded u|
        # (every valid neighbour of an expanded vertex is evaluated exactly once).
        adj = graph.host_adjacency()
        st = np.full(nq, graph.entry_point, dtype=np.int64) if starts is None else \
            np.broadcast_to(np.asarray(starts, dtype=np.int64), (nq,))
        for i in lossy:
            nb = adj[tids_h[i, : int(hops_h[i])]].ravel()
            evals_h[i] = np.unique(np.append(nb[nb >= 0], st[i])).size
    # key words decode as f32 bits, or as the integer distance of a u8 source (search.py:148-153)
    word = np.uint32 if u8 else np.float32
    tdst_h = tdst_h.view(word)
    out = []
    for i in range(nq):
        kk = keys[i][keys[i] != _UMAX]
        h = int(hops_h[i])
        out.append(SearchResult(
            frontier_ids=(kk & np.uint64(0xFFFFFFFF)).astype(np.int32),
            frontier_dists=(kk >> np.uint64(32)).astype(np.uint32).view(word).astype(np.float64),
            visited_ids=tids_h[i, :h].copy(),
            visited_dists=tdst_h[i, :h].astype(np.float64),
            stats=SearchStats(hops=h, distance_evals=int(evals_h[i])),
        ))
    return out


def beam_search(graph, source, query, params: SearchParams, start: int | None = None) -> SearchResult:
    return run_beam_searches(graph, source, np.atleast_2d(query), params.beam_width, start)[0]


def search_knn(graph, source, query, params: SearchParams, start: int | None = None,
               exact_data=None) -> list[Candidate]:
    """search.py:323-348."""
    if params.rerank and not isinstance(source, VectorDataset) and _is_rabitq(source) and exact_data is None:
        raise ValueError("rerank over a quantized source requires exact_data")
    graph = as_graph(graph)
    _validate(graph, params.beam_width)
    q_dev = _queries_to_device(query, _is_u8(source))
    ids, dists = _knn_device(graph, source, q_dev, params, exact_data, _starts(graph, start, 1))
    ids, dists = ids.cpu().numpy()[0], dists.cpu().numpy()[0]
    keep = ids >= 0
    return [Candidate(int(i), float(d)) for i, d in zip(ids[keep], dists[keep])]


def _knn_device(graph: GraphIndex, source, q_dev, params: SearchParams, exact_data=None, starts_dev=None):
    torch = _lib.require_cuda()
    nq = q_dev.shape[0]
    rerank = params.rerank and _is_rabitq(source)
    if rerank and exact_data is None:
        raise ValueError("rerank over a quantized source requires exact_data")
    _check_counts(graph, source, exact_data, rerank)
    bound = _Bound(source, q_dev, params.estimator)
    L, k = params.beam_width, params.k
    fk, *_ = _launch(graph, bound, L, starts_dev, 0)
    ids = torch.empty((nq, k), dtype=torch.int32, device=q_dev.device)
    dists = torch.empty((nq, k), dtype=torch.float64, device=q_dev.device)
    if nq == 0:
        return ids, dists
    st = _lib.stream_ptr()
    if rerank:
        rows, rdims = _rerank_rows(exact_data)
        if rdims != q_dev.shape[1]:
            raise ValueError(f"query dims {q_dev.shape[1]} != dataset dims {rdims}")
        _lib.check(_lib.lib().jb_rerank_topk(_lib.ptr(rows), rdims, _lib.ptr(q_dev), nq, _lib.ptr(fk), L, k,
                                             _lib.ptr(ids), _lib.ptr(dists), st))
    else:
        fn = _lib.lib().jb_frontier_topk_u8 if bound.kind == _lib.SRC_EXACT_U8 else _lib.lib().jb_frontier_topk
        _lib.check(fn(_lib.ptr(fk), nq, L, k, _lib.ptr(ids), _lib.ptr(dists), st))
    return ids, dists


def search_knn_batch(graph, source, queries, params: SearchParams, exact_data=None):
    """search.py:351-383: (ids int32 [nq,k] padded -1, dists f64 [nq,k] padded +inf).

    Host arrays in and out, through the native host pipeline jb_search_knn_host
    (pinned staging, H2D, bind, search, rerank/top-k, D2H in chunks over two
    streams; csrc/pipeline.cu).
    """
    graph = as_graph(graph)
    _validate(graph, params.beam_width)
    if params.rerank and _is_rabitq(source) and exact_data is None:
        raise ValueError("rerank over a quantized source requires exact_data")
    if _is_u8(source):  # u8 rows: one device search + top-k (the host pipeline stages f32 queries)
        ids, dists = _knn_device(graph, source, _queries_to_device(queries, True), params, exact_data)
        return tuple(_to_host(ids, dists))
    q = np.atleast_2d(np.asarray(queries))
    q = np.ascontiguousarray(q, dtype=np.float32)
    nq = q.shape[0]
    ids, dists = _host_results(nq, params.k)
    plan = _knn_plan(graph, source, q.shape[1], params, exact_data)
    _lib.check(_lib.lib().jb_search_knn_host(_lib.C.byref(plan), _lib.ptr(q), nq, _lib.ptr(ids), _lib.ptr(dists),
                                             _lib.stream_ptr()))
    return ids, dists


def _host_results(nq: int, k: int):
    """int32 ids / f64 dists result arrays in page-locked host memory (numpy views
    of pinned torch tensors, cached by torch's host allocator), so the pipeline's
    device-to-host copies land in them directly instead of via staging."""
    torch = _lib.require_cuda()
    ids = torch.empty((nq, k), dtype=torch.int32, pin_memory=True).numpy()
    dists = torch.empty((nq, k), dtype=torch.float64, pin_memory=True).numpy()
    return ids, dists


# Host-API pipeline chunk (queries per chunk; 0 = library default). Tuning hook.
PIPELINE = {"chunk": int(os.environ.get("JB_HOST_CHUNK", "0")), "device_chunk": int(os.environ.get("JB_DEVICE_CHUNK", "0"))}


def _knn_plan(graph: GraphIndex, source, D: int, params: SearchParams, exact_data=None):
    """jb_knn_plan for jb_search_knn_host: graph + distance source as device pointers."""
    _check_counts(graph, source, exact_data, params.rerank and _is_rabitq(source))
    adj, _ = graph.device()
    plan = _lib.KnnPlan()
    a = plan.search
    a.adjacency = _lib.ptr(adj)
    a.degree_cap = graph.degree_cap
    a.active_count = graph.active_count
    a.start_vertex = graph.entry_point
    a.beam_width = params.beam_width
    a.hash_slots = int(TUNING["hash_slots"])
    a.dims = D
    if _is_rabitq(source):
        from .rabitq import as_rabitq

        idx = as_rabitq(source)
        if D != idx.dims:
            raise ValueError(f"query dims {D} != index dims {idx.dims}")
        dev = idx.device()
        a.source = _lib.SRC_RABITQ
        a.records, a.record_bytes, a.bits = _lib.ptr(dev.records), dev.record_bytes, idx.bits
        if params.estimator == "popcount":
            a.source = _lib.SRC_RABITQ_FAST
            pl, pb = idx.device_planes()
            a.records, a.record_bytes = _lib.ptr(pl), pb
        plan.centroid, plan.rotation = _lib.ptr(dev.centroid), _lib.ptr(dev.rotation)
        if params.rerank:
            rows, rdims = _rerank_rows(exact_data)
            if rdims != D:
                raise ValueError(f"query dims {D} != dataset dims {rdims}")
            plan.rerank_data = _lib.ptr(rows)
    else:
        ds = as_dataset(source)
        if D != ds.dims:
            raise ValueError(f"query dims {D} != dataset dims {ds.dims}")
        rows = ds.device()
        a.source = _lib.SRC_EXACT
        a.data, a.data_norms = _lib.ptr(rows.x), _lib.ptr(rows.norms)
        scr = _screen(ds)
        if scr is not None:
            a.screen, a.screen_center = _lib.ptr(scr[0]), _lib.ptr(scr[1])
    plan.k = params.k
    plan.chunk = int(PIPELINE["chunk"])
    return plan


def search_knn_batch_device(graph, source, q_dev, params: SearchParams, exact_data=None):
    """HBM-resident variant: queries and results stay torch CUDA tensors (no host sync).
    One native call (jb_search_knn_device): the batch is split over two streams so
    the second half's search kernel fills the SMs the first half's tail leaves idle;
    the current stream waits for both."""
    graph = as_graph(graph)
    _validate(graph, params.beam_width)
    if params.rerank and _is_rabitq(source) and exact_data is None:
        raise ValueError("rerank over a quantized source requires exact_data")
    torch = _lib.require_cuda()
    if _is_u8(source):
        return _knn_device(graph, source, _queries_to_device(q_dev, True), params, exact_data)
    q_dev = q_dev.to(dtype=torch.float32).contiguous()
    nq = q_dev.shape[0]
    ids = torch.empty((nq, params.k), dtype=torch.int32, device=q_dev.device)
    dists = torch.empty((nq, params.k), dtype=torch.float64, device=q_dev.device)
    plan = _knn_plan(graph, source, q_dev.shape[1], params, exact_data)
    plan.chunk = int(PIPELINE["device_chunk"])
    _lib.check(_lib.lib().jb_search_knn_device(_lib.C.byref(plan), _lib.ptr(q_dev), nq, _lib.ptr(ids),
                                               _lib.ptr(dists), _lib.stream_ptr()))
    return ids, dists
