"""Batch-parallel construction and streaming insertion on B200 (mirror of build.py).

  BuildParams     build.py:35-62   same fields, defaults and validation
  batch_insert    build.py:296-348 one jb_batch_insert call: phase-1 batched
                  search, phase-2 warp prune + reverse triples, phase-3 sorted
                  group merge with one owner warp per target, then connectivity
                  repair — all on device, mutating the HBM adjacency in place
  build           build.py:389-424 R+1 doubling schedule, entry -> global medoid
  insert_stream   build.py:427-447 max_batch chunks
  _refine_pass    build.py:351-386 two_pass refinement, one jb_refine_batch per batch

Element kinds: f32 rows (einsum-order f32 distances) and u8 rows (exact integer
distances). `quantizer=` (a RaBitQIndex) switches every construction distance to
the RaBitQ estimate against the pivot's bound row (build.py:105-111, 124-129).
"""

from __future__ import annotations

import itertools

import os
import sys
import time
import warnings
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .core import ElementKind, as_dataset
from .graph import GraphIndex, as_graph, medoid, write_back
from .search import MAX_BEAM_WIDTH, MAX_DEGREE_CAP

__all__ = ["BuildParams", "EdgeBuffer", "batch_insert", "build", "insert_stream"]


@dataclass(frozen=True)
class BuildParams:
    degree_cap: int = 64
    build_beam_width: int = 128
    alpha: float = 1.2
    max_batch: int = 100_000
    two_pass: bool = False
    always_prune: bool = False
    reverse_all_visited: bool = False
    # Extension (not in beamann): 0 = the reference's exact connectivity repair;
    # > 0 = donors from a beam search of this width (SURVEY.md §8 B6 approximate mode)
    repair_beam_width: int = 0

    def __post_init__(self):
        if self.degree_cap < 2:
            raise ValueError("degree_cap must be >= 2")
        if self.degree_cap > MAX_DEGREE_CAP:
            raise ValueError(f"degree_cap must be <= {MAX_DEGREE_CAP} (the search kernel's neighbour chunks)")
        if self.alpha < 1.0:
            raise ValueError("alpha must be >= 1")
        if not 1 <= self.build_beam_width <= MAX_BEAM_WIDTH:
            raise ValueError(f"build_beam_width must be in [1, {MAX_BEAM_WIDTH}]")
        if self.max_batch < 1:
            raise ValueError("max_batch must be >= 1")
        if not 0 <= self.repair_beam_width <= MAX_BEAM_WIDTH:
            raise ValueError(f"repair_beam_width must be in [0, {MAX_BEAM_WIDTH}]")
        if self.build_beam_width < self.degree_cap:
            warnings.warn("build_beam_width below degree_cap gives sparse candidate sets", stacklevel=2)


class EdgeBuffer:
    """Host (target, source, dist) triple buffer with the reference's ordering
    (build.py:65-102). The device path keeps its triples in HBM; this class is
    kept for API compatibility."""

    def __init__(self):
        self._t, self._s, self._d = [], [], []

    def add(self, targets, source: int, dists) -> None:
        t = np.asarray(targets, dtype=np.int64).ravel()
        self._t.append(t)
        self._s.append(np.full(t.size, source, dtype=np.int64))
        self._d.append(np.asarray(dists, dtype=np.float64).ravel())

    def __len__(self) -> int:
        return sum(t.size for t in self._t)

    def sorted_triples(self):
        if not self._t:
            e = np.empty(0, dtype=np.int64)
            return e, e.copy(), np.empty(0, dtype=np.float64)
        t, s, d = np.concatenate(self._t), np.concatenate(self._s), np.concatenate(self._d)
        o = np.lexsort((s, d, t))
        return t[o], s[o], d[o]

    def groups(self):
        t, s, d = self.sorted_triples()
        if not t.size:
            return
        uniq, starts = np.unique(t, return_index=True)
        bounds = np.append(starts, t.size)
        for i, v in enumerate(uniq):
            yield int(v), s[bounds[i]:bounds[i + 1]], d[bounds[i]:bounds[i + 1]]


def _validate_range(graph: GraphIndex, dataset, new_ids: range):
    """build.py:227-243 (same messages)."""
    start, stop = new_ids.start, new_ids.stop
    if new_ids.step != 1:
        raise ValueError("new id range must be contiguous")
    if start < stop and start < graph.active_count:
        raise ValueError(f"id range [{start}, {stop}) overlaps active vertices (< {graph.active_count})")
    if start != graph.active_count and start < stop:
        raise ValueError(f"id range must start at active_count={graph.active_count}, got {start}")
    if stop > dataset.count:
        raise ValueError("id range exceeds dataset count")
    if stop > graph.capacity:
        raise ValueError("id range exceeds graph capacity")
    return start, stop


def _bound_rows(quantizer, ds):
    """Quantized construction (build.py:105-111, 124-129): the dataset's rows bound
    as RaBitQ queries (rotated, query_add, query_sumq), the pivot side of every
    construction distance. One jb_rabitq_bind over all rows, cached per dataset."""
    from .rabitq import as_rabitq

    idx = as_rabitq(quantizer)
    if ds.element_kind is not ElementKind.F32:
        raise ValueError("quantized construction requires f32 data")
    if idx.dims != ds.dims:
        raise ValueError(f"quantizer dims {idx.dims} != dataset dims {ds.dims}")
    cache = getattr(idx, "_jb_bound", None)
    if cache is not None and cache[0] is ds:
        return idx, cache[1]
    torch = _lib.require_cuda()
    dev, x = idx.device(), ds.device().x
    n, D = x.shape
    rot = torch.empty((n, D), dtype=torch.float32, device=x.device)
    qa = torch.empty(n, dtype=torch.float32, device=x.device)
    qs = torch.empty(n, dtype=torch.float32, device=x.device)
    if n:
        _lib.check(_lib.lib().jb_rabitq_bind(_lib.ptr(x), n, D, idx.bits, _lib.ptr(dev.centroid), _lib.ptr(dev.rotation),
                                             _lib.ptr(rot), _lib.ptr(qa), _lib.ptr(qs), _lib.stream_ptr()))
    idx._jb_bound = (ds, (rot, qa, qs))
    return idx, (rot, qa, qs)


_TOKENS = itertools.count(1)


def _rows_token(dev) -> int:
    """A never-reused identity of a dataset's device rows (the prune-closure key: a
    device address can be reused by another dataset after the first is freed)."""
    tok = getattr(dev, "_closure_token", None)
    if tok is None:
        tok = next(_TOKENS)
        try:
            dev._closure_token = tok
        except AttributeError:  # immutable holder: no reuse across calls, closure restarts
            pass
    return tok


def _args(graph: GraphIndex, ds, params: BuildParams, start: int, stop: int, quantizer=None):
    adj, deg = graph.device()
    dev = ds.device()
    a = _lib.InsertArgs()
    a.adjacency, a.degrees = _lib.ptr(adj), _lib.ptr(deg)
    a.degree_cap, a.capacity = graph.degree_cap, graph.capacity
    a.dims, a.count = dev.dims, dev.count
    if ds.element_kind is ElementKind.U8:
        a.element_kind, a.data_u8, a.norms_u32 = _lib.KIND_U8, _lib.ptr(dev.x), _lib.ptr(dev.norms)
    else:
        a.element_kind, a.data, a.data_norms = _lib.KIND_F32, _lib.ptr(dev.x), _lib.ptr(dev.norms)
    a.build_beam_width = params.build_beam_width
    a.alpha = float(params.alpha)
    a.always_prune = int(params.always_prune)
    a.reverse_all_visited = int(params.reverse_all_visited)
    a.repair_beam_width = int(params.repair_beam_width)
    a.start, a.stop = start, stop
    a.entry_point = graph.entry_point
    # prune closure (extension): f32 rows only; any other build writes rows without
    # maintaining it, so it is invalidated
    if quantizer is None and ds.element_kind is not ElementKind.U8:
        a.closure = _lib.ptr(graph.device_closure(_rows_token(dev)))
        # int8 screen records for the phase-1 exact search (extension; JB_SCREEN=0: off)
        scr = ds.device_screen() if os.environ.get("JB_SCREEN", "1") != "0" else None
        if scr is not None:
            a.screen, a.screen_center = _lib.ptr(scr[0]), _lib.ptr(scr[1])
    else:
        graph.invalidate_closure()
    if quantizer is not None:
        idx, (rot, qa, qs) = _bound_rows(quantizer, ds)
        if idx.count < max(stop, graph.active_count):
            raise ValueError(f"quantizer covers {idx.count} rows, the batch needs {max(stop, graph.active_count)}")
        rec = idx.device()
        a.quantized, a.records, a.record_bytes, a.bits = 1, _lib.ptr(rec.records), rec.record_bytes, idx.bits
        a.bound_rotated, a.bound_qadd, a.bound_qsumq = _lib.ptr(rot), _lib.ptr(qa), _lib.ptr(qs)
    return a


# Work counters accumulated over batch_insert calls (jb_insert_args.stats_out_host):
# phase-1 hops / distance evals, phase-2 prune candidates, phase-3 touched targets,
# reverse triples, repair bridges, stranded rows through the tensor-core donor
# screen and those rescanned exactly. Read by bench.py for the insert roofline.
WORK_FIELDS = ("search_hops", "search_evals", "prune_candidates", "merge_targets", "reverse_triples", "bridges",
               "donor_tc_rows", "donor_tc_redo")
WORK = np.zeros(8, dtype=np.int64)


def _run(fn, graph: GraphIndex, a) -> int:
    entry = np.zeros(1, dtype=np.int64)
    bridges = np.zeros(1, dtype=np.int64)
    a.entry_point_out_host = entry.ctypes.data
    a.bridges_out_host = bridges.ctypes.data
    a.stats_out_host = WORK.ctypes.data
    try:
        _lib.check(fn(_lib.C.byref(a), _lib.stream_ptr()))
    finally:
        graph.mark_device_modified()
    graph.entry_point = int(entry[0])
    return int(bridges[0])


def _check_supported(params: BuildParams, quantizer):
    if params.degree_cap < 2:
        raise ValueError("degree_cap must be >= 2")


def batch_insert(graph, dataset, new_ids: range, params: BuildParams, quantizer=None) -> None:
    """build.py:296-348: insert a contiguous id range as one three-phase batch (in place)."""
    caller, graph = graph, as_graph(graph)
    ds = as_dataset(dataset)
    start, stop = _validate_range(graph, ds, new_ids)
    if start == stop:
        return
    _check_supported(params, quantizer)
    if graph.degree_cap != params.degree_cap:
        raise ValueError("graph degree_cap differs from params.degree_cap")
    a = _args(graph, ds, params, start, stop, quantizer)
    graph.last_bridges = _run(_lib.lib().jb_batch_insert, graph, a)
    graph.active_count = stop
    write_back(graph, caller)


def _repair(graph: GraphIndex, ds, params: BuildParams, quantizer=None) -> int:
    a = _args(graph, ds, params, 0, graph.active_count, quantizer)
    return _run(_lib.lib().jb_repair_connectivity, graph, a)


def build(dataset, params: BuildParams, quantizer=None) -> GraphIndex:
    """build.py:389-424: bulk build with the R+1 doubling batch schedule."""
    ds = as_dataset(dataset)
    if ds.count == 0:
        raise ValueError("cannot build over an empty dataset")
    _check_supported(params, quantizer)
    pass_params = replace(params, alpha=1.0) if params.two_pass else params
    prof = os.environ.get("JB_PROFILE") == "1"
    t0 = time.perf_counter()
    graph = GraphIndex(capacity=ds.count, degree_cap=params.degree_cap)
    global_medoid = medoid(ds)
    if prof:
        print(f"[jb] medoid {1e3 * (time.perf_counter() - t0):.2f}ms", file=sys.stderr)
    size = params.degree_cap + 1
    pos = 0
    while pos < ds.count:
        stop = min(ds.count, pos + size)
        t1 = time.perf_counter()
        batch_insert(graph, ds, range(pos, stop), pass_params, quantizer)
        if global_medoid < graph.active_count and graph.entry_point != global_medoid:
            graph.entry_point = global_medoid
            _repair(graph, ds, params, quantizer)
        if prof:
            print(f"[jb] batch wall [{pos}, {stop}) {1e3 * (time.perf_counter() - t1):.2f}ms", file=sys.stderr)
        pos = stop
        size = min(size * 2, params.max_batch)
    if params.two_pass:
        _refine_pass(graph, ds, params, quantizer)
    return graph


def _refine_pass(graph, dataset, params: BuildParams, quantizer=None) -> None:
    """build.py:351-386: re-run search + prune for every active vertex at the final
    alpha, in max_batch batches (one native call each), then connectivity repair."""
    graph = as_graph(graph)
    ds = as_dataset(dataset)
    _check_supported(params, quantizer)
    n = graph.active_count
    for lo in range(0, n, params.max_batch):
        hi = min(n, lo + params.max_batch)
        a = _args(graph, ds, params, lo, hi, quantizer)
        a.active_count = n
        _run(_lib.lib().jb_refine_batch, graph, a)
    graph.last_bridges = _repair(graph, ds, params, quantizer)


def insert_stream(graph, dataset, new_range: range, params: BuildParams, quantizer=None) -> None:
    """build.py:427-447."""
    if len(new_range) == 0:
        return
    caller, graph = graph, as_graph(graph)
    ds = as_dataset(dataset)
    _validate_range(graph, ds, new_range)
    pos = new_range.start
    while pos < new_range.stop:
        stop = min(new_range.stop, pos + params.max_batch)
        batch_insert(graph, ds, range(pos, stop), params, quantizer)
        pos = stop
    write_back(graph, caller)
