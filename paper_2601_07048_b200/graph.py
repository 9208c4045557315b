"""Graph store with an HBM mirror, medoid and robust prune (mirror of graph.py).

`GraphIndex` keeps the reference's public contract (graph.py:36-156): a
fixed-stride int32 adjacency slab `(capacity, R)` padded with -1, `degrees`,
`entry_point`, `active_count`, invariant-checked `set_neighbors`, `validate`,
and the byte-identical `graph.bin` save/load.

B200 layout: the same slab lives in HBM (R=32: one 128 B row per vertex, one
sector-aligned request per hop). Kernels mutate the device slab during
construction; the host arrays are refreshed lazily, so `build`/`insert_stream`
never pay a full-slab download per batch. `adjacency` / `degrees` are numpy
views that track writes: reading them costs at most one download and never a
re-upload; an in-place write through indexing (`g.adjacency[u, :] = ...`,
including through slices of it) marks the host copy modified, so the next
device use uploads it. Writes that bypass `__setitem__` (np.copyto, ufunc
`out=`, or a plain `np.asarray` view) must be followed by
`mark_host_modified()`.
"""

from __future__ import annotations

import threading
from pathlib import Path
from typing import Callable, NamedTuple

import numpy as np

from . import _lib

__all__ = ["Candidate", "GraphIndex", "medoid", "robust_prune"]

_GRAPH_MAGIC = 0x56414D47  # graph.py:21
_GRAPH_VERSION = 1
_NO_NEIGHBOR = -1


class FormatError(ValueError):
    """A file does not conform to the expected binary layout (io.py:42)."""


class Candidate(NamedTuple):
    id: int
    dist: float


class _TrackedArray(np.ndarray):
    """ndarray view whose item assignment marks its GraphIndex's host copy modified.
    Views (slices) inherit the owner; arrays computed from it (ufunc results) do not."""

    def __array_finalize__(self, obj):
        owner = getattr(obj, "_jb_owner", None)
        self._jb_owner = owner if (owner is not None and self.base is not None) else None

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        owner = self._jb_owner
        if owner is not None:
            owner._host_dirty = True

    def __array_wrap__(self, arr, context=None, return_scalar=False):
        # ufunc / reduction results are new arrays, not views of the slab: plain ndarray / scalar
        arr = arr.view(np.ndarray)
        return arr[()] if return_scalar else arr


def _tracked(arr: np.ndarray, owner) -> np.ndarray:
    v = arr.view(_TrackedArray)
    v._jb_owner = owner
    return v


class GraphIndex:
    def __init__(self, capacity: int, degree_cap: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if degree_cap < 1:
            raise ValueError("degree_cap must be >= 1")
        self.capacity = int(capacity)
        self.degree_cap = int(degree_cap)
        # host slab, materialised on first host use: a graph built on the device never
        # pays for page-faulting (and uploading) an all-empty capacity x R host array
        self._adj_store = None
        self._deg_store = None
        self.entry_point = 0
        self.active_count = 0
        self._dev_adj = None
        self._dev_deg = None
        self._host_dirty = True    # host may differ from device -> upload before device use
        self._dev_dirty = False    # device newer -> download before host use
        self._lock = threading.RLock()
        self.h2d_bytes = 0         # slab bytes uploaded so far (instrumentation)
        self.d2h_bytes = 0         # slab bytes downloaded so far
        self._dev_closure = None   # per-vertex prune closure (jb_insert_args.closure), device f64
        self._closure_key = None   # the f32 dataset the closure flags were computed against

    @property
    def _adj(self) -> np.ndarray:
        if self._adj_store is None:
            self._adj_store = np.full((self.capacity, self.degree_cap), _NO_NEIGHBOR, dtype=np.int32)
        return self._adj_store

    @_adj.setter
    def _adj(self, value: np.ndarray) -> None:
        self._adj_store = value

    @property
    def _deg(self) -> np.ndarray:
        if self._deg_store is None:
            self._deg_store = np.zeros(self.capacity, dtype=np.int32)
        return self._deg_store

    @_deg.setter
    def _deg(self, value: np.ndarray) -> None:
        self._deg_store = value

    # ---- host view -------------------------------------------------------
    def _sync_host(self) -> None:
        if self._dev_dirty:
            with self._lock:
                if self._dev_dirty:
                    if self._adj_store is None:  # first host use: the download is the slab
                        self._adj_store = self._dev_adj.cpu().numpy()
                        self._deg_store = self._dev_deg.cpu().numpy()
                    else:
                        self._adj[:] = self._dev_adj.cpu().numpy()
                        self._deg[:] = self._dev_deg.cpu().numpy()
                    self.d2h_bytes += self._adj.nbytes + self._deg.nbytes
                    self._dev_dirty = False

    @property
    def adjacency(self) -> np.ndarray:
        """The (capacity, R) slab; writes through indexing are tracked (module doc)."""
        self._sync_host()
        return _tracked(self._adj, self)

    @adjacency.setter
    def adjacency(self, value) -> None:
        self._sync_host()
        value = np.ascontiguousarray(value, dtype=np.int32)
        if value.shape != (self.capacity, self.degree_cap):
            raise ValueError(f"adjacency must have shape {(self.capacity, self.degree_cap)}")
        self._adj = value.view(np.ndarray).copy() if isinstance(value, _TrackedArray) else value
        self._host_dirty = True

    @property
    def degrees(self) -> np.ndarray:
        self._sync_host()
        return _tracked(self._deg, self)

    @degrees.setter
    def degrees(self, value) -> None:
        self._sync_host()
        value = np.ascontiguousarray(value, dtype=np.int32)
        if value.shape != (self.capacity,):
            raise ValueError(f"degrees must have shape {(self.capacity,)}")
        self._deg = value.view(np.ndarray).copy() if isinstance(value, _TrackedArray) else value
        self._host_dirty = True

    def host_adjacency(self) -> np.ndarray:
        """Up-to-date host slab for read-only internal use (untracked)."""
        self._sync_host()
        return self._adj

    def mark_host_modified(self) -> None:
        """Declare host-side writes that bypassed the tracked views."""
        self._sync_host()
        self._host_dirty = True

    def degree(self, u: int) -> int:
        self._sync_host()
        return int(self._deg[u])

    def neighbors(self, u: int) -> np.ndarray:
        self._sync_host()
        return self._adj[u, : self._deg[u]].copy()

    def set_neighbors(self, u: int, ids) -> None:
        """graph.py:60-75: replace u's adjacency (<= degree_cap, distinct, no self-loop)."""
        ids = np.asarray(ids, dtype=np.int32).ravel()
        if ids.size > self.degree_cap:
            raise ValueError(f"neighbor list of length {ids.size} exceeds degree cap {self.degree_cap}")
        if ids.size:
            if ids.min() < 0 or ids.max() >= self.active_count:
                raise ValueError("neighbor id out of range")
            if (ids == u).any():
                raise ValueError(f"self-loop on vertex {u}")
            if np.unique(ids).size != ids.size:
                raise ValueError(f"duplicate neighbor ids for vertex {u}")
        self._sync_host()
        row = self._adj[u]
        row[: ids.size] = ids
        row[ids.size:] = _NO_NEIGHBOR
        self._deg[u] = ids.size
        self._host_dirty = True

    def validate(self) -> None:
        """graph.py:77-96: full invariant scan (vectorized)."""
        n = self.active_count
        if n == 0:
            return
        if not (0 <= self.entry_point < n):
            raise AssertionError("entry point out of range")
        self._sync_host()
        degs = self._deg[:n]
        if (degs < 0).any() or (degs > self.degree_cap).any():
            raise AssertionError("degree outside [0, degree_cap]")
        rows = self._adj[:n]
        live = np.arange(self.degree_cap)[None, :] < degs[:, None]
        vals = np.where(live, rows, 0)
        bad = live & ((vals < 0) | (vals >= n))
        if bad.any():
            raise AssertionError(f"vertex {int(np.nonzero(bad.any(axis=1))[0][0])}: neighbor id out of range")
        selfl = live & (vals == np.arange(n)[:, None])
        if selfl.any():
            raise AssertionError(f"vertex {int(np.nonzero(selfl.any(axis=1))[0][0])}: self-loop")
        srt = np.sort(np.where(live, rows, -1 - np.arange(self.degree_cap)[None, :]), axis=1)
        dup = (srt[:, 1:] == srt[:, :-1]) & (srt[:, 1:] >= 0)
        if dup.any():
            raise AssertionError(f"vertex {int(np.nonzero(dup.any(axis=1))[0][0])}: duplicate neighbors")

    # ---- device mirror ---------------------------------------------------
    def device(self):
        """(adjacency [capacity, R] int32, degrees [capacity] int32) in HBM, up to date."""
        torch = _lib.require_cuda()
        with self._lock:
            if self._dev_adj is None and self._adj_store is None and self._deg_store is None:
                # never touched on the host: the empty slab is created in HBM
                self._dev_adj = torch.full((self.capacity, self.degree_cap), _NO_NEIGHBOR, dtype=torch.int32,
                                           device="cuda")
                self._dev_deg = torch.zeros(self.capacity, dtype=torch.int32, device="cuda")
                self._host_dirty = False
            elif self._dev_adj is None:
                self._dev_adj = torch.from_numpy(self._adj).to("cuda")
                self._dev_deg = torch.from_numpy(self._deg).to("cuda")
                self.h2d_bytes += self._adj.nbytes + self._deg.nbytes
                self._host_dirty = False
            elif self._host_dirty:
                self._dev_adj.copy_(torch.from_numpy(self._adj))
                self._dev_deg.copy_(torch.from_numpy(self._deg))
                self.h2d_bytes += self._adj.nbytes + self._deg.nbytes
                self._host_dirty = False
                self.invalidate_closure()  # rows written on the host: no row is known to be closed
        return self._dev_adj, self._dev_deg

    def device_closure(self, key):
        """Per-vertex prune closure (jb_insert_args.closure) for f32 builds against the
        dataset identified by `key`; zeroed when the dataset changes or rows are
        written outside the library's prune kernels."""
        torch = _lib.require_cuda()
        with self._lock:
            if self._dev_closure is None:
                self._dev_closure = torch.zeros(self.capacity, dtype=torch.float64, device="cuda")
            elif self._closure_key != key:
                self._dev_closure.zero_()
            self._closure_key = key
        return self._dev_closure

    def invalidate_closure(self) -> None:
        if self._dev_closure is not None:
            self._dev_closure.zero_()

    def mark_device_modified(self) -> None:
        """Called after kernels wrote the device slab."""
        self._dev_dirty = True
        self._host_dirty = False

    # ---- persistence (graph.py:101-156), byte-identical -------------------
    def save(self, path) -> None:
        path = Path(path)
        self._sync_host()
        header = np.array([_GRAPH_MAGIC, _GRAPH_VERSION, self.degree_cap, 0], dtype="<u4")
        tail = np.array([self.active_count, self.entry_point], dtype="<u8")
        n = self.active_count
        slab = self._adj[:n].astype("<i4", copy=True)
        cols = np.arange(self.degree_cap)[None, :]
        slab[cols >= self._deg[:n, None]] = _NO_NEIGHBOR
        with open(path, "wb") as fh:
            fh.write(header.tobytes())
            fh.write(tail.tobytes())
            fh.write(self._deg[:n].astype("<i4", copy=False).tobytes())
            fh.write(np.ascontiguousarray(slab).tobytes())

    @classmethod
    def load(cls, path, capacity: int | None = None) -> "GraphIndex":
        path = Path(path)
        try:
            raw = path.read_bytes()
        except FileNotFoundError:
            raise FormatError(f"{path}: file not found") from None
        if len(raw) < 32:
            raise FormatError(f"{path}: too short for a graph header")
        magic, version, degree_cap, _ = (int(v) for v in np.frombuffer(raw, "<u4", count=4))
        if magic != _GRAPH_MAGIC:
            raise FormatError(f"{path}: bad magic {magic:#x}")
        if version != _GRAPH_VERSION:
            raise FormatError(f"{path}: unsupported version {version}")
        active_count, entry_point = (int(v) for v in np.frombuffer(raw, "<u8", count=2, offset=16))
        expected = 32 + active_count * 4 + active_count * degree_cap * 4
        if len(raw) != expected:
            raise FormatError(f"{path}: expected {expected} bytes, got {len(raw)}")
        if capacity is None:
            capacity = max(active_count, 1)
        if capacity < active_count:
            raise ValueError("capacity smaller than stored active_count")
        g = cls(capacity, degree_cap)
        g._deg[:active_count] = np.frombuffer(raw, "<i4", count=active_count, offset=32)
        g._adj[:active_count] = np.frombuffer(
            raw, "<i4", count=active_count * degree_cap, offset=32 + active_count * 4
        ).reshape(active_count, degree_cap)
        g.active_count = active_count
        g.entry_point = entry_point
        g.validate()
        return g


def as_graph(obj) -> GraphIndex:
    """Accept this package's GraphIndex, or adopt a reference beamann.GraphIndex (drop-in)."""
    if isinstance(obj, GraphIndex):
        return obj
    if all(hasattr(obj, a) for a in ("adjacency", "degrees", "entry_point", "active_count", "degree_cap")):
        g = GraphIndex(obj.adjacency.shape[0], obj.degree_cap)
        g._adj = obj.adjacency
        g._deg = obj.degrees
        g.entry_point = obj.entry_point
        g.active_count = obj.active_count
        return g
    raise TypeError(f"unsupported graph {type(obj).__name__}")


def write_back(graph: GraphIndex, obj) -> None:
    """After a mutating call on a graph adopted from a beamann GraphIndex (as_graph),
    bring the caller's object up to date: the adopted host arrays are the caller's own
    arrays, so syncing the host copy writes them in place; counters are copied."""
    if obj is None or obj is graph:
        return
    graph._sync_host()
    obj.active_count = graph.active_count
    obj.entry_point = graph.entry_point


def medoid(dataset) -> int:
    """graph.py:159-171 on device: f64 mean (sequential), f64 2-lane distances, lowest id."""
    from .core import as_dataset

    ds = as_dataset(dataset)
    if ds.count == 0:
        raise ValueError("medoid of an empty dataset")
    dev = ds.device()
    out = np.zeros(1, dtype=np.int64)
    fn = _lib.lib().jb_medoid_u8 if dev.kind.value == "u8" else _lib.lib().jb_medoid
    _lib.check(fn(_lib.ptr(dev.x), dev.count, dev.dims, out.ctypes.data, _lib.stream_ptr()))
    return int(out[0])


def robust_prune(p: int, candidate_ids, candidate_dists, *, alpha: float, degree_cap: int,
                 dist_fn: Callable | None = None, dataset=None) -> tuple[np.ndarray, np.ndarray]:
    """graph.py:174-228 on device.

    Distance sources, in order:
      * `dataset=` (or a `dist_fn` exposing `.dataset`) of f32 rows: one warp computes
        the pairwise distances itself (build.py:120-134 rounding; jb_robust_prune);
      * u8 rows, a reference-style `_PairwiseDistances` (beamann's: `_x` rows and an
        optional `_quantizer`), or a `dist_fn` exposing `.quantizer`: the candidates'
        pairwise matrix is evaluated by the bound-source kernel (jb_bound_distances:
        pivot bound as the query, build.py:105-134) and pruned by jb_robust_prune_matrix;
      * any other callable `dist_fn(pivot, ids)`: called once per candidate for its
        matrix row (the user's own code, as in the reference), pruned on device.
    Returns kept (int32 ids, f64 dists) in extraction order.
    """
    if alpha < 1.0:
        raise ValueError("alpha must be >= 1")
    if degree_cap < 1:
        raise ValueError("degree_cap must be >= 1")
    ids = np.asarray(candidate_ids, dtype=np.int64).ravel()
    dists = np.asarray(candidate_dists, dtype=np.float64).ravel()
    if ids.shape != dists.shape:
        raise ValueError("candidate ids and dists length mismatch")
    if (ids == p).any():
        raise ValueError("candidate set must not contain the pivot")
    if np.unique(ids).size != ids.size:
        raise ValueError("candidate set must be deduplicated")
    if ids.size == 0:
        return ids.astype(np.int32), dists
    source, quantizer = _prune_source(dist_fn, dataset)
    from .core import ElementKind, as_dataset

    if source is not None and quantizer is None and as_dataset(source).element_kind is ElementKind.F32:
        d32 = dists.astype(np.float32)
        if np.array_equal(d32.astype(np.float64), dists):
            return _prune_f32_rows(as_dataset(source), p, ids, d32, alpha, degree_cap)
    if source is not None:
        dmat = _pair_matrix_device(as_dataset(source), quantizer, ids)
    else:
        if dist_fn is None:
            raise ValueError("robust_prune needs dist_fn or dataset")
        dmat = np.stack([np.asarray(dist_fn(int(c), ids), dtype=np.float64).reshape(ids.size) for c in ids])
    return _prune_matrix(dmat, ids, dists, alpha, degree_cap)


def _prune_source(dist_fn, dataset):
    """(dataset-like rows, quantizer or None) behind a dist_fn, or (None, None) for an opaque callable."""
    if dataset is not None:
        return dataset, getattr(dist_fn, "quantizer", None) if dist_fn is not None else None
    if dist_fn is None:
        return None, None
    ds = getattr(dist_fn, "dataset", None)
    if ds is not None:
        return ds, getattr(dist_fn, "quantizer", None)
    x = getattr(dist_fn, "_x", None)  # beamann build._PairwiseDistances (build.py:105-134)
    if isinstance(x, np.ndarray) and x.ndim == 2:
        q = getattr(dist_fn, "_quantizer", None)
        ds = getattr(dist_fn, "_jb_dataset", None)  # HBM copy cached on the caller's object
        if ds is None:
            from .core import VectorDataset

            ds = VectorDataset(x.astype(np.uint8) if x.dtype == np.int64 else x)  # u8 rows widened by the reference
            try:
                setattr(dist_fn, "_jb_dataset", ds)
            except AttributeError:
                pass
        return ds, q
    return None, None


def _prune_f32_rows(ds, p, ids, d32, alpha, degree_cap):
    torch = _lib.require_cuda()
    dev = ds.device()
    if ids.max() >= dev.count or p >= dev.count or p < 0 or ids.min() < 0:
        raise IndexError("vertex id out of range")
    t_ids = torch.from_numpy(ids.astype(np.int32)).cuda()
    t_d = torch.from_numpy(d32).cuda()
    piv = torch.tensor([p], dtype=torch.int64, device="cuda")
    offs = torch.tensor([0, ids.size], dtype=torch.int64, device="cuda")
    out_i = torch.empty(degree_cap, dtype=torch.int32, device="cuda")
    out_d = torch.empty(degree_cap, dtype=torch.float32, device="cuda")
    out_n = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().jb_robust_prune(_lib.ptr(dev.x), _lib.ptr(dev.norms), dev.dims, _lib.ptr(piv), 1,
                                          _lib.ptr(offs), _lib.ptr(t_ids), _lib.ptr(t_d), float(alpha),
                                          degree_cap, _lib.ptr(out_i), _lib.ptr(out_d), _lib.ptr(out_n),
                                          _lib.stream_ptr()))
    n = int(out_n.item())
    return out_i[:n].cpu().numpy(), out_d[:n].cpu().numpy().astype(np.float64)


def _pair_matrix_device(ds, quantizer, ids):
    """dmat[i, j] = d(ids[i] as pivot, ids[j]) on device: the candidate rows bound as queries
    (build.py:120-134 exact rows / u8; build.py:124-129 quantized: bind(x[pivot]))."""
    from .search import BoundDistances

    torch = _lib.require_cuda()
    if ids.max() >= ds.count or ids.min() < 0:
        raise IndexError("vertex id out of range")
    n = ids.size
    rows = torch.from_numpy(np.ascontiguousarray(ds.data[ids]))
    if quantizer is not None:
        from .rabitq import as_rabitq

        bound = as_rabitq(quantizer).bind(rows.numpy())
    else:
        bound = BoundDistances(ds, rows.numpy())
    t_ids = torch.from_numpy(ids).cuda()
    qr = torch.arange(n, device="cuda").repeat_interleave(n)
    cols = t_ids.repeat(n)
    return bound.distances_device(qr, cols).reshape(n, n).to(torch.float64)


def _prune_matrix(dmat, ids, dists, alpha, degree_cap):
    torch = _lib.require_cuda()
    n = ids.size
    dm = (dmat if isinstance(dmat, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(dmat))).to(
        "cuda", torch.float64).contiguous()
    t_ids = torch.from_numpy(ids).cuda()
    t_d = torch.from_numpy(np.ascontiguousarray(dists)).cuda()
    pos = torch.empty(degree_cap, dtype=torch.int32, device="cuda")
    cnt = torch.empty(1, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().jb_robust_prune_matrix(_lib.ptr(dm), _lib.ptr(t_ids), _lib.ptr(t_d), n, float(alpha),
                                                 degree_cap, _lib.ptr(pos), _lib.ptr(cnt), _lib.stream_ptr()))
    k = int(cnt.item())
    sel = pos[:k].long().cpu().numpy()
    return ids[sel].astype(np.int32), dists[sel].astype(np.float64)
