"""Graph store with an HBM mirror, medoid and robust prune (mirror of graph.py).

`GraphIndex` keeps the reference's public contract (graph.py:36-156): a
fixed-stride int32 adjacency slab `(capacity, R)` padded with -1, `degrees`,
`entry_point`, `active_count`, invariant-checked `set_neighbors`, `validate`,
and the byte-identical `graph.bin` save/load.

B200 layout: the same slab lives in HBM (R=32: one 128 B row per vertex, one
sector-aligned request per hop). Kernels mutate the device slab during
construction; the host arrays are refreshed lazily, so `build`/`insert_stream`
never pay a full-slab download per batch. Reading `adjacency`/`degrees` from
the host marks the host copy as possibly modified, so the next device use
re-uploads it.
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


class GraphIndex:
    def __init__(self, capacity: int, degree_cap: int):
        if capacity < 1:
            raise ValueError("capacity must be >= 1")
        if degree_cap < 1:
            raise ValueError("degree_cap must be >= 1")
        self.capacity = int(capacity)
        self.degree_cap = int(degree_cap)
        self._adj = np.full((capacity, degree_cap), _NO_NEIGHBOR, dtype=np.int32)
        self._deg = np.zeros(capacity, dtype=np.int32)
        self.entry_point = 0
        self.active_count = 0
        self._dev_adj = None
        self._dev_deg = None
        self._host_dirty = True    # host may differ from device -> upload before device use
        self._dev_dirty = False    # device newer -> download before host use
        self._lock = threading.RLock()

    # ---- host view -------------------------------------------------------
    def _sync_host(self) -> None:
        if self._dev_dirty:
            with self._lock:
                if self._dev_dirty:
                    self._adj[:] = self._dev_adj.cpu().numpy()
                    self._deg[:] = self._dev_deg.cpu().numpy()
                    self._dev_dirty = False

    @property
    def adjacency(self) -> np.ndarray:
        self._sync_host()
        self._host_dirty = True
        return self._adj

    @adjacency.setter
    def adjacency(self, value) -> None:
        self._sync_host()
        self._adj = np.asarray(value, dtype=np.int32)
        self._host_dirty = True

    @property
    def degrees(self) -> np.ndarray:
        self._sync_host()
        self._host_dirty = True
        return self._deg

    @degrees.setter
    def degrees(self, value) -> None:
        self._sync_host()
        self._deg = np.asarray(value, dtype=np.int32)
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
            if self._dev_adj is None:
                self._dev_adj = torch.from_numpy(self._adj).to("cuda")
                self._dev_deg = torch.from_numpy(self._deg).to("cuda")
                self._host_dirty = False
            elif self._host_dirty:
                self._dev_adj.copy_(torch.from_numpy(self._adj))
                self._dev_deg.copy_(torch.from_numpy(self._deg))
                self._host_dirty = False
        return self._dev_adj, self._dev_deg

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
    """graph.py:174-228 on device (one warp per pivot).

    The reference takes an arbitrary `dist_fn`; the device path computes the
    same pairwise distances itself (build.py:105-134 semantics), so it needs
    the dataset: pass `dataset=` or a `dist_fn` that exposes `.dataset`.
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
    if dataset is None:
        dataset = getattr(dist_fn, "dataset", None)
    if dataset is None:
        raise ValueError("device robust_prune needs the dataset (dataset= or dist_fn.dataset)")
    from .core import as_dataset

    dev = as_dataset(dataset).device()
    torch = _lib.require_cuda()
    d32 = dists.astype(np.float32)
    if not np.array_equal(d32.astype(np.float64), dists):
        raise ValueError("candidate distances must be f32-representable (they come from f32 kernels)")
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
