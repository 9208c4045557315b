"""Recall / throughput measurement (mirror of the reference's bench.py).

  recall_at_k   bench.py:44-66   distance-threshold matching, eps = 1e-6 relative
  run_queries   bench.py:69-91   one batched device call (threads are unnecessary)
  sweep         bench.py:94-137  warmup + timed pass per beam width, recall, QPS
  SweepPoint / write_sweep_csv   io.py:39, 172-180 column layout
  exact_knn     oracle.py:20-62  exact f64 top-k (ground truth) on the GPU (jb_exact_knn)
"""

from __future__ import annotations

import csv
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import DistanceKind, VectorDataset, as_dataset
from .search import SearchParams, search_knn_batch

__all__ = ["SweepPoint", "GroundTruth", "exact_knn", "exact_knn_device", "recall_at_k", "run_queries", "sweep",
           "write_sweep_csv"]

_RELATIVE_EPS = 1e-6
SWEEP_CSV_HEADER = ("beam_width", "k", "recall", "qps", "mean_latency_us")


@dataclass(frozen=True)
class GroundTruth:
    ids: np.ndarray        # (nq, k) int32
    distances: np.ndarray  # (nq, k) float32, rows non-decreasing

    @property
    def query_count(self) -> int:
        return self.ids.shape[0]

    @property
    def k(self) -> int:
        return self.ids.shape[1]


def exact_knn_device(x_dev, q_dev, k: int, inner_product: bool = False):
    """Exact top-k on HBM-resident f32 rows/queries: (ids int32 [nq,k], dists f32 [nq,k])
    ranked by (f64 score, id) like oracle.py:44-58, as device tensors."""
    torch = _lib.require_cuda()
    n, D = x_dev.shape
    nq = q_dev.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}]")
    if q_dev.shape[1] != D:
        raise ValueError(f"dimension mismatch: data {D}, queries {q_dev.shape[1]}")
    x_dev = x_dev.to(torch.float32).contiguous()
    q_dev = q_dev.to(torch.float32).contiguous()
    ids = torch.empty((nq, k), dtype=torch.int32, device=x_dev.device)
    ds = torch.empty((nq, k), dtype=torch.float32, device=x_dev.device)
    _lib.check(_lib.lib().jb_exact_knn_kind(_lib.ptr(x_dev), n, D, _lib.ptr(q_dev), nq, k, int(inner_product),
                                            _lib.ptr(ids), _lib.ptr(ds), _lib.stream_ptr()))
    return ids, ds


def exact_knn(data, queries, k: int, distance_kind=DistanceKind.SQUARED_EUCLIDEAN) -> GroundTruth:
    """oracle.py:20-62: exhaustive top-k per query in f64, ties broken by id;
    inner product ranks by -(q . x) (the stored distances are the negated products)."""
    if distance_kind not in (DistanceKind.SQUARED_EUCLIDEAN, DistanceKind.INNER_PRODUCT):
        raise ValueError(f"unsupported distance kind {distance_kind}")
    torch = _lib.require_cuda()
    ds = as_dataset(data) if not isinstance(data, np.ndarray) else VectorDataset(data)
    qs = as_dataset(queries) if not isinstance(queries, np.ndarray) else VectorDataset(queries)
    if not 1 <= k <= ds.count:
        raise ValueError(f"k must be in [1, {ds.count}]")
    if ds.dims != qs.dims:
        raise ValueError(f"dimension mismatch: data {ds.dims}, queries {qs.dims}")
    if ds.element_kind is not qs.element_kind:
        raise ValueError("data and queries must share an element kind")
    # u8 rows are scored on exact f32 copies (the reference scores x.astype(f64))
    q_dev = torch.from_numpy(np.ascontiguousarray(qs.data, dtype=np.float32)).cuda()
    ids, dists = exact_knn_device(ds.device_f32(), q_dev, k, distance_kind is DistanceKind.INNER_PRODUCT)
    return GroundTruth(ids=ids.cpu().numpy(), distances=dists.cpu().numpy())


@dataclass(frozen=True)
class SweepPoint:
    beam_width: int
    k: int
    recall: float
    qps: float
    mean_latency_us: float


def recall_at_k(result_ids, gt, k: int) -> float:
    """Mean fraction of the exact top-k recovered; ties at the k-th distance count."""
    if not 1 <= k <= gt.k:
        raise ValueError(f"k must be in [1, {gt.k}]")
    res = np.asarray(result_ids)
    if res.shape[0] != gt.query_count:
        raise ValueError(f"result rows {res.shape[0]} != ground-truth queries {gt.query_count}")
    if res.ndim != 2 or res.shape[1] < k:
        raise ValueError(f"need at least {k} ids per query")
    gd = gt.distances.astype(np.float64)
    thr = gd[:, k - 1] + _RELATIVE_EPS * np.abs(gd[:, k - 1])
    ok = gd <= thr[:, None]
    got = res[:, :k].astype(np.int64)
    hit = np.zeros(got.shape, dtype=bool)
    for j in range(gt.k):  # membership in the within-threshold GT set
        hit |= (got == gt.ids[:, j:j + 1].astype(np.int64)) & ok[:, j:j + 1]
    return float(hit.sum(axis=1).mean() / k)


def run_queries(graph, source, queries, params: SearchParams, exact_data=None, workers: int = 1):
    """bench.py:69-91: top-k for a query batch, optionally split across worker
    threads exactly as the reference splits it. Each thread's search_knn_batch
    runs on its own native context (streams, pinned staging), so the calls are
    re-entrant; one batch (workers=1) is the fastest use of the GPU."""
    queries = np.atleast_2d(np.asarray(queries))
    if workers <= 1 or queries.shape[0] < 2 * workers:
        return search_knn_batch(graph, source, queries, params, exact_data)
    from concurrent.futures import ThreadPoolExecutor

    chunks = np.array_split(np.arange(queries.shape[0]), workers)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        futures = [pool.submit(search_knn_batch, graph, source, queries[c], params, exact_data)
                   for c in chunks if c.size]
        parts = [f.result() for f in futures]
    return np.concatenate([p_[0] for p_ in parts], axis=0), np.concatenate([p_[1] for p_ in parts], axis=0)


# the reference's CSV plus the GPU run's context columns,
# written only when asked for (the default file stays byte-compatible with io.py:172-180)
SWEEP_CSV_EXTRA = ("gpus", "inserts_per_s", "alg_bytes_per_query", "hbm_frac", "cpu_qps", "cpu_cores")


def write_sweep_csv(path, points, extra: dict | None = None) -> None:
    """io.py:172-180 (same header and number formats: qps and latency %.2f). `extra` (optional) maps any of
    SWEEP_CSV_EXTRA to one value per point (a scalar applies to every point); those
    columns are appended after the reference's five."""
    cols = []
    if extra:
        unknown = set(extra) - set(SWEEP_CSV_EXTRA)
        if unknown:
            raise ValueError(f"unknown sweep CSV columns {sorted(unknown)}; allowed {SWEEP_CSV_EXTRA}")
        cols = [c for c in SWEEP_CSV_EXTRA if c in extra]

    def cell(c, i):
        v = extra[c]
        v = v[i] if isinstance(v, (list, tuple, np.ndarray)) else v
        return "" if v is None else (f"{v:.6g}" if isinstance(v, float) else str(v))

    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(SWEEP_CSV_HEADER + tuple(cols))
        for i, p in enumerate(points):
            w.writerow([p.beam_width, p.k, f"{p.recall:.6f}", f"{p.qps:.2f}", f"{p.mean_latency_us:.2f}"] +
                       [cell(c, i) for c in cols])


def sweep(graph, source, queries, gt, k: int, beam_widths, *, rerank: bool = False, exact_data=None,
          workers: int = 1, warmup: bool = True, csv_path=None, csv_extra: dict | None = None) -> list[SweepPoint]:
    """bench.py:94-137: per beam width one untimed warmup pass, then a timed pass
    (host queries in, host ids out) for QPS, and recall against `gt`."""
    if k > gt.k:
        raise ValueError(f"k={k} exceeds ground-truth depth {gt.k}")
    queries = np.atleast_2d(np.asarray(queries))
    nq = queries.shape[0]
    pts = []
    for beam in beam_widths:
        params = SearchParams(beam_width=int(beam), k=k, rerank=rerank)
        if warmup:
            run_queries(graph, source, queries, params, exact_data, workers)
        t0 = time.perf_counter()
        ids, _ = run_queries(graph, source, queries, params, exact_data, workers)
        el = time.perf_counter() - t0
        pts.append(SweepPoint(int(beam), k, recall_at_k(ids, gt, k), nq / el, el / nq * 1e6))
    if csv_path is not None:
        write_sweep_csv(csv_path, pts, csv_extra)
    return pts
