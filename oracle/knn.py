"""ORACLE — test infrastructure only. Exact kNN and recall.

  * exact_knn: f64 xn - 2 q.x + qn, clamp, stable argsort   oracle.py:20-62
  * exact_knn(inner_product=True): -(q @ x.T), stable sort oracle.py:53-54
  * mips_augment: [x, sqrt(M^2 - |x|^2)], [q, 0]            core.py:169-206
  * recall_at_k: distance-threshold matching, eps 1e-6      bench.py:44-66
"""

from __future__ import annotations

import numpy as np

QBLOCK = 256
EPS = 1e-6


def exact_knn(data: np.ndarray, queries: np.ndarray, k: int, inner_product: bool = False):
    x = data.astype(np.float64)
    qa = queries.astype(np.float64)
    xn = np.einsum("nd,nd->n", x, x)
    ids = np.empty((qa.shape[0], k), dtype=np.int32)
    ds = np.empty((qa.shape[0], k), dtype=np.float32)
    for lo in range(0, qa.shape[0], QBLOCK):
        q = qa[lo:lo + QBLOCK]
        if inner_product:
            s = -(q @ x.T)
        else:
            s = xn[None, :] - 2.0 * (q @ x.T) + np.einsum("bd,bd->b", q, q)[:, None]
            np.maximum(s, 0.0, out=s)
        o = np.argsort(s, axis=1, kind="stable")[:, :k]
        ids[lo:lo + QBLOCK] = o
        ds[lo:lo + QBLOCK] = np.take_along_axis(s, o, axis=1)
    return ids, ds


def mips_augment(data: np.ndarray, queries: np.ndarray):
    """core.py:169-206: returns (aug_data, aug_queries, max_norm)."""
    d64 = data.astype(np.float64)
    nsq = np.einsum("nd,nd->n", d64, d64)
    max_sq = float(nsq.max())
    extra = np.sqrt(np.maximum(max_sq - nsq, 0.0)).astype(np.float32)
    aq = np.hstack([queries, np.zeros((queries.shape[0], 1), dtype=np.float32)])
    return np.hstack([data, extra[:, None]]), aq, float(np.sqrt(max_sq))


def recall_at_k(result_ids, gt_ids: np.ndarray, gt_dists: np.ndarray, k: int) -> float:
    g = gt_dists.astype(np.float64)
    thr = g[:, k - 1] + EPS * np.abs(g[:, k - 1])
    tot = 0.0
    for i in range(len(result_ids)):
        got = np.asarray(result_ids[i], dtype=np.int64)[:k]
        tot += np.isin(got, gt_ids[i][g[i] <= thr[i]]).sum() / k
    return tot / len(result_ids)


def merge_shard_topk(ids_all: np.ndarray, dists_all: np.ndarray, offsets, k: int):
    """Global top-k by (dist, global id) from per-shard lists [S, nq, k] (-1 = padding).
    The checker for the device merge."""
    S, nq, _ = ids_all.shape
    out_i = np.full((nq, k), -1, dtype=np.int64)
    out_d = np.full((nq, k), np.inf)
    for q in range(nq):
        cand = [(float(dists_all[s, q, j]), int(ids_all[s, q, j]) + int(offsets[s]))
                for s in range(S) for j in range(ids_all.shape[2]) if ids_all[s, q, j] >= 0]
        cand.sort()
        for j, (d, g) in enumerate(cand[:k]):
            out_i[q, j], out_d[q, j] = g, d
    return out_i, out_d
