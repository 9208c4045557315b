"""ORACLE — test infrastructure only. Greedy beam search, restated in numpy.

Follows the reference's search engine:
  * keys: (f32 bits of max(d, 0)) << 32 | id            search.py:139-156
  * exact distances (xn - 2 <x,q>) + qn, clamped at 0    search.py:89-130
  * lockstep expansion of the first unvisited slot,
    exact seen set, stable merge truncated to L           search.py:171-269
  * run_beam_searches validation + chunking              search.py:272-304
  * rerank by einsum(x-q, x-q), lexsort((ids, d))         search.py:318-320, 366-383
"""

from __future__ import annotations

import numpy as np

UMAX = np.uint64(0xFFFFFFFFFFFFFFFF)
LOW32 = np.uint64(0xFFFFFFFF)
SEEN_BUDGET = 1 << 28  # search.py:39


def pack(d: np.ndarray, ids: np.ndarray, integer: bool = False) -> np.ndarray:
    """search.py:139-145: f32 bits of max(d, 0), or the raw integer distance (u8)."""
    if integer:
        hi = np.asarray(d).astype(np.uint64)
    else:
        hi = np.maximum(np.asarray(d, dtype=np.float32), np.float32(0)).view(np.uint32).astype(np.uint64)
    return (hi << np.uint64(32)) | np.asarray(ids).astype(np.uint64)


def unpack_dist(keys: np.ndarray, integer: bool = False) -> np.ndarray:
    """search.py:148-152: high word -> f32 -> f64 (or integer -> f64)."""
    hi = keys >> np.uint64(32)
    if integer:
        return hi.astype(np.float64)
    return hi.astype(np.uint32).view(np.float32).astype(np.float64)


def unpack_id(keys: np.ndarray) -> np.ndarray:
    return (keys & LOW32).astype(np.int64)


class ExactSource:
    """search.py:89-130: f32 rows, norms from einsum, distances in the data role;
    u8 rows: the same identity in exact int64 (search.py:92-99), no clamp."""

    def __init__(self, data: np.ndarray, queries: np.ndarray):
        self.integer = np.asarray(data).dtype == np.uint8
        if self.integer:
            if np.asarray(queries).dtype != np.uint8:
                raise ValueError("u8 dataset requires u8 queries")
            self.x = np.asarray(data).astype(np.int64)
            self.q = np.atleast_2d(queries).astype(np.int64)
        else:
            self.x = np.ascontiguousarray(data, dtype=np.float32)
            self.q = np.ascontiguousarray(np.atleast_2d(queries), dtype=np.float32)
        self.xn = np.einsum("nd,nd->n", self.x, self.x)
        self.qn = np.einsum("qd,qd->q", self.q, self.q)

    def __call__(self, qrows: np.ndarray, ids: np.ndarray) -> np.ndarray:
        dots = np.einsum("md,md->m", self.x[ids], self.q[qrows])
        d = self.xn[ids] - 2 * dots + self.qn[qrows]
        return d if self.integer else np.maximum(d, np.float32(0))


class Result:
    __slots__ = ("frontier_ids", "frontier_dists", "visited_ids", "visited_dists", "hops", "evals")

    def __init__(self, fi, fd, vi, vd, hops, evals):
        self.frontier_ids, self.frontier_dists = fi, fd
        self.visited_ids, self.visited_dists = vi, vd
        self.hops, self.evals = hops, evals


def _lockstep(adjacency: np.ndarray, n_active: int, dist, qrows: np.ndarray,
              starts: np.ndarray, width: int) -> list[Result]:
    nq = len(qrows)
    beam = np.full((nq, width), UMAX, dtype=np.uint64)
    done = np.ones((nq, width), dtype=bool)          # "expanded or empty"
    seen = np.zeros((nq, n_active), dtype=bool)
    evals = np.ones(nq, dtype=np.int64)
    hops = np.zeros(nq, dtype=np.int64)
    integer = getattr(dist, "integer", False)
    beam[:, 0] = pack(dist(qrows, starts), starts, integer)
    done[:, 0] = False
    seen[np.arange(nq), starts] = True
    log_q, log_id, log_d = [], [], []

    live = np.arange(nq)
    while live.size:
        pending = ~done[live]
        live = live[pending.any(axis=1)]
        if not live.size:
            break
        slot = (~done[live]).argmax(axis=1)
        ukeys = beam[live, slot]
        done[live, slot] = True
        uid = unpack_id(ukeys)
        hops[live] += 1
        log_q.append(live)
        log_id.append(uid.astype(np.int32))
        log_d.append(unpack_dist(ukeys, integer))

        nbr = adjacency[uid]
        ok = nbr >= 0
        nbr_safe = np.where(ok, nbr, 0)
        fresh = ok & ~seen[live[:, None], nbr_safe]
        cand = np.full(nbr.shape, UMAX, dtype=np.uint64)
        r, c = np.nonzero(fresh)
        if r.size:
            ids = nbr[r, c].astype(np.int64)
            qsel = live[r]
            cand[r, c] = pack(dist(qrows[qsel], ids), ids, integer)
            seen[qsel, ids] = True
            evals[live] += np.bincount(r, minlength=live.size)
        merged = np.concatenate([beam[live], cand], axis=1)
        merged_done = np.concatenate([done[live], ~fresh], axis=1)
        order = np.argsort(merged, axis=1, kind="stable")[:, :width]
        rows = np.arange(live.size)[:, None]
        beam[live] = merged[rows, order]
        done[live] = merged_done[rows, order]

    if log_q:
        q_all = np.concatenate(log_q)
        by_q = np.argsort(q_all, kind="stable")
        id_all = np.concatenate(log_id)[by_q]
        d_all = np.concatenate(log_d)[by_q]
    else:
        id_all = np.empty(0, np.int32)
        d_all = np.empty(0, np.float64)
    ends = np.concatenate([[0], np.cumsum(hops)])
    out = []
    for i in range(nq):
        k = beam[i][beam[i] != UMAX]
        out.append(Result(unpack_id(k).astype(np.int32), unpack_dist(k, integer),
                          id_all[ends[i]:ends[i + 1]], d_all[ends[i]:ends[i + 1]],
                          int(hops[i]), int(evals[i])))
    return out


def beam_search(adjacency: np.ndarray, n_active: int, entry: int, dist, nq: int, width: int,
                starts=None) -> list[Result]:
    """run_beam_searches (search.py:272-304) over a bound distance callable."""
    if n_active == 0:
        raise ValueError("search on an empty graph")
    if not 1 <= width <= 1024:
        raise ValueError("beam_width must be in [1, 1024]")
    st = np.broadcast_to(np.asarray(entry if starts is None else starts, dtype=np.int64), (nq,)).copy()
    if st.size and (st.min() < 0 or st.max() >= n_active):
        raise ValueError("start vertex out of range")
    step = max(1, SEEN_BUDGET // max(n_active, 1))
    res: list[Result] = []
    for lo in range(0, nq, step):
        hi = min(nq, lo + step)
        res.extend(_lockstep(adjacency, n_active, dist, np.arange(lo, hi), st[lo:hi], width))
    return res


def rerank_rows(data: np.ndarray, query: np.ndarray, ids: np.ndarray) -> np.ndarray:
    """search.py:318-320: einsum over the direct difference, f32."""
    diff = data[ids].astype(np.float32) - np.asarray(query, dtype=np.float32)
    return np.einsum("md,md->m", diff, diff)


def topk(results: list[Result], k: int, queries=None, rerank_data=None):
    """search_knn_batch tail (search.py:366-383)."""
    nq = len(results)
    ids_out = np.full((nq, k), -1, dtype=np.int32)
    d_out = np.full((nq, k), np.inf, dtype=np.float64)
    for i, r in enumerate(results):
        ids, ds = r.frontier_ids, r.frontier_dists
        if rerank_data is not None and ids.size:
            ex = rerank_rows(rerank_data, queries[i], ids).astype(np.float64)
            o = np.lexsort((ids, ex))
            ids, ds = ids[o], ex[o]
        t = min(k, ids.size)
        ids_out[i, :t] = ids[:t]
        d_out[i, :t] = ds[:t]
    return ids_out, d_out
