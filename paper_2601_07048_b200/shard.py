"""Sharded index across the GPUs of one box (north-star 4).

Partition: each rank owns one shard — its own graph, exact rows and optional
RaBitQ codes — and a fixed global-id base `shard_start` (contiguous ranges
[s*N/G, (s+1)*N/G) for a bulk-built index, `rank * shard_capacity` for one that
grows by streaming inserts). Inserts are routed to the owning shard and run
`batch_insert` locally (reference build.py:296-348, 427-447): no cross-GPU
exchange on the insert path. Per query batch:

  1. the root rank's queries are broadcast (NCCL, NVLink),
  2. every rank runs the single-GPU kernels on its shard,
  3. each shard's top-k is packed into 16-byte {f64 dist, i64 global id}
     records (jb_pack_shard_topk) and ONE all-gather moves them, and
  4. every rank merges on device by (dist, global id) (jb_merge_shard_records).

No step synchronizes the host when the batch shape is known to every rank
(`nq=`); the shard offsets are gathered once when the index is created. One
process per GPU; `torch.distributed` (backend "nccl") is the plumbing. The
protocol functions take injectable `local_search` / `merge` callables so the
same code path runs in world-size-2 gloo tests on CPU.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["shard_range", "sharded_knn", "merge_topk_device", "ShardedIndex", "RECORD_WORDS"]

RECORD_WORDS = 2  # one exchange record = {f64 dist, i64 global id} = 2 x int64


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous shard [start, stop) of `n_total` global ids for `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n_total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def merge_topk_device(ids_all, dists_all, offsets, k: int):
    """[S, nq, k] local (int32, f64) lists -> global top-k (int64 ids, f64 dists) on device."""
    torch = _lib.require_cuda()
    S, nq, kk = ids_all.shape
    out_i = torch.empty((nq, k), dtype=torch.int64, device=ids_all.device)
    out_d = torch.empty((nq, k), dtype=torch.float64, device=ids_all.device)
    offs = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    _lib.check(_lib.lib().jb_merge_shard_topk(_lib.ptr(ids_all.contiguous()), _lib.ptr(dists_all.contiguous()), S, nq,
                                              k, offs.ctypes.data, _lib.ptr(out_i), _lib.ptr(out_d),
                                              _lib.stream_ptr()))
    return out_i, out_d


def pack_topk_device(ids, dists, offset: int):
    """(int32 local ids, f64 dists) [nq, k] -> int64 [nq, 2k] exchange records (device)."""
    torch = _lib.require_cuda()
    nq, k = ids.shape
    out = torch.empty((nq, RECORD_WORDS * k), dtype=torch.int64, device=ids.device)
    _lib.check(_lib.lib().jb_pack_shard_topk(_lib.ptr(ids.contiguous()), _lib.ptr(dists.contiguous()), nq, k,
                                             int(offset), _lib.ptr(out), _lib.stream_ptr()))
    return out


def merge_records_device(records, k: int):
    """All-gathered records [S, nq, 2k] -> global top-k (int64 ids, f64 dists) (device)."""
    torch = _lib.require_cuda()
    S, nq, _ = records.shape
    out_i = torch.empty((nq, k), dtype=torch.int64, device=records.device)
    out_d = torch.empty((nq, k), dtype=torch.float64, device=records.device)
    _lib.check(_lib.lib().jb_merge_shard_records(_lib.ptr(records.contiguous()), S, nq, k, _lib.ptr(out_i),
                                                 _lib.ptr(out_d), _lib.stream_ptr()))
    return out_i, out_d


def pack_topk_host(ids, dists, offset: int):
    """Host restatement of jb_pack_shard_topk (the CPU protocol tests' pack)."""
    import torch

    i = ids.to(torch.int64)
    g = torch.where(i >= 0, i + int(offset), torch.full_like(i, -1))
    rec = torch.stack([dists.to(torch.float64).view(torch.int64), g], dim=2)
    return rec.reshape(ids.shape[0], RECORD_WORDS * ids.shape[1])


def sharded_knn(local_search, queries, k: int, shard_start: int, group=None, root: int = 0, merge=None,
                device=None, nq: int | None = None, dims: int | None = None, pack=None):
    """Broadcast -> local search -> pack -> one all-gather -> merge.

    local_search(q) -> (ids int32 [nq,k], dists f64 [nq,k]) in shard-local ids.
    `queries` is a tensor on the root rank; other ranks may pass None. When every
    rank passes `nq` and `dims`, nothing is read back to the host; otherwise the
    root broadcasts the shape first (one small host read).
    merge(records [S, nq, 2k], k) -> global (int64 ids, f64 dists) on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import comm

    rank = dist.get_rank(group)
    dev = device if device is not None else (queries.device if queries is not None else torch.device("cpu"))
    if nq is None or dims is None:
        shape = torch.zeros(2, dtype=torch.int64, device=dev)
        if rank == root:
            shape[0], shape[1] = queries.shape[0], queries.shape[1]
        comm.broadcast(shape, src=root, group=group)
        nq, dims = (int(v) for v in shape.tolist())
    if rank != root:
        queries = torch.empty((nq, dims), dtype=torch.float32, device=dev)
    comm.broadcast(queries, src=root, group=group)
    ids, ds = local_search(queries)
    ids = ids.to(device=dev, dtype=torch.int32)
    ds = ds.to(device=dev, dtype=torch.float64)
    rec = (pack or (pack_topk_device if dev.type == "cuda" else pack_topk_host))(ids, ds, shard_start)
    all_rec = comm.all_gather(rec, group=group)  # [world, nq, 2k]
    return (merge or merge_records_device)(all_rec, k)


class ShardedIndex:
    """One rank's view of a sharded index: its graph, exact rows, optional RaBitQ
    codes, and the global id base of its shard.

    Bulk-built: `ShardedIndex(graph, dataset, shard_start, rabitq=...)`.
    Streaming: `ShardedIndex.empty(dims, shard_capacity, degree_cap)` then
    `insert_batch(rows, params)` on every rank — the new rows are broadcast from
    the root and split contiguously across the shards; each rank inserts its
    slice into its own graph (global id = rank * shard_capacity + local id).
    """

    def __init__(self, graph, dataset, shard_start: int, rabitq=None, group=None):
        import torch.distributed as dist

        self.graph, self.dataset, self.shard_start = graph, dataset, int(shard_start)
        self.rabitq, self.group = rabitq, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self._rows = None  # device row buffer (streaming shards)
        self._offsets = None

    @classmethod
    def empty(cls, dims: int, shard_capacity: int, degree_cap: int, group=None) -> "ShardedIndex":
        import torch.distributed as dist

        from .graph import GraphIndex

        torch = _lib.require_cuda()
        rank = dist.get_rank(group)
        si = cls(GraphIndex(shard_capacity, degree_cap), None, rank * shard_capacity, group=group)
        si._rows = torch.empty((shard_capacity, dims), dtype=torch.float32, device="cuda")
        return si

    @property
    def offsets(self) -> np.ndarray:
        """Global id base of every shard (gathered once, cached)."""
        if self._offsets is None:
            import torch

            from . import comm

            _lib.require_cuda()
            t = torch.tensor([self.shard_start], dtype=torch.int64, device="cuda")
            self._offsets = comm.all_gather(t, group=self.group).reshape(-1).cpu().numpy()
        return self._offsets

    def global_ids(self, local_ids):
        return np.asarray(local_ids, dtype=np.int64) + self.shard_start

    def insert_batch(self, rows, params, nb: int | None = None, root: int = 0):
        """Route a batch of new rows to the shards: broadcast from `root`, each rank
        inserts rows [shard_range(nb, rank, world)) into its graph (batch_insert,
        reference build.py:296-348). Returns this rank's new global ids."""
        import torch

        from . import comm
        from .build import batch_insert
        from .core import VectorDataset

        if self._rows is None:
            raise ValueError("insert_batch needs a streaming shard (ShardedIndex.empty)")
        if self.rabitq is not None:
            raise ValueError("RaBitQ shards are fit once; refit after streaming inserts")
        D = self._rows.shape[1]
        if nb is None:
            shape = torch.zeros(1, dtype=torch.int64, device="cuda")
            if self.rank == root:
                shape[0] = rows.shape[0]
            comm.broadcast(shape, src=root, group=self.group)
            nb = int(shape.item())
        if self.rank == root:
            buf = rows if isinstance(rows, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(rows, np.float32))
            buf = buf.to("cuda", dtype=torch.float32).contiguous()
        else:
            buf = torch.empty((nb, D), dtype=torch.float32, device="cuda")
        comm.broadcast(buf, src=root, group=self.group)
        lo, hi = shard_range(nb, self.rank, self.world)
        start = self.graph.active_count
        stop = start + (hi - lo)
        if stop > self._rows.shape[0]:
            raise ValueError("shard capacity exceeded")
        self._rows[start:stop] = buf[lo:hi]
        self.dataset = VectorDataset.from_device(self._rows[:stop])
        if stop > start:
            batch_insert(self.graph, self.dataset, range(start, stop), params)
        return np.arange(start, stop, dtype=np.int64) + self.shard_start

    def _local(self, params):
        from .search import search_knn_batch_device

        source = self.rabitq if self.rabitq is not None else self.dataset
        return lambda qq: search_knn_batch_device(self.graph, source, qq, params, exact_data=self.dataset)

    def search_knn_batch_device(self, q_dev, params, nq: int | None = None, root: int = 0):
        """Global top-k over all shards from device queries on `root` (None elsewhere);
        every rank gets the merged (int64 global ids, f64 dists) device tensors. With
        `nq` given on every rank the call never synchronizes the host."""
        torch = _lib.require_cuda()
        dims = self.dataset.dims if self.dataset is not None else self._rows.shape[1]
        return sharded_knn(self._local(params), q_dev, params.k, self.shard_start, group=self.group, root=root,
                           device=torch.device("cuda"), nq=nq, dims=dims if nq is not None else None)

    def search_knn_batch(self, queries, params, root: int = 0):
        """Host queries on `root` (None elsewhere) -> merged device results on every rank."""
        torch = _lib.require_cuda()
        q = None
        if queries is not None:
            q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(queries, dtype=np.float32))
            q = q.to("cuda", non_blocking=True)
        return self.search_knn_batch_device(q, params, root=root)
