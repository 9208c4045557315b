"""Sharded search across the GPUs of one box (north-star 4).

Partition: contiguous global-id ranges, shard s = [s*N/G, (s+1)*N/G); each rank
builds and owns its own graph (+ RaBitQ codes) over its shard, and inserts are
routed to the owning shard with no cross-GPU exchange. Per query batch:

  1. the root rank's queries are broadcast (NCCL, NVLink),
  2. every rank runs the single-GPU kernels on its shard,
  3. per-shard top-k lists (int32 local id + f64 dist, k*12 B per query) are
     all-gathered (NCCL) and
  4. merged on device by (dist, global id) with jb_merge_shard_topk.

One process per GPU; `torch.distributed` (backend "nccl") is the plumbing.
The protocol is written against injectable `local_search` / `merge` callables so
the same code path is exercised by world-size-2 gloo tests on CPU.
"""

from __future__ import annotations

import numpy as np

from . import _lib

__all__ = ["shard_range", "sharded_knn", "merge_topk_device", "ShardedIndex"]


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


def sharded_knn(local_search, queries, k: int, shard_start: int, group=None, root: int = 0, merge=None,
                device=None):
    """Broadcast -> local search -> all-gather -> merge.

    local_search(q) -> (ids int32 [nq,k], dists f64 [nq,k]) in shard-local ids.
    `queries` is a tensor on the root rank (shape known to all ranks through a
    small broadcast of the shape first); other ranks may pass None.
    Returns global (int64 ids, f64 dists) on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import comm

    rank = dist.get_rank(group)
    dev = device if device is not None else (queries.device if queries is not None else torch.device("cpu"))
    shape = torch.zeros(2, dtype=torch.int64, device=dev)
    if rank == root:
        shape[0], shape[1] = queries.shape[0], queries.shape[1]
    comm.broadcast(shape, src=root, group=group)
    nq, D = int(shape[0]), int(shape[1])
    if rank != root:
        queries = torch.empty((nq, D), dtype=torch.float32, device=dev)
    comm.broadcast(queries, src=root, group=group)
    ids, ds = local_search(queries)
    ids = ids.to(device=dev, dtype=torch.int32).contiguous()
    ds = ds.to(device=dev, dtype=torch.float64).contiguous()
    all_ids = comm.all_gather(ids, group=group)   # [world, nq, k]
    all_d = comm.all_gather(ds, group=group)
    offs = torch.tensor([shard_start], dtype=torch.int64, device=dev)
    offsets = comm.all_gather(offs, group=group).reshape(-1).cpu().numpy()
    if merge is None:
        merge = merge_topk_device
    return merge(all_ids, all_d, offsets, k)


class ShardedIndex:
    """One rank's view of a sharded index: its graph, exact rows, optional RaBitQ
    codes, and the global id offset of its shard."""

    def __init__(self, graph, dataset, shard_start: int, rabitq=None, group=None):
        self.graph, self.dataset, self.shard_start = graph, dataset, int(shard_start)
        self.rabitq, self.group = rabitq, group

    def search_knn_batch(self, queries, params, root: int = 0):
        """Global top-k over all shards; every rank gets the merged result."""
        from .search import search_knn_batch_device

        torch = _lib.require_cuda()
        q = None
        if queries is not None:
            q = queries if isinstance(queries, torch.Tensor) else torch.from_numpy(
                np.ascontiguousarray(queries, dtype=np.float32))
            q = q.to("cuda", non_blocking=True)
        source = self.rabitq if self.rabitq is not None else self.dataset
        return sharded_knn(
            lambda qq: search_knn_batch_device(self.graph, source, qq, params, exact_data=self.dataset),
            q, params.k, self.shard_start, group=self.group, root=root, device=torch.device("cuda"))
