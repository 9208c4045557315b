"""GPU: the device top-k merge of the sharded path (jb_merge_shard_topk) equals
the oracle merge by (dist, global id), including padding and cross-shard ties."""

import numpy as np
import pytest

from oracle.knn import merge_shard_topk

pytestmark = pytest.mark.gpu


def test_merge_kernel_matches_oracle():
    import torch

    from paper_2601_07048_b200.shard import merge_topk_device

    rng = np.random.default_rng(4)
    S, nq, k = 5, 300, 10
    d = np.sort(rng.integers(0, 50, size=(S, nq, k)).astype(np.float64), axis=2)  # many ties
    ids = np.zeros((S, nq, k), dtype=np.int32)
    for s in range(S):
        for q in range(nq):
            ids[s, q] = np.sort(rng.choice(1000, size=k, replace=False))
    # (dist, id) sorted within each shard list, as the search emits them
    for s in range(S):
        for q in range(nq):
            o = np.lexsort((ids[s, q], d[s, q]))
            ids[s, q], d[s, q] = ids[s, q][o], d[s, q][o]
    ids[2, :50, 6:] = -1   # short lists padded with -1
    d[2, :50, 6:] = np.inf
    offs = [0, 1000, 2000, 3000, 4000]
    gi, gd = merge_topk_device(torch.from_numpy(ids).cuda(), torch.from_numpy(d).cuda(), offs, k)
    ei, ed = merge_shard_topk(ids, d, offs, k)
    np.testing.assert_array_equal(gi.cpu().numpy(), ei)
    np.testing.assert_array_equal(gd.cpu().numpy(), ed)


def _sharded_worker(rank, world, port, out):
    """One rank of a world-size-2 gloo job on the single GPU: ShardedIndex over the
    product kernels (bulk-built shard search, and streaming shard-routed inserts)."""
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    try:
        import paper_2601_07048_b200 as jb
        from paper_2601_07048_b200.shard import ShardedIndex, shard_range

        x, q = _shard_data()
        lo, hi = shard_range(len(x), rank, world)
        params = jb.BuildParams(degree_cap=12, build_beam_width=24, alpha=1.2, max_batch=200)
        ds = jb.VectorDataset(x[lo:hi])
        g = jb.build(ds, params)
        si = ShardedIndex(g, ds, lo)
        sp = jb.SearchParams(beam_width=24, k=5)
        qd = torch.from_numpy(q).cuda()
        gi, gd = si.search_knn_batch_device(qd if rank == 0 else None, sp, nq=len(q))
        gi2, gd2 = si.search_knn_batch(q if rank == 0 else None, sp)
        assert torch.equal(gi, gi2) and torch.equal(gd, gd2)
        assert list(si.offsets) == [shard_range(len(x), r, world)[0] for r in range(world)]
        # streaming: two routed batches into empty shards of capacity 1000
        ss = ShardedIndex.empty(x.shape[1], 1000, 12)
        ids1 = ss.insert_batch(x[:500] if rank == 0 else None, params, nb=500)
        ids2 = ss.insert_batch(x[500:900] if rank == 0 else None, params)
        out[rank] = dict(ids=gi.cpu().numpy(), d=gd.cpu().numpy(), adj=ss.graph.adjacency[:ss.graph.active_count].copy(),
                         gids=np.concatenate([ids1, ids2]))
    finally:
        dist.destroy_process_group()


def _shard_data():
    g = np.random.default_rng(8)
    return g.standard_normal((1500, 16)).astype(np.float32), g.standard_normal((40, 16)).astype(np.float32)


def test_sharded_index_gloo_world2_matches_oracle():
    import socket

    import torch.multiprocessing as mp

    from oracle import search as osearch
    from oracle import vamana
    from paper_2601_07048_b200.shard import shard_range

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_sharded_worker, args=(2, port, out), nprocs=2, join=True)
    x, q = _shard_data()
    per, offs = [], []
    for r in range(2):
        lo, hi = shard_range(len(x), r, 2)
        og = vamana.build(x[lo:hi], R=12, L=24, alpha=1.2, max_batch=200)
        res = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x[lo:hi], q), len(q), 24)
        per.append(osearch.topk(res, 5))
        offs.append(lo)
    ei, ed = merge_shard_topk(np.stack([p[0] for p in per]), np.stack([p[1] for p in per]), offs, 5)
    for r in range(2):
        np.testing.assert_array_equal(out[r]["ids"], ei)
        np.testing.assert_array_equal(out[r]["d"], ed)
        # routed inserts: rank r got rows [shard_range(500)) then [shard_range(400)) of the second batch
        a = shard_range(500, r, 2)
        b = shard_range(400, r, 2)
        rows = np.concatenate([x[a[0]:a[1]], x[500 + b[0]:500 + b[1]]])
        og = vamana.Graph(1000, 12)
        vamana.batch_insert(og, rows, 0, a[1] - a[0], 12, 24, 1.2)
        vamana.batch_insert(og, rows, a[1] - a[0], len(rows), 12, 24, 1.2)
        np.testing.assert_array_equal(out[r]["adj"], og.adj[:len(rows)])
        np.testing.assert_array_equal(out[r]["gids"], np.arange(len(rows)) + r * 1000)
