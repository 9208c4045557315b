"""CPU-only (gloo, world size 2): the sharded-search protocol of
paper_2601_07048_b200.shard — query broadcast from the root, per-shard search,
all-gather of per-shard top-k, merge by (dist, global id). The per-shard search
and the merge are injected (oracle restatements), so this exercises exactly the
distributed code path the NCCL ranks run, without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_07048_b200.shard import pack_topk_host, shard_range, sharded_knn

N, D, NQ, K, L = 1200, 16, 40, 5, 24


def _data():
    g = np.random.default_rng(3)
    return g.standard_normal((N, D)).astype(np.float32), g.standard_normal((NQ, D)).astype(np.float32)


def _local(x, lo, hi, q, k):
    from oracle import search as osearch
    from oracle import vamana

    og = vamana.build(x[lo:hi], R=12, L=L, alpha=1.2)
    res = osearch.beam_search(og.adj, og.active, og.entry, osearch.ExactSource(x[lo:hi], q), len(q), L)
    return osearch.topk(res, k)


def _merge(records, k):
    """All-gathered exchange records [S, nq, 2k] ({f64 dist, i64 global id}) -> the oracle merge."""
    from oracle.knn import merge_shard_topk

    r = records.numpy().reshape(records.shape[0], records.shape[1], k, 2)
    d = r[..., 0].copy().view(np.float64)
    gid = r[..., 1]
    ids = np.where(gid >= 0, gid, -1).astype(np.int32)
    i, d = merge_shard_topk(ids, d, [0] * records.shape[0], k)
    return torch.from_numpy(i), torch.from_numpy(d)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, q = _data()
        lo, hi = shard_range(N, rank, world)

        def local_search(qt):
            ids, ds = _local(x, lo, hi, qt.numpy(), K)
            return torch.from_numpy(ids), torch.from_numpy(ds)

        qt = torch.from_numpy(q) if rank == 0 else None
        # shape broadcast path (non-root ranks do not know the batch shape) ...
        gi, gd = sharded_knn(local_search, qt, K, lo, merge=_merge, device=torch.device("cpu"))
        # ... and the sync-free path with the shape known on every rank
        gi2, gd2 = sharded_knn(local_search, qt, K, lo, merge=_merge, device=torch.device("cpu"), nq=NQ, dims=D)
        assert torch.equal(gi, gi2) and torch.equal(gd, gd2)
        out[rank] = (gi.numpy().tolist(), gd.numpy().tolist())
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_partition():
    for n, w in ((10, 3), (1_000_000, 8), (7, 7), (5, 8)):
        rs = [shard_range(n, r, w) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 3, 3)


def test_sharded_search_gloo_world2_matches_single_process_merge():
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    x, q = _data()
    from oracle.knn import merge_shard_topk

    per = []
    for r in range(2):
        lo, hi = shard_range(N, r, 2)
        per.append(_local(x, lo, hi, q, K))
    exp_i, exp_d = merge_shard_topk(np.stack([p[0] for p in per]), np.stack([p[1] for p in per]),
                                    [shard_range(N, r, 2)[0] for r in range(2)], K)
    for r in range(2):
        gi, gd = out[r]
        np.testing.assert_array_equal(np.asarray(gi), exp_i)
        np.testing.assert_array_equal(np.asarray(gd), exp_d)
    # merged ids are global and come from both shards
    assert (exp_i >= N // 2).any() and (exp_i < N // 2).any()


def test_pack_records_host_layout():
    ids = torch.tensor([[3, -1], [0, 7]], dtype=torch.int32)
    d = torch.tensor([[1.5, float("inf")], [0.0, 2.25]], dtype=torch.float64)
    r = pack_topk_host(ids, d, 100).numpy().reshape(2, 2, 2)
    assert r[0, 0, 1] == 103 and r[0, 1, 1] == -1 and r[1, 1, 1] == 107
    assert r[1, 1, 0:1].view(np.float64)[0] == 2.25
