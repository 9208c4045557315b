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
