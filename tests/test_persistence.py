"""graph.bin / rabitq.bin byte-identity with the reference's own writers
(graph.py:101-156, rabitq.py:183-222). The fixtures tests/golden/graph_g33.bin and
rabitq_m4.bin were written by beamann's save() (tests/golden/make_golden.py
persistence). CPU: load -> save round trips byte for byte and the loaded arrays
equal the oracle's; GPU: a device build / fit saved by this package is the
reference's file, byte for byte."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, gaussian, golden
from oracle import rabitq as orq

GRAPH_BIN = os.path.join(GOLDEN, "graph_g33.bin")
RABITQ_BIN = os.path.join(GOLDEN, "rabitq_m4.bin")


def _bytes(p):
    with open(p, "rb") as fh:
        return fh.read()


def test_graph_bin_load_save_round_trip(tmp_path):
    from paper_2601_07048_b200.graph import GraphIndex

    g = GraphIndex.load(GRAPH_BIN)
    f = golden("g33")
    np.testing.assert_array_equal(g.adjacency[:g.active_count], f["adjacency"])
    assert g.entry_point == int(f["entry"])
    out = tmp_path / "graph.bin"
    g.save(out)
    assert _bytes(out) == _bytes(GRAPH_BIN)
    g2 = GraphIndex.load(GRAPH_BIN, capacity=1000)  # spare capacity for inserts
    assert g2.capacity == 1000 and g2.active_count == 800
    g2.save(out)
    assert _bytes(out) == _bytes(GRAPH_BIN)


def test_rabitq_bin_load_save_round_trip(tmp_path):
    from paper_2601_07048_b200.rabitq import RaBitQIndex

    idx = RaBitQIndex.load(RABITQ_BIN)
    c, codes, meta = orq.fit(gaussian(300, 40, 71), 4, 72)
    np.testing.assert_array_equal(idx.codes, codes)
    np.testing.assert_array_equal(idx.meta.view(np.uint32), meta.view(np.uint32))
    np.testing.assert_array_equal(idx.centroid, c)
    assert (idx.bits, idx.rotation_seed, idx.dims) == (4, 72, 40)
    out = tmp_path / "rabitq.bin"
    idx.save(out)
    assert _bytes(out) == _bytes(RABITQ_BIN)


def test_truncated_files_raise_format_error(tmp_path):
    from paper_2601_07048_b200.graph import FormatError, GraphIndex
    from paper_2601_07048_b200.rabitq import RaBitQIndex

    for src, cls in ((GRAPH_BIN, GraphIndex), (RABITQ_BIN, RaBitQIndex)):
        p = tmp_path / "bad.bin"
        p.write_bytes(_bytes(src)[:-4])
        with pytest.raises(ValueError, match="expected"):
            cls.load(p)
        with pytest.raises(FormatError):
            cls.load(tmp_path / "missing.bin")


@pytest.mark.gpu
def test_device_build_and_fit_save_the_reference_files(tmp_path):
    import paper_2601_07048_b200 as jb

    g = jb.build(jb.VectorDataset(gaussian(800, 33, 5)), jb.BuildParams(degree_cap=8, build_beam_width=16, alpha=1.3))
    g.save(tmp_path / "graph.bin")
    assert _bytes(tmp_path / "graph.bin") == _bytes(GRAPH_BIN)
    idx = jb.rabitq_fit(jb.VectorDataset(gaussian(300, 40, 71)), bits=4, seed=72)
    idx.save(tmp_path / "rabitq.bin")
    assert _bytes(tmp_path / "rabitq.bin") == _bytes(RABITQ_BIN)


@pytest.mark.gpu
def test_reference_written_files_search_on_device():
    import paper_2601_07048_b200 as jb
    from oracle import search as osearch

    x, q = gaussian(800, 33, 5), gaussian(40, 33, 6)
    g = jb.GraphIndex.load(GRAPH_BIN)
    res = jb.run_beam_searches(g, jb.VectorDataset(x), q, 16)
    f = golden("g33")
    ores = osearch.beam_search(f["adjacency"], 800, int(f["entry"]), osearch.ExactSource(x, q), len(q), 16)
    for r, o in zip(res, ores):
        np.testing.assert_array_equal(r.frontier_ids, o.frontier_ids)
        np.testing.assert_array_equal(r.visited_ids, o.visited_ids)
    idx = jb.RaBitQIndex.load(RABITQ_BIN)
    xr = gaussian(300, 40, 71)
    gr = jb.build(jb.VectorDataset(xr), jb.BuildParams(degree_cap=8, build_beam_width=16))
    ids, _ = jb.search_knn_batch(gr, idx, gaussian(10, 40, 3), jb.SearchParams(beam_width=16, k=5, rerank=True),
                                 exact_data=jb.VectorDataset(xr))
    assert ids.shape == (10, 5) and (ids >= 0).all()
