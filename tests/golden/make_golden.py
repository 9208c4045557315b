"""Generate golden fixtures by running the LIVE reference (`beamann`) in this container.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Reads /root/reference/pkg/src (read-only; present only in the build container,
never on the GPU box). Writes tests/golden/*.npz. Inputs are regenerated from
seeds in the tests (numpy PCG64 is deterministic), so only outputs are stored.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import beamann as ref  # noqa: E402
from beamann.search import run_beam_searches  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def lowrank(n, d, d_int, noise, seed):
    """SURVEY.md Appendix B generator (same recipe as paper_2601_07048_b200.core.gen_lowrank)."""
    g = np.random.default_rng(seed)
    a = g.standard_normal((d_int, d)) / np.sqrt(d_int)
    x = g.standard_normal((n, d_int)) @ a + noise * g.standard_normal((n, d))
    return x.astype(np.float32)


def ragged(results):
    out = {}
    for name in ("frontier_ids", "frontier_dists", "visited_ids", "visited_dists"):
        parts = [getattr(r, name) for r in results]
        out[name] = np.concatenate(parts) if parts else np.empty(0)
        out[name + "_len"] = np.array([p.size for p in parts], dtype=np.int64)
    out["hops"] = np.array([r.stats.hops for r in results], dtype=np.int64)
    out["evals"] = np.array([r.stats.distance_evals for r in results], dtype=np.int64)
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} B)")


def graph_fixture(name, data, R, L, alpha, max_batch=100_000):
    ds = ref.VectorDataset(data)
    t = time.time()
    g = ref.build(ds, ref.BuildParams(degree_cap=R, build_beam_width=L, alpha=alpha, max_batch=max_batch))
    print(f"{name}: reference build {data.shape} in {time.time() - t:.1f}s")
    n = g.active_count
    return g, dict(adjacency=g.adjacency[:n].copy(), degrees=g.degrees[:n].copy(),
                   entry=np.int64(g.entry_point), active=np.int64(n))


def two_pass():
    """6. two_pass build (insertion at alpha=1, refinement at the final alpha) in several refine batches."""
    data = ref.gen_synthetic(1500, 32, seed=21).data
    t = time.time()
    g = ref.build(ref.VectorDataset(data), ref.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2,
                                                           max_batch=400, two_pass=True))
    print(f"two_pass: reference build {data.shape} in {time.time() - t:.1f}s")
    n = g.active_count
    save("two_pass", adjacency=g.adjacency[:n].copy(), degrees=g.degrees[:n].copy(), entry=np.int64(g.entry_point))


def u8_rows(n, d, seed):
    """BigANN-like u8 rows: a low-rank f32 sample affinely mapped to [0, 255] and rounded."""
    x = lowrank(n, d, 8, 0.05, seed)
    lo, hi = x.min(), x.max()
    return np.clip(np.rint((x - lo) / (hi - lo) * 255.0), 0, 255).astype(np.uint8)


def u8():
    """7. u8 element kind: integer-distance build (several batches), search trace, top-k, GT, medoid."""
    rows = u8_rows(2600, 32, seed=31)
    data, q = rows[:2500], rows[2500:]
    ds = ref.VectorDataset(data)
    t = time.time()
    g = ref.build(ds, ref.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2, max_batch=700))
    print(f"u8: reference build {data.shape} in {time.time() - t:.1f}s")
    n = g.active_count
    res = run_beam_searches(g, ds, q, 32)
    ids, dists = ref.search_knn_batch(g, ds, q, ref.SearchParams(beam_width=32, k=10))
    gt = ref.exact_knn(ds, ref.VectorDataset(q), 10)
    save("u8", adjacency=g.adjacency[:n].copy(), degrees=g.degrees[:n].copy(), entry=np.int64(g.entry_point),
         active=np.int64(n), **{"L32_" + k: v for k, v in ragged(res).items()}, knn_ids=ids, knn_dists=dists,
         gt_ids=gt.ids, gt_dists=gt.distances, medoid=np.int64(ref.medoid(ds)))


def quantized():
    """8. quantized construction: build with a RaBitQ quantizer (m=1 and m=4), two_pass at m=4."""
    data = ref.gen_synthetic(1200, 32, seed=51).data
    ds = ref.VectorDataset(data)
    out = {}
    for bits, two in ((1, False), (4, False), (4, True)):
        idx = ref.rabitq_fit(ds, bits=bits, seed=52)
        t = time.time()
        g = ref.build(ds, ref.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2, max_batch=300, two_pass=two),
                      quantizer=idx)
        tag = f"m{bits}" + ("_2p" if two else "")
        print(f"quantized {tag}: reference build {data.shape} in {time.time() - t:.1f}s")
        n = g.active_count
        out[tag + "_adjacency"] = g.adjacency[:n].copy()
        out[tag + "_degrees"] = g.degrees[:n].copy()
        out[tag + "_entry"] = np.int64(g.entry_point)
    save("quantized", **out)


def mips():
    """9. MIPS: mips_augment, inner-product ground truth, build + search on the augmented rows."""
    data = ref.gen_synthetic(2000, 24, seed=61).data * np.linspace(0.5, 2.0, 2000, dtype=np.float32)[:, None]
    q = ref.gen_synthetic(60, 24, seed=62).data
    ad, aq = ref.mips_augment(ref.VectorDataset(data), ref.VectorDataset(q))
    gt = ref.exact_knn(ref.VectorDataset(data), ref.VectorDataset(q), 10, ref.DistanceKind.INNER_PRODUCT)
    g = ref.build(ad.dataset, ref.BuildParams(degree_cap=16, build_beam_width=32, alpha=1.2))
    ids, dists = ref.search_knn_batch(g, ad.dataset, aq.dataset.data, ref.SearchParams(beam_width=32, k=10))
    save("mips", aug_data=ad.dataset.data, aug_queries=aq.dataset.data, max_norm=np.float64(ad.max_norm),
         gt_ids=gt.ids, gt_dists=gt.distances, adjacency=g.adjacency[:g.active_count].copy(),
         degrees=g.degrees[:g.active_count].copy(), entry=np.int64(g.entry_point), knn_ids=ids, knn_dists=dists)


def c1_graph():
    """10. BASELINE config 1 at full size (100K x 128 Gaussian, R=32, L=64, alpha=1.2): the
    reference build takes ~13 min here; only hashes are committed (c1_graph.json)."""
    import hashlib
    import json

    x = ref.gen_synthetic(100_000, 128, seed=0).data
    t = time.time()
    g = ref.build(ref.VectorDataset(x), ref.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
    n = g.active_count
    out = {"what": "reference (beamann) build of BASELINE config 1: gen_synthetic(100000, 128, seed=0), "
                   "BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2); SHA-1 of the int32 adjacency "
                   "[100000, 32] and degrees, and the entry point",
           "made_by": f"tests/golden/make_golden.py c1_graph ({time.time() - t:.0f} s on the container CPU)",
           "adjacency_sha1": hashlib.sha1(np.ascontiguousarray(g.adjacency[:n]).tobytes()).hexdigest(),
           "degrees_sha1": hashlib.sha1(np.ascontiguousarray(g.degrees[:n]).tobytes()).hexdigest(),
           "entry": int(g.entry_point)}
    with open(os.path.join(HERE, "c1_graph.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def bench_rabitq():
    """11. The bench workload's RaBitQ fit + query bind at full size (1M x 128 m=1): hashes only
    (bench_rabitq.json). Rows from workload.lowrank (the generator both bench arms use)."""
    import hashlib
    import json

    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    import workload

    x = workload.lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
    q = workload.lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
    t = time.time()
    idx = ref.rabitq_fit(ref.VectorDataset(x), bits=1, seed=1)
    b = idx.bind(q)
    sha = lambda a: hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    out = {"what": "reference (beamann) rabitq_fit(bits=1, seed=1) of the bench index rows gen_lowrank(1000000, 128, "
                   "seed=1, d_int=16, noise=0.05, basis_seed=0) and bind() of its 10000 queries gen_lowrank(10000, "
                   "128, seed=1000003, ...): SHA-1 of codes, meta, centroid, rotated queries, query_add, query_sumq",
           "made_by": f"tests/golden/make_golden.py bench_rabitq (beamann.rabitq_fit + RaBitQIndex.bind, "
                      f"{time.time() - t:.1f} s)",
           "codes": sha(idx.codes), "meta": sha(idx.meta), "centroid": sha(idx.centroid),
           "rotated": sha(b._rotated), "qadd": sha(b._qadd), "sumq": sha(b._qsumq)}
    with open(os.path.join(HERE, "bench_rabitq.json"), "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")


def persistence():
    """12. Byte-exact files written by the reference's own writers (graph.py:101-117,
    rabitq.py:183-192): graph.bin of the g33 build and rabitq.bin of an m=4 fit."""
    data33 = ref.gen_synthetic(800, 33, seed=5).data
    g = ref.build(ref.VectorDataset(data33), ref.BuildParams(degree_cap=8, build_beam_width=16, alpha=1.3))
    g.save(os.path.join(HERE, "graph_g33.bin"))
    x = ref.gen_synthetic(300, 40, seed=71).data
    idx = ref.rabitq_fit(ref.VectorDataset(x), bits=4, seed=72)
    idx.save(os.path.join(HERE, "rabitq_m4.bin"))
    for f in ("graph_g33.bin", "rabitq_m4.bin"):
        print(f"wrote {f} ({os.path.getsize(os.path.join(HERE, f))} B)")


def main():
    # 1. exact search + build on a small Gaussian graph (D=32, R=16, L=32)
    data = ref.gen_synthetic(3000, 32, seed=0).data
    g, gf = graph_fixture("g32", data, R=16, L=32, alpha=1.2)
    q = ref.gen_synthetic(200, 32, seed=1).data
    res = run_beam_searches(g, ref.VectorDataset(data), q, 32)
    res8 = run_beam_searches(g, ref.VectorDataset(data), q, 8)
    ids, dists = ref.search_knn_batch(g, ref.VectorDataset(data), q, ref.SearchParams(beam_width=32, k=10))
    save("g32", **gf, **{"L32_" + k: v for k, v in ragged(res).items()},
         **{"L8_" + k: v for k, v in ragged(res8).items()}, knn_ids=ids, knn_dists=dists)

    # 2. odd dims (non-16B-aligned rows), D=33, R=8
    data33 = ref.gen_synthetic(800, 33, seed=5).data
    g33, gf33 = graph_fixture("g33", data33, R=8, L=16, alpha=1.3)
    q33 = ref.gen_synthetic(64, 33, seed=6).data
    res33 = run_beam_searches(g33, ref.VectorDataset(data33), q33, 16)
    save("g33", **gf33, **{"L16_" + k: v for k, v in ragged(res33).items()})

    # 3. low-rank 128-d build (R=32, L=64) + incremental inserts in 2% batches
    data128 = lowrank(4000, 128, 12, 0.05, seed=7)
    g128, gf128 = graph_fixture("g128", data128, R=32, L=64, alpha=1.2)
    q128 = lowrank(100, 128, 12, 0.05, seed=8)
    res128 = run_beam_searches(g128, ref.VectorDataset(data128), q128, 64)
    inc = ref.GraphIndex(capacity=4000, degree_cap=32)
    p = ref.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=80)
    ds128 = ref.VectorDataset(data128)
    ref.batch_insert(inc, ds128, range(0, 33), p)
    ref.insert_stream(inc, ds128, range(33, 1200), p)
    save("g128", **gf128, **{"L64_" + k: v for k, v in ragged(res128).items()},
         inc_adjacency=inc.adjacency[:1200].copy(), inc_degrees=inc.degrees[:1200].copy(),
         inc_entry=np.int64(inc.entry_point))

    # 4. RaBitQ fit / bind / quantized search + rerank on the g32 graph and 128-d data
    fx = {}
    x = ref.gen_synthetic(2000, 128, seed=2).data
    qq = ref.gen_synthetic(50, 128, seed=4).data
    for bits in (1, 2, 4, 8):
        idx = ref.rabitq_fit(ref.VectorDataset(x), bits=bits, seed=3)
        b = idx.bind(qq)
        fx[f"m{bits}_centroid"] = idx.centroid
        fx[f"m{bits}_codes"] = idx.codes
        fx[f"m{bits}_meta"] = idx.meta
        fx[f"m{bits}_rotated"] = b._rotated
        fx[f"m{bits}_qadd"] = b._qadd
        fx[f"m{bits}_sumq"] = b._qsumq
    idx1 = ref.rabitq_fit(ref.VectorDataset(data), bits=1, seed=11)
    idx4 = ref.rabitq_fit(ref.VectorDataset(data), bits=4, seed=11)
    for tag, idx in (("q1", idx1), ("q4", idx4)):
        r = run_beam_searches(g, idx, q, 32)
        fx.update({f"{tag}_" + k: v for k, v in ragged(r).items()})
        i2, d2 = ref.search_knn_batch(g, idx, q, ref.SearchParams(beam_width=32, k=10, rerank=True),
                                      exact_data=ref.VectorDataset(data))
        fx[f"{tag}_rr_ids"] = i2
        fx[f"{tag}_rr_dists"] = d2
    save("rabitq", **fx)

    # 5. exact kNN ground truth and medoid
    gt = ref.exact_knn(ref.VectorDataset(data), ref.VectorDataset(q), 20)
    save("misc", gt_ids=gt.ids, gt_dists=gt.distances,
         medoid32=np.int64(ref.medoid(ref.VectorDataset(data))),
         medoid128=np.int64(ref.medoid(ref.VectorDataset(data128))))


if __name__ == "__main__":
    # no arguments: every fixture; otherwise the named generators (e.g. two_pass)
    names = sys.argv[1:]
    if not names:
        main()
        two_pass()
        u8()
        quantized()
        mips()
    for n in names:
        globals()[n]()
