"""Secondary measurements for the other BASELINE.json configs (DESIGN.md numbers).
bench.py stays the single headline harness (configs[1]); this script runs:

  c1  synthetic 100K x 128 Gaussian, R=32 L_build=64 alpha=1.2, 10K queries, k=10, EXACT
      distances, L sweep 16..256 (the reference's own CPU-runnable config): device QPS,
      recall, ids checked identical to the oracle on a sample, oracle CPU QPS
  c3  GIST-shaped 1M x 960 low-rank (d_int=16 default, --dint), RaBitQ m=4 + fp32 rerank: QPS at recall 0.95
  c4  DEEP-shaped 96-d low-rank: bulk build of the first N0, then insert_stream in batches of
      100K interleaved with a 10K-query exact search after every batch (inserts/s, QPS)
  c5  one 12.5M x 96 shard of the 100M x 96 index (the per-GPU work at 8 GPUs)
  u8  BigANN-shaped 1M x 128 u8 rows (the paper's headline dataset kind; not a BASELINE
      config): exact integer-distance build and search, QPS at recall 0.95

    python bench_configs.py c1|c3|c4|c5|u8 [--n N] [--total T] [--dint D]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _timed(fn, reps=5, warm=2):
    import torch

    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    evs = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        evs.append((a, b))
    torch.cuda.synchronize()
    return float(np.mean([a.elapsed_time(b) for a, b in evs]))


def _warm_build(jb, x, params):
    """Untimed build on a prefix of the same rows (min(n/4, 250K)) so the timed build
    does not pay the process's one-time costs (module loads, pool growth), as in
    bench.py."""
    import torch

    nw = min(len(x) // 4, 250_000)
    if nw > params.degree_cap + 1:
        jb.build(jb.VectorDataset(x[:nw]), params)
    torch.cuda.synchronize()


def c1(args):
    import torch

    import paper_2601_07048_b200 as jb
    from oracle import search as osearch

    x = jb.gen_synthetic(args.n or 100_000, 128, seed=0).data
    q = jb.gen_synthetic(10_000, 128, seed=1).data
    ds = jb.VectorDataset(x)
    R, Lb = args.R or 32, args.lbuild or 64
    _warm_build(jb, x, jb.BuildParams(degree_cap=R, build_beam_width=Lb, alpha=1.2))
    t0 = time.perf_counter()
    g = jb.build(ds, jb.BuildParams(degree_cap=R, build_beam_width=Lb, alpha=1.2))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    q_dev = torch.from_numpy(q).cuda()
    gi, gd = bench._gt_device(ds.device().x, q_dev, 100)
    gt = jb.GroundTruth(gi.cpu().numpy(), gd.cpu().numpy().astype(np.float32))
    out = {"config": "c1", "n": len(x), "build_s": round(t_build, 3), "inserts_per_s": round(len(x) / t_build, 1),
           "sweep": []}
    for L in (16, 32, 64, 128, 256):
        sp = jb.SearchParams(beam_width=L, k=10)
        ms = _timed(lambda: jb.search_knn_batch_device(g, ds, q_dev, sp))
        ids, _ = jb.search_knn_batch_device(g, ds, q_dev, sp)
        r = jb.recall_at_k(ids.cpu().numpy(), gt, 10)
        out["sweep"].append({"L": L, "recall": round(r, 4), "qps_device": round(10_000 / (ms / 1e3), 1),
                             "ms": round(ms, 3)})
    # parity on the GPU-built graph + CPU oracle speed at L=64 (1 process)
    ns = 1000
    t0 = time.perf_counter()
    ores = osearch.beam_search(np.ascontiguousarray(g.adjacency), g.active_count, g.entry_point,
                               osearch.ExactSource(x, q[:ns]), ns, 64)
    el = time.perf_counter() - t0
    res = jb.run_beam_searches(g, ds, q[:ns], 64)
    same = all(np.array_equal(a.frontier_ids, b.frontier_ids) and np.array_equal(a.visited_ids, b.visited_ids)
               for a, b in zip(res, ores))
    out["oracle_cpu_qps_L64_1proc"] = round(ns / el, 1)
    out["frontier_and_trace_identical_to_oracle"] = same
    return out


def c3(args):
    import torch

    import paper_2601_07048_b200 as jb

    n = args.n or 1_000_000
    dint = args.dint or 16
    x = jb.gen_lowrank(n, 960, seed=1, d_int=dint, noise=0.05, basis_seed=0)
    q = jb.gen_lowrank(10_000, 960, seed=1_000_003, d_int=dint, noise=0.05, basis_seed=0)
    ds = jb.VectorDataset(x)
    R, Lb = args.R or 32, args.lbuild or 64
    _warm_build(jb, x, jb.BuildParams(degree_cap=R, build_beam_width=Lb, alpha=1.2))
    t0 = time.perf_counter()
    g = jb.build(ds, jb.BuildParams(degree_cap=R, build_beam_width=Lb, alpha=1.2))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    idx = jb.rabitq_fit(ds, bits=4, seed=1)
    torch.cuda.synchronize()
    t_fit = time.perf_counter() - t0
    q_dev = torch.from_numpy(q).cuda()
    gi, gd = bench._gt_device(ds.device().x, q_dev, 100)
    gt = jb.GroundTruth(gi.cpu().numpy(), gd.cpu().numpy().astype(np.float32))
    out = {"config": "c3", "n": n, "dims": 960, "d_int": dint, "R": R, "L_build": Lb, "bits": 4,
           "build_s": round(t_build, 2),
           "inserts_per_s": round(n / t_build, 1), "rabitq_fit_s": round(t_fit, 3),
           "bytes_per_vector": {"f32": 3840, "rabitq_record": int(jb._lib.lib().jb_rabitq_record_bytes(960, 4))},
           "sweep": [], "sweep_popcount": []}
    for est, key in (("reference", "sweep"), ("popcount", "sweep_popcount")):
        for L in bench.SWEEP:
            sp = jb.SearchParams(beam_width=L, k=10, rerank=True, estimator=est)
            ms = _timed(lambda: jb.search_knn_batch_device(g, idx, q_dev, sp, exact_data=ds), reps=3, warm=1)
            ids, _ = jb.search_knn_batch_device(g, idx, q_dev, sp, exact_data=ds)
            r = jb.recall_at_k(ids.cpu().numpy(), gt, 10)
            out[key].append({"L": L, "recall": round(r, 4), "qps_device": round(10_000 / (ms / 1e3), 1)})
            if r >= 0.95:
                break
    return out


def c4(args):
    import torch

    import paper_2601_07048_b200 as jb

    total = args.total or 10_000_000
    n0 = args.n or 1_000_000
    x = jb.gen_lowrank(total, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
    q = jb.gen_lowrank(10_000, 96, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
    ds = jb.VectorDataset(x)
    ds.device()
    params = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000,
                            repair_beam_width=args.repair_beam)
    g = jb.GraphIndex(capacity=total, degree_cap=32)
    _warm_build(jb, x[:n0], params)
    t0 = time.perf_counter()
    # bulk phase on the first n0 rows: same schedule as build() over a prefix
    size, pos = params.degree_cap + 1, 0
    while pos < n0:
        stop = min(n0, pos + size)
        jb.batch_insert(g, ds, range(pos, stop), params)
        pos, size = stop, min(size * 2, params.max_batch)
    torch.cuda.synchronize()
    t_bulk = time.perf_counter() - t0
    q_dev = torch.from_numpy(q).cuda()
    sp = jb.SearchParams(beam_width=64, k=10)
    ins_t, qps = [], []
    pos = n0
    while pos < total:
        stop = min(total, pos + params.max_batch)
        t0 = time.perf_counter()
        jb.insert_stream(g, ds, range(pos, stop), params)
        torch.cuda.synchronize()
        ins_t.append((stop - pos, time.perf_counter() - t0))
        # (the first call also allocates the search context: warm it once)
        ms = _timed(lambda: jb.search_knn_batch_device(g, ds, q_dev, sp), reps=1, warm=0 if qps else 1)
        qps.append(10_000 / (ms / 1e3))
        pos = stop
    ids, _ = jb.search_knn_batch_device(g, ds, q_dev, sp)
    gi, gd = bench._gt_device(ds.device().x, q_dev, 100)
    gt = jb.GroundTruth(gi.cpu().numpy(), gd.cpu().numpy().astype(np.float32))
    return {"config": "c4", "total": total, "bulk_n": n0, "repair_beam_width": args.repair_beam,
            "bulk_inserts_per_s": round(n0 / t_bulk, 1),
            "stream_batches": len(ins_t),
            "stream_inserts_per_s": round(sum(n for n, _ in ins_t) / sum(t for _, t in ins_t), 1),
            "stream_inserts_per_s_first_last": [round(ins_t[0][0] / ins_t[0][1], 1),
                                                round(ins_t[-1][0] / ins_t[-1][1], 1)] if ins_t else None,
            "search_qps_L64_exact_first_last": [round(qps[0], 1), round(qps[-1], 1)] if qps else None,
            "final_recall_at_10_L64": round(jb.recall_at_k(ids.cpu().numpy(), gt, 10), 4)}


def c5(args):
    """One shard of the 100M x 96 index at 8 GPUs (12.5M rows): the per-GPU work of
    the weak-scaling configuration, built and searched on one B200. Exact and
    RaBitQ-1 + rerank sweeps to recall@10 >= 0.95 against the shard's own exact GT."""
    import torch

    import paper_2601_07048_b200 as jb

    n = args.n or 12_500_000
    t0 = time.perf_counter()
    x = jb.gen_lowrank(n, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
    q = jb.gen_lowrank(10_000, 96, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
    t_gen = time.perf_counter() - t0
    ds = jb.VectorDataset(x)
    ds.device()
    bp = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000,
                        repair_beam_width=args.repair_beam)
    _warm_build(jb, x, bp)
    t0 = time.perf_counter()
    g = jb.build(ds, bp)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    idx = jb.rabitq_fit(ds, bits=1, seed=1)
    idx4 = jb.rabitq_fit(ds, bits=4, seed=1)
    q_dev = torch.from_numpy(q).cuda()
    gi, gd = bench._gt_device(ds.device().x, q_dev, 100)
    gt = jb.GroundTruth(gi.cpu().numpy(), gd.cpu().numpy().astype(np.float32))
    out = {"config": "c5-shard", "n": n, "repair_beam_width": args.repair_beam, "dims": 96, "gen_s": round(t_gen, 1), "build_s": round(t_build, 2),
           "inserts_per_s": round(n / t_build, 1), "hbm_bytes": {"vectors": n * 96 * 4, "graph": n * 32 * 4}}
    for name, src, kw in (("exact", ds, {}),
                          ("rabitq4_popcount_rerank", idx4, dict(rerank=True, estimator="popcount")),
                          ("rabitq1_popcount_rerank", idx, dict(rerank=True, estimator="popcount"))):
        pts = []
        for L in bench.SWEEP:
            sp = jb.SearchParams(beam_width=L, k=10, **kw)
            ms = _timed(lambda: jb.search_knn_batch_device(g, src, q_dev, sp, exact_data=ds), reps=3, warm=1)
            ids, _ = jb.search_knn_batch_device(g, src, q_dev, sp, exact_data=ds)
            r = jb.recall_at_k(ids.cpu().numpy(), gt, 10)
            pts.append({"L": L, "recall": round(r, 4), "qps_device": round(10_000 / (ms / 1e3), 1)})
            if r >= 0.95:
                break
        out[name] = pts
    return out


def u8(args):
    """BigANN-shaped u8: low-rank rows (d_int 16) mapped affinely to [0, 255]."""
    import torch

    import paper_2601_07048_b200 as jb

    n = args.n or 1_000_000
    x = jb.gen_lowrank(n + 10_000, 128, seed=1, d_int=args.dint or 16, noise=0.05, basis_seed=0)
    lo, hi = float(x.min()), float(x.max())
    rows = np.clip(np.rint((x - lo) / (hi - lo) * 255.0), 0, 255).astype(np.uint8)
    data, q = rows[:n], rows[n:]
    ds = jb.VectorDataset(data)
    ds.device()
    _warm_build(jb, data, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000))
    t0 = time.perf_counter()
    g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    q_dev = torch.from_numpy(q).cuda()
    gi, gd = bench._gt_device(ds.device_f32(), q_dev.float(), 100)
    gt = jb.GroundTruth(gi.cpu().numpy(), gd.cpu().numpy().astype(np.float32))
    out = {"config": "u8-bigann-shaped", "n": n, "dims": 128, "build_s": round(t_build, 2),
           "inserts_per_s": round(n / t_build, 1), "bytes_per_vector": 128}
    pts = []
    for L in bench.SWEEP:
        sp = jb.SearchParams(beam_width=L, k=10)
        ms = _timed(lambda: jb.search_knn_batch_device(g, ds, q_dev, sp), reps=3, warm=1)
        ids, _ = jb.search_knn_batch_device(g, ds, q_dev, sp)
        r = jb.recall_at_k(ids.cpu().numpy(), gt, 10)
        pts.append({"L": L, "recall": round(r, 4), "qps_device": round(10_000 / (ms / 1e3), 1)})
        if r >= 0.95:
            break
    out["exact_u8"] = pts
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("config", choices=["c1", "c3", "c4", "c5", "u8"])
    p.add_argument("--dint", type=int, default=0)
    p.add_argument("--R", type=int, default=0, help="c3: degree cap (default 32)")
    p.add_argument("--lbuild", type=int, default=0, help="c3: build beam width (default 64)")
    p.add_argument("--n", type=int, default=0)
    p.add_argument("--total", type=int, default=0)
    p.add_argument("--repair-beam", type=int, default=0,
                   help="c4/c5: approximate connectivity repair (BuildParams.repair_beam_width; 0 = exact)")
    p.add_argument("--out", default="")
    args = p.parse_args()
    import torch

    torch.cuda.set_device(0)
    res = {"c1": c1, "c3": c3, "c4": c4, "c5": c5, "u8": u8}[args.config](args)
    line = json.dumps(res)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


if __name__ == "__main__":
    main()
