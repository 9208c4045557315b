"""Benchmark: QPS at recall@10 >= 0.95 on a SIFT-1M-shaped synthetic index (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

Workload (per GPU shard): 1M x 128 f32 low-rank synthetic rows (workload.lowrank,
SURVEY.md Appendix B: d_int=16, noise 0.05), Vamana R=32, L_build=64, alpha=1.2,
max_batch=100K; RaBitQ 1-bit codes (seed 1) + fp32 rerank of the full beam, 10K
queries, k=10. The beam width L* is the smallest of a sweep whose recall@10
(reference recall_at_k semantics, exact f64 ground truth) reaches 0.95; a step is
one search of the 10K-query batch at L* (bind + search + rerank).

--impl b200 (default): everything on the GPU through the product library. `value`
is device-timed with inputs resident in HBM (L2 flushed between steps, outside the
timed events); `e2e` is the public API `search_knn_batch` with host queries in and
host ids/dists out. N>1: contiguous 1M-row shards per rank, queries broadcast over
NCCL, per-shard top-k all-gathered and merged on device; a unit is one
(query, shard) search, so per-GPU work is fixed (weak scaling).

--impl reference: the reference's algorithm on the host CPU only. This process
never imports the product package and never touches the GPU: it builds the same
1M index with the C restatement of beamann's batch_insert (oracle/c/jbo.c, every
host core; its graph hash equals the GPU arm's), fits RaBitQ with the numpy
restatement of beamann's fit, computes the ground truth on the CPU, calibrates L*
the same way, and times the reference search path (C port, all host threads;
the numpy port's 1-process and all-process figures are reported beside it). Its
`value` is the fastest of the three CPU variants.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402  (numpy only; shared by both arms)

SWEEP = (16, 24, 32, 48, 64, 80, 96, 104, 112, 120, 128, 144, 160, 192, 256, 384, 512, 768, 1024)
INDEX = {"R": 32, "L_build": 64, "alpha": 1.2, "max_batch": 100000}


def log(*a):
    if int(os.environ.get("RANK", "0")) == 0:
        print("[bench]", *a, file=sys.stderr, flush=True)


def _args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", default="c2", choices=["c2", "c5"],
                   help="c2: BASELINE configs[1] (1M x 128 per shard, RaBitQ-1); c5: configs[4], one 12.5M x 96 "
                        "shard of the 100M x 96 index per GPU (RaBitQ-4 + rerank)")
    p.add_argument("--shard-rows", dest="n", type=int, default=1_000_000, help="vectors per shard (GPU)")
    p.add_argument("--data", default="lowrank", choices=["lowrank", "gaussian"],
                   help="synthetic rows: low-rank (default) or the reference's iid Gaussian gen_synthetic")
    p.add_argument("--queries", dest="nq", type=int, default=10_000)
    p.add_argument("--dim", type=int, default=128)
    p.add_argument("--k", type=int, default=10)
    p.add_argument("--bits", type=int, default=1)
    p.add_argument("--target", type=float, default=0.95)
    p.add_argument("--beam", type=int, default=0, help="skip the sweep and use this L")
    p.add_argument("--stream-rows", dest="stream", type=int, default=20_000,
                   help="rows of the streaming batch_insert compared with the CPU port (0 = skip)")
    p.add_argument("--cpu-seconds", type=float, default=6.0, help="per numpy-port CPU sample")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--out", default="")
    p.add_argument("--hash-slots", type=int, default=0, help="visited-table slots per query (0 = library default)")
    p.add_argument("--estimator", default="auto", choices=["auto", "reference", "popcount"],
                   help="RaBitQ estimator; auto times both and reports the faster at the recall target")
    a = p.parse_args()
    if a.config == "c5":
        # DEEP-shaped 100M x 96 sharded over 8 GPUs: 12.5M rows per shard (BASELINE configs[4])
        a.n = a.n if a.n != 1_000_000 else 12_500_000
        a.dim = 96 if a.dim == 128 else a.dim
        a.bits = 4 if a.bits == 1 else a.bits
        a.stream = 0
        a.no_cpu = True
    return a


# ---------------------------------------------------------------------------
# shared by both arms


def _data(args, rank: int = 0):
    if args.data == "gaussian":  # the reference's gen_synthetic rows (core.py:209-233)
        return workload.gaussian(args.n, args.dim, 1 + rank), workload.gaussian(args.nq, args.dim, 1_000_003)
    x = workload.lowrank(args.n, args.dim, seed=1 + rank, d_int=16, noise=0.05, basis_seed=0)
    q = workload.lowrank(args.nq, args.dim, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
    return x, q


def _stream_rows(args):
    if args.data == "gaussian":
        return workload.gaussian(args.stream, args.dim, 777_001)
    return workload.lowrank(args.stream, args.dim, seed=777_001, d_int=16, noise=0.05, basis_seed=0)


def _graph_sha(adj: np.ndarray, deg: np.ndarray, active: int, entry: int) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(adj[:active], dtype=np.int32).tobytes())
    h.update(np.ascontiguousarray(deg[:active], dtype=np.int32).tobytes())
    h.update(np.int64(entry).tobytes())
    return h.hexdigest()[:16]


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _recall(ids, gt_i, gt_d, k):
    from oracle import knn as oknn  # recall_at_k semantics (reference bench.py:44-66)

    return oknn.recall_at_k(ids, gt_i, gt_d, k)


def _config(args, world, L):
    """Identical in both arms (same workload, same L*)."""
    shape = "SIFT-1M-shaped" if args.config == "c2" else f"DEEP-100M-shaped (one shard of {8 * args.n} at 8 GPUs)"
    rows = "iid Gaussian" if args.data == "gaussian" else "low-rank (d_int=16, noise 0.05)"
    return {"workload": f"{shape} synthetic {args.n}x{args.dim} {rows} "
                        f"per shard, RaBitQ {args.bits}-bit + fp32 rerank, {args.nq} queries, k={args.k}",
            "index": dict(INDEX), "beam_width": L, "shards": world, "parallelism": f"shard{world}",
            "l2": "flushed between timed steps (256 MB write, outside the events)"}


def _json_base(args, world, L):
    return {
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "metric": "QPS at recall@10=0.95", "unit": "queries/s", "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config(args, world, L),
    }


# ---------------------------------------------------------------------------
# reference arm (CPU only; never imports paper_2601_07048_b200)


def _np_search_task(payload):
    """numpy oracle port of beamann's search path: bind, lockstep RaBitQ search, rerank, top-k."""
    from oracle import rabitq as orq
    from oracle import search as osr

    (adj, active, entry, codes, meta, bits, dims, centroid, seed, x, qs, L, k) = payload
    rot, qadd, sumq = orq.bind(qs, centroid, bits, seed)
    src = orq.QuantSource(codes, meta, bits, dims, rot, qadd, sumq)
    res = osr.beam_search(adj, active, entry, src, len(qs), L)
    ids, _ = osr.topk(res, k, queries=qs, rerank_data=x)
    return np.asarray(ids)


_SHARED = {}


def _np_task(bounds):
    lo, hi = bounds
    s = _SHARED
    return _np_search_task((s["adj"], s["active"], s["entry"], s["codes"], s["meta"], s["bits"], s["dims"],
                            s["centroid"], s["seed"], s["x"], s["q"][lo:hi], s["L"], s["k"]))


def _np_search_sample(shared: dict, nq: int, procs: int, seconds: float):
    """Time the numpy port on a bounded query sample (~`seconds`); returns (n, elapsed, ids)."""
    import multiprocessing as mp

    _SHARED.clear()
    _SHARED.update(shared)
    t0 = time.perf_counter()
    _np_task((0, 40))
    per_q = (time.perf_counter() - t0) / 40
    n = int(max(40, min(nq, seconds / per_q * max(procs, 1) * 0.8)))
    n = max(procs, n - n % max(procs, 1))
    if procs <= 1:
        t0 = time.perf_counter()
        ids = _np_task((0, n))
        return n, time.perf_counter() - t0, ids
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    cuts = np.linspace(0, n, procs + 1).astype(int)
    with mp.get_context("fork").Pool(procs) as pool:
        pool.map(_np_task, [(0, 4)] * procs)  # fork + import warm-up
        t0 = time.perf_counter()
        parts = pool.map(_np_task, list(zip(cuts[:-1], cuts[1:])))
        el = time.perf_counter() - t0
    return n, el, np.concatenate(parts)


def _c_knn(g, quant, x, q, L, k, threads):
    """The C port of beamann's search_knn_batch path: bind (numpy, as beamann), lockstep
    RaBitQ search, exact rerank + top-k."""
    from oracle import cref

    keys, _, _ = cref.search_rabitq(g.adj, g.active, g.entry, quant, q, L, threads=threads)
    return cref.rerank_topk(x, q, cref.frontier_ids(keys), k, threads=threads)


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # under torchrun, rank 0 alone runs the CPU reference
    from oracle import cref, vamana

    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    x, q = _data(args)
    t_gen = time.perf_counter() - t0
    rows = cref.Rows(x, threads)
    t0 = time.perf_counter()
    g = cref.build(x, INDEX["R"], INDEX["L_build"], INDEX["alpha"], INDEX["max_batch"], threads=threads, rows=rows)
    t_build = time.perf_counter() - t0
    sha = _graph_sha(g.adj, g.deg, g.active, g.entry)
    log(f"[reference] C-port build {t_build:.1f}s ({args.n / t_build:.0f} inserts/s, {threads} threads) graph {sha}")
    t0 = time.perf_counter()
    quant = cref.Quantized.fit(x, args.bits, 1)
    t_fit = time.perf_counter() - t0
    t0 = time.perf_counter()
    gt_i, gt_d = cref.exact_knn(x, q, 100, threads=threads)
    gt_d = gt_d.astype(np.float32)
    log(f"[reference] fit {t_fit:.1f}s ground truth {time.perf_counter() - t0:.1f}s")

    pts, L = [], None
    for Lc in ((args.beam,) if args.beam else SWEEP):
        ids, _ = _c_knn(g, quant, x, q, Lc, args.k, threads)
        r = _recall(ids, gt_i, gt_d, args.k)
        pts.append({"L": Lc, "recall": round(r, 4)})
        log(f"[reference] sweep L={Lc} recall@{args.k}={r:.4f}")
        if r >= args.target:
            L = Lc
            break
    L = L or pts[-1]["L"]

    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        ids_c, _ = _c_knn(g, quant, x, q, L, args.k, threads)
        times.append(time.perf_counter() - t0)
    tt = times[args.warmup:]
    c_value = args.nq * len(tt) / sum(tt)

    shared = dict(adj=g.adj, active=g.active, entry=g.entry, codes=quant.codes, meta=quant.meta, bits=args.bits,
                  dims=args.dim, centroid=quant.centroid, seed=1, x=x, q=q, L=L, k=args.k)
    variants = {"c_port_threads": {"value": round(c_value, 1), "cores": threads,
                                   "sample": f"all {args.nq} queries per step, {args.steps} timed steps"}}
    n1, e1, ids1 = _np_search_sample(shared, args.nq, 1, args.cpu_seconds)
    variants["numpy_port_1proc"] = {"value": round(n1 / e1, 1), "cores": 1, "sample": f"first {n1} queries",
                                    "ids_identical_to_c_port": bool(np.array_equal(ids1, ids_c[:n1]))}
    nP, eP, idsP = _np_search_sample(shared, args.nq, threads, args.cpu_seconds)
    variants["numpy_port_procs"] = {"value": round(nP / eP, 1), "cores": threads,
                                    "sample": f"first {nP} queries over {threads} forked processes",
                                    "ids_identical_to_c_port": bool(np.array_equal(idsP, ids_c[:nP]))}
    best = max(variants, key=lambda v: variants[v]["value"])
    value = variants[best]["value"]
    log(f"[reference] L={L} " + ", ".join(f"{v} {variants[v]['value']:.0f} q/s" for v in variants))

    inserts = {"bulk_build": {"inserts_per_s": round(args.n / t_build, 1), "cores": threads, "kind": "port",
                              "graph_sha": sha, "sample": f"whole {args.n}-row build, C port"}}
    if args.stream:
        xs = _stream_rows(args)
        xa = np.concatenate([x, xs])
        gs = cref.Graph(args.n + args.stream, INDEX["R"])
        gs.adj[:args.n], gs.deg[:args.n], gs.active, gs.entry = g.adj, g.deg, g.active, g.entry
        rows2 = cref.Rows(xa, threads)
        t0 = time.perf_counter()
        cref.batch_insert(gs, rows2, args.n, args.n + args.stream, INDEX["L_build"], INDEX["alpha"], threads=threads)
        t_s = time.perf_counter() - t0
        inserts["stream_batch"] = {"inserts_per_s": round(args.stream / t_s, 1), "cores": threads, "kind": "port",
                                   "graph_sha": _graph_sha(gs.adj, gs.deg, gs.active, gs.entry),
                                   "sample": f"one {args.stream}-row batch_insert into the {args.n}-row graph, C port"}
        # numpy port (beamann's own batch_insert restated): a bounded batch into the same graph;
        # per-insert rate extrapolated from this batch size
        nb = 300
        vg = vamana.Graph(args.n + nb, INDEX["R"])
        vg.adj[:args.n], vg.deg[:args.n], vg.active, vg.entry = g.adj, g.deg, g.active, g.entry
        xv = np.ascontiguousarray(xa[:args.n + nb])
        t0 = time.perf_counter()
        vamana.batch_insert(vg, xv, args.n, args.n + nb, INDEX["R"], INDEX["L_build"], INDEX["alpha"])
        t_v = time.perf_counter() - t0
        cg = cref.Graph(args.n + nb, INDEX["R"])
        cg.adj[:args.n], cg.deg[:args.n], cg.active, cg.entry = g.adj, g.deg, g.active, g.entry
        cref.batch_insert(cg, cref.Rows(xv, threads), args.n, args.n + nb, INDEX["L_build"], INDEX["alpha"],
                          threads=threads)
        inserts["numpy_port_1proc"] = {"inserts_per_s": round(nb / t_v, 1), "cores": 1, "kind": "port",
                                       "extrapolated": True,
                                       "sample": f"one {nb}-row batch_insert into the {args.n}-row graph, numpy port",
                                       "identical_to_c_port": bool(np.array_equal(vg.adj, cg.adj))}
        log(f"[reference] inserts: " + ", ".join(f"{k} {v['inserts_per_s']:.0f}/s" for k, v in inserts.items()))

    # Under torchrun with N > 1 the GPU arm searches N shards of args.n rows (weak
    # scaling; every query visits every shard). The CPU reference on the same host
    # cores would search the N shards one after another: the shard-0 rate divided
    # by N (the shards are statistically identical; sample stated in cpu_baseline).
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        value = round(value / world, 1)
        for v in variants.values():
            v["value"] = round(v["value"] / world, 1)
            v["sample"] += f"; shard 0 timed, {world} shards -> rate / {world}"
    out = _json_base(args, world, L)
    out.update({
        "impl": "reference", "value": value, "ms_per_step": round(1e3 * args.nq / value, 2),
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": variants[best]["cores"], "kind": "port",
                         "cpu_model": _cpu_model(), "host_threads": threads,
                         "sample": f"{best}: {variants[best]['sample']}"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "variants": variants, "inserts": inserts, "recall_at_10": next(p["recall"] for p in pts if p["L"] == L),
        "sweep": pts, "setup_s": {"gen": round(t_gen, 1), "build": round(t_build, 1), "fit": round(t_fit, 1)},
        "note": "reference algorithm restated (oracle/: C port pinned to the reference's fixtures, numpy port); "
                "CPU only, no GPU, product package not imported",
    })
    line = json.dumps(out)
    print(line, flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write(line + "\n")


# ---------------------------------------------------------------------------
# B200 arm


class Clocks:
    """SM clock + throttle-reason sampling DURING the timed region (B200_PROFILING.md
    clocks line), via NVML polled every ~2 ms (nvidia-smi's 200 ms loop would miss
    a sub-second timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _poll(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _ncu_record(workload_key: str):
    """Per-launch DRAM bytes + warp instructions of the search kernel from the committed
    ncu --set full capture of the same launch (profiles/search_kernel_traffic.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "search_kernel_traffic.json")) as fh:
            t = json.load(fh)
        for rec in (t if isinstance(t, list) else [t]):  # one record per profiled workload
            if rec.get("workload") == workload_key:
                return rec
    except Exception:
        pass
    return {}


def _dist():
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # one process per GPU over NCCL; BENCH_DIST_BACKEND=gloo runs the same multi-rank
        # logic with host-staged collectives (used to test N>1 on a single-GPU box)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        dev = local % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        local = dev
    else:
        torch.cuda.set_device(0)
    return world, rank, local


def _gt_device(x_dev, q_dev, k: int):
    """Exact top-k ground truth on the GPU (jb_exact_knn: f64 scores, ties by id,
    oracle.exact_knn semantics) as (int64 ids, f64 dists) tensors. Measurement only."""
    import paper_2601_07048_b200 as jb

    i, d = jb.measure.exact_knn_device(x_dev, q_dev, k)
    return i.long(), d.double()


def _setup(args, world, rank):
    """Data, device build, RaBitQ fit, ground truth (merged across shards)."""
    import importlib

    import torch

    import paper_2601_07048_b200 as jb

    t0 = time.perf_counter()
    shard_start = rank * args.n
    x, q = _data(args, rank)
    ds = jb.VectorDataset(x)
    ds.device()
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0

    params = jb.BuildParams(degree_cap=INDEX["R"], build_beam_width=INDEX["L_build"], alpha=INDEX["alpha"],
                            max_batch=INDEX["max_batch"])
    # untimed warm-up build (first-call kernel attributes; the stream-ordered pool grows to the
    # size of a max_batch=100K insert batch, which a production process has done long before)
    jb.build(jb.VectorDataset(x[: min(args.n, 250_000)]), params)
    torch.cuda.synchronize()
    jbuild = importlib.import_module("paper_2601_07048_b200.build")  # the package re-exports build()
    jbuild.WORK[:] = 0
    t0 = time.perf_counter()
    graph = jb.build(ds, params)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    work = dict(zip(jbuild.WORK_FIELDS, (int(v) for v in jbuild.WORK)))
    t0 = time.perf_counter()
    idx = jb.rabitq_fit(ds, bits=args.bits, seed=1)
    torch.cuda.synchronize()
    t_fit = time.perf_counter() - t0
    q_dev = torch.from_numpy(q).cuda()
    gt_i, gt_d = _gt_device(ds.device().x, q_dev, 100)
    gt_i = gt_i + shard_start
    if world > 1:
        from paper_2601_07048_b200 import comm

        all_i, all_d = comm.all_gather(gt_i), comm.all_gather(gt_d)
        ci = all_i.permute(1, 0, 2).reshape(args.nq, -1)
        cd = all_d.permute(1, 0, 2).reshape(args.nq, -1)
        o = torch.argsort(ci, dim=1)
        ci, cd = torch.gather(ci, 1, o), torch.gather(cd, 1, o)
        o = torch.argsort(cd, dim=1, stable=True)[:, :100]
        gt_i, gt_d = torch.gather(ci, 1, o), torch.gather(cd, 1, o)
    log(f"gen {t_gen:.1f}s build {t_build:.1f}s ({args.n / t_build:.0f} inserts/s) fit {t_fit:.2f}s")
    return dict(jb=jb, x=x, q=q, ds=ds, graph=graph, idx=idx, q_dev=q_dev, gt_i=gt_i.cpu().numpy(),
                gt_d=gt_d.cpu().numpy().astype(np.float32), shard_start=shard_start, t_gen=t_gen, t_build=t_build,
                t_fit=t_fit, params=params, work=work)


def _insert_roofline(S, args, peak):
    """Algorithmic bytes of the bulk build (SURVEY.md §8d C4 formula, from the
    build's own work counters) over its wall time. Phase 1: hops x (4R+4)
    adjacency + evals x (4D+4) rows + 4D per new row; phase 2: one row per prune
    candidate; phase 3: each touched target's R existing rows plus one row per
    reverse triple (upper bound: ~all targets re-prune at R=32); row writes
    4R per new vertex and touched target. Repair scans are not counted."""
    w, D, R = S["work"], args.dim, INDEX["R"]
    row = 4 * D + 4
    b = (w["search_hops"] * (4 * R + 4) + w["search_evals"] * row + args.n * 4 * D
         + w["prune_candidates"] * row
         + (w["merge_targets"] * R + w["reverse_triples"]) * row
         + (args.n + w["merge_targets"]) * 4 * R)
    gbs = b / S["t_build"] / 1e9
    return {"bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 4),
            "alg_bytes": int(b), "alg_bytes_per_insert": round(b / args.n, 1), "work": w,
            "timed": "whole bulk build (wall clock, synchronized)", "traffic": None,
            "note": "alg_bytes count every evaluated neighbour's f32 row; phase 1 reads fewer where the int8 screen "
                    "(extension) runs (search_kernel_roofline.screened)"}


def _insert_search_roofline(S, args, peak):
    """The build's dominant HBM kernel alone: the phase-1 traced exact search
    (`beam_search_kernel<EXACT>`, rows staged by cp.async.bulk) over 100K dataset
    rows as queries at L_build on the built graph, CUDA events on the launching
    stream. Algorithmic bytes = hops x (4R + 4) + reference-defined evals
    (jb_count_evals: |{start} U N(expanded)|) x (4D + 4) + 4D per query."""
    import torch

    from paper_2601_07048_b200 import search as jsearch

    jb = S["jb"]
    g, ds = S["graph"], S["ds"]
    nq = min(100_000, args.n)
    q = ds.device().x[:nq].contiguous()
    L, R, D = INDEX["L_build"], INDEX["R"], args.dim
    cap = 4 * L + 64

    def timed(bound):
        out = None
        for _ in range(2):
            out = jsearch._launch(g, bound, L, None, cap)
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            out = jsearch._launch(g, bound, L, None, cap)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return out, float(np.median(ts))

    # the kernel as the build runs it (int8 screen records where they pay, extension)
    # and without the screen: every evaluated neighbour's f32 row read, i.e. the
    # algorithmic bytes below are what that kernel moves
    scr_bound = jsearch._Bound(ds, q)
    plain = jsearch._Bound(ds, q)
    plain.screen = None
    out, ms = timed(plain)
    scr_ms = timed(scr_bound)[1] if getattr(scr_bound, "screen", None) is not None else None
    _, hops, evals, _, tids, _ = out
    adj, _ = g.device()
    ev = evals.clone()
    jb._lib.check(jb._lib.lib().jb_count_evals(jb._lib.ptr(adj), R, jb._lib.ptr(tids), cap, jb._lib.ptr(hops), None,
                                              g.entry_point, None, nq, jb._lib.ptr(ev), jb._lib.stream_ptr()))
    torch.cuda.synchronize()
    h, e = hops.double().sum().item(), ev.double().sum().item()
    alg = h * (4 * R + 4) + e * (4 * D + 4) + nq * 4 * D
    gbs = alg / (ms / 1e3) / 1e9
    res = {"kernel": "beam_search_kernel<EXACT> (build phase-1 traced search, no screen)", "queries": nq, "L": L,
           "bound": "hbm", "achieved": round(gbs, 1), "peak": peak, "unit": "GB/s", "frac": round(gbs / peak, 4),
           "kernel_ms": round(ms, 3), "alg_bytes": int(alg), "hops_per_query": round(h / nq, 2),
           "evals_reference_per_query": round(e / nq, 1)}
    if scr_ms is not None:
        res["screened"] = {
            "kernel_ms": round(scr_ms, 3), "speedup": round(ms / scr_ms, 3),
            "note": "as the build runs it: int8 screen records (extension, identical results) drop neighbours "
                    "provably worse than the full beam's worst key before their f32 row is read; ncu at 1M x 128: "
                    "37.1 GB DRAM read per 100K queries vs 66.3 GB unscreened (tools/exp_screen.py), so it "
                    "reads fewer bytes than alg_bytes and is latency-bound, not HBM-bound"}
    return res


def _search_fn(S, world, L, k, est="reference"):
    """Returns f(q_dev) -> (global ids, dists) running the full per-batch path."""
    jb = S["jb"]
    sp = jb.SearchParams(beam_width=L, k=k, rerank=True, estimator=est)
    if world == 1:
        return lambda qd: jb.search_knn_batch_device(S["graph"], S["idx"], qd, sp, exact_data=S["ds"])
    from paper_2601_07048_b200 import shard

    si = shard.ShardedIndex(S["graph"], S["ds"], S["shard_start"], rabitq=S["idx"])
    return lambda qd: si.search_knn_batch_device(qd, sp, nq=qd.shape[0])


def _calibrate(S, args, world, est="reference"):
    """Smallest L of the sweep reaching the recall target (recall_at_k semantics)."""
    import torch

    pts = []
    chosen = None
    widths = (args.beam,) if args.beam else SWEEP
    for L in widths:
        ids, _ = _search_fn(S, world, L, args.k, est)(S["q_dev"])
        torch.cuda.synchronize()
        r = _recall(ids.cpu().numpy(), S["gt_i"], S["gt_d"], args.k)
        pts.append({"L": L, "recall": round(r, 4)})
        log(f"sweep [{est}] L={L} recall@{args.k}={r:.4f}")
        if r >= args.target and chosen is None:
            chosen = L
            break
    if chosen is None:
        chosen = widths[-1]
    return chosen, pts


def _alg_bytes(S, L, est="reference"):
    """SURVEY.md §8(d) algorithmic bytes of one search launch over the batch:
    per query sum_hops(4R + 4) adjacency + evals x (record bytes) + 4D query, where
    evals is the REFERENCE's count |{start} U N(expanded)| (search.py:171-269),
    computed on device from the kernel's own expansion trace. The kernel's own eval
    counter (re-evaluations after visited-table evictions included) is reported
    beside it; it does not enter `achieved`."""
    import torch

    from paper_2601_07048_b200 import search as jsearch

    jb = S["jb"]
    g, idx = S["graph"], S["idx"]
    bound = jsearch._Bound(idx, S["q_dev"], est)
    cap = 4 * L + 64
    fk, hops, evals, flags, tids, _ = jsearch._launch(g, bound, L, None, cap)
    torch.cuda.synchronize()
    nq = S["q_dev"].shape[0]
    assert int(hops.max()) <= cap, "trace capacity"
    adj, _ = g.device()
    uniq = torch.empty(nq, dtype=torch.int64, device=hops.device)
    pos = torch.arange(cap, device=hops.device)
    for lo in range(0, nq, 1000):
        hi = min(nq, lo + 1000)
        live = pos[None, :] < hops[lo:hi, None].long()
        t = torch.where(live, tids[lo:hi].long(), torch.zeros_like(tids[lo:hi], dtype=torch.long))
        nb = adj[t]                                               # [b, cap, R] (slots past hops: row 0, masked)
        nb = torch.where(live[:, :, None] & (nb >= 0), nb, torch.full_like(nb, -1)).reshape(hi - lo, -1)
        nb = torch.cat([nb, torch.full((hi - lo, 1), g.entry_point, dtype=nb.dtype, device=nb.device)], 1)
        s, _ = torch.sort(nb, dim=1)
        new = torch.ones_like(s, dtype=torch.bool)
        new[:, 1:] = s[:, 1:] != s[:, :-1]
        uniq[lo:hi] = (new & (s >= 0)).sum(1)
    D = S["x"].shape[1]
    R = g.degree_cap
    code_meta = (D * idx.bits + 7) // 8 + 8
    h = hops.double().sum().item()
    e_ref = uniq.double().sum().item()
    e_dev = evals.double().sum().item()
    search_bytes = h * (4 * R + 4) + e_ref * code_meta + nq * 4 * D
    valid = (fk != -1).sum().item()
    rerank_bytes = valid * 4 * D + nq * 4 * D
    return dict(search_bytes=search_bytes, rerank_bytes=rerank_bytes, hops=h / nq, evals_ref=e_ref / nq,
                evals_dev=e_dev / nq, lossy=int(flags.sum().item()),
                record_bytes=jb._lib.lib().jb_rabitq_record_bytes(D, idx.bits))


def _timed_steps(S, args, world, L, clocks_idx, est="reference"):
    """W warmup + K timed steps of the product's HBM-resident path (one
    search_knn_batch_device call = bind + search + rerank on two lanes, or the
    sharded path with NCCL), CUDA events on the calling stream around each step,
    L2 flushed between steps outside the events."""
    import torch
    import torch.distributed as dist

    q_dev = S["q_dev"]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    step = _search_fn(S, world, L, args.k, est)

    for i in range(args.warmup):
        flush.fill_(float(i))
        step(q_dev)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(clocks_idx) as clk:
        t0 = time.perf_counter()
        # Queue ahead: a ~20 ms device spin (before the first event) lets the host
        # enqueue every step, so the per-step events time device work only, not
        # Python launch gaps between kernels.
        torch.cuda._sleep(int(20e-3 * 1.9e9))
        torch.cuda.nvtx.range_push("timed")
        for i in range(args.steps):
            flush.fill_(float(i + 100))
            evs[i][0].record()
            step(q_dev)
            evs[i][1].record()
        torch.cuda.nvtx.range_pop()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    if world > 1:
        dist.barrier()
    step_ms = [evs[i][0].elapsed_time(evs[i][1]) for i in range(args.steps)]
    tot = float(sum(step_ms))
    if world > 1:
        from paper_2601_07048_b200 import comm

        t = torch.tensor([tot], dtype=torch.float64, device="cuda")
        tot = float(comm.all_reduce_max(t).item())
    # two lanes x (rotate GEMM + bind finish + search + rerank) (+ merge kernel when sharded)
    launches_per_step = 8 + (1 if world > 1 else 0)
    return dict(total_ms=tot, step_ms=step_ms, wall_s=wall, clocks=clk.summary(),
                launches=launches_per_step * args.steps)


def _kernel_times(S, args, L, est="reference"):
    """The dominant kernel alone (roofline): K launches of the beam-search kernel on
    one stream over the full 10K batch, CUDA events on that stream, L2 flushed between
    launches outside the events; the bind and rerank kernels timed the same way. The
    search launches sit in NVTX range "kernel_alone" so the committed ncu capture is
    of exactly this launch (profiles/profile_round.sh)."""
    import torch

    from paper_2601_07048_b200 import _lib
    from paper_2601_07048_b200 import search as jsearch

    g, idx, ds = S["graph"], S["idx"], S["ds"]
    q_dev = S["q_dev"]
    nq, k = q_dev.shape[0], args.k
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rows = ds.device()
    out_i = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    out_d = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    st = _lib.stream_ptr()
    n = max(3, args.steps)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(n + 1)]
    torch.cuda.synchronize()
    torch.cuda._sleep(int(20e-3 * 1.9e9))
    for i in range(n + 1):  # first launch is warm-up
        flush.fill_(float(i))
        ev = evs[i]
        ev[0].record()
        bound = jsearch._Bound(idx, q_dev, est)
        ev[1].record()
        if i == n:
            torch.cuda.nvtx.range_push("kernel_alone")
        fk, *_ = jsearch._launch(g, bound, L, None, 0)
        if i == n:
            torch.cuda.nvtx.range_pop()
        ev[2].record()
        _lib.check(_lib.lib().jb_rerank_topk(_lib.ptr(rows.x), rows.dims, _lib.ptr(q_dev), nq, _lib.ptr(fk), L, k,
                                             _lib.ptr(out_i), _lib.ptr(out_d), st))
        ev[3].record()
    torch.cuda.synchronize()
    ms = lambda a, b: float(np.mean([evs[i][a].elapsed_time(evs[i][b]) for i in range(1, n + 1)]))
    return dict(bind_ms=ms(0, 1), search_ms=ms(1, 2), rerank_ms=ms(2, 3))


def _e2e(S, args, world, L, est="reference"):
    """Public API with host buffers: H2D queries, search, D2H ids + dists, every step."""
    import torch
    import torch.distributed as dist

    jb = S["jb"]
    sp = jb.SearchParams(beam_width=L, k=args.k, rerank=True, estimator=est)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    # the step's inputs live in pinned host memory (the contract's H2D source)
    qh_t = torch.empty(S["q"].shape, dtype=torch.float32, pin_memory=True)
    qh = qh_t.numpy()
    qh[...] = S["q"]
    times = []
    if world == 1:
        for i in range(args.warmup + args.steps):
            flush.fill_(float(i))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ids, ds = jb.search_knn_batch(S["graph"], S["idx"], qh, sp, exact_data=S["ds"])
            times.append(time.perf_counter() - t0)
        d2h = ids.nbytes + ds.nbytes
    else:
        from paper_2601_07048_b200 import comm
        from paper_2601_07048_b200.shard import ShardedIndex

        si = ShardedIndex(S["graph"], S["ds"], S["shard_start"], rabitq=S["idx"])
        rank = dist.get_rank()
        for i in range(args.warmup + args.steps):
            flush.fill_(float(i))
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            gi, gd = si.search_knn_batch(qh if rank == 0 else None, sp)
            if rank == 0:
                ids, ds = gi.cpu().numpy(), gd.cpu().numpy()
            torch.cuda.synchronize()
            dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
            times.append(float(comm.all_reduce_max(dt).item()))
        d2h = args.nq * args.k * (8 + 8)
    tt = times[args.warmup:]
    units = args.nq * world
    return {"value": round(units * len(tt) / sum(tt), 1), "unit": "queries/s",
            "h2d_bytes_per_step": int(qh.nbytes), "d2h_bytes_per_step": int(d2h)}


def _cpu_search_baseline(S, args, L):
    """cpu_baseline leg: the C port of beamann's search path (oracle/cref.py, all host
    threads) on the GPU-built index at L with the bit-exact estimator, ids checked
    identical to the GPU's. Bounded to ~cpu_seconds of work."""
    from oracle import cref

    threads = os.cpu_count() or 1
    g, idx = S["graph"], S["idx"]
    cg = cref.Graph(g.capacity, g.degree_cap)
    cg.adj[:], cg.deg[:] = g.adjacency, g.degrees
    cg.active, cg.entry = g.active_count, g.entry_point
    quant = cref.Quantized(idx.centroid, idx.codes, idx.meta, idx.bits, idx.rotation_seed)
    t0 = time.perf_counter()
    ids, _ = _c_knn(cg, quant, S["x"], S["q"][:500], L, args.k, threads)
    per_q = (time.perf_counter() - t0) / 500
    n = int(min(args.nq, max(500, args.cpu_seconds / per_q)))
    t0 = time.perf_counter()
    ids, _ = _c_knn(cg, quant, S["x"], S["q"][:n], L, args.k, threads)
    el = time.perf_counter() - t0
    gpu_ids, _ = _search_fn(S, 1, L, args.k, "reference")(S["q_dev"][:n])
    return {"value": round(n / el, 1), "unit": "queries/s", "cores": threads, "kind": "port",
            "cpu_model": _cpu_model(),
            "sample": f"first {n} of the {args.nq} queries, C port of the reference search path (bind, lockstep "
                      f"RaBitQ search, exact rerank) at L={L}, {threads} threads",
            "ids_identical_to_gpu": bool(np.array_equal(ids, gpu_ids.cpu().numpy()))}, cg


def _stream_insert(S, args, cg):
    """One streaming batch_insert of `--stream-rows` new rows into the 1M graph: on the GPU
    (public API) and with the C port of the reference (all host threads) on the same
    graph; the resulting graphs must be identical."""
    import torch

    from oracle import cref

    jb = S["jb"]
    n, s, R = args.n, args.stream, INDEX["R"]
    xs = _stream_rows(args)
    xa = np.concatenate([S["x"], xs])
    ds2 = jb.VectorDataset(xa)
    ds2.device()
    g2 = jb.GraphIndex(n + s, R)
    adj = np.full((n + s, R), -1, dtype=np.int32)
    deg = np.zeros(n + s, dtype=np.int32)
    adj[:n], deg[:n] = cg.adj, cg.deg
    g2.adjacency, g2.degrees = adj, deg
    g2.active_count, g2.entry_point = cg.active, cg.entry
    g2.device()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    jb.batch_insert(g2, ds2, range(n, n + s), S["params"])
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    gpu_sha = _graph_sha(g2.adjacency, g2.degrees, g2.active_count, g2.entry_point)
    threads = os.cpu_count() or 1
    gs = cref.Graph(n + s, R)
    gs.adj[:n], gs.deg[:n], gs.active, gs.entry = cg.adj, cg.deg, cg.active, cg.entry
    rows2 = cref.Rows(xa, threads)
    t0 = time.perf_counter()
    cref.batch_insert(gs, rows2, n, n + s, INDEX["L_build"], INDEX["alpha"], threads=threads)
    t_cpu = time.perf_counter() - t0
    same = bool(np.array_equal(gs.adj, g2.adjacency) and gs.entry == g2.entry_point)
    del ds2, g2
    return {"rows": s, "base_rows": n, "inserts_per_s": round(s / t_gpu, 1), "graph_sha": gpu_sha,
            "timed": "one batch_insert call (wall clock, synchronized)",
            "cpu_baseline": {"inserts_per_s": round(s / t_cpu, 1), "cores": threads, "kind": "port",
                             "sample": f"the same {s}-row batch_insert, C port of the reference, {threads} threads",
                             "identical_graph": same}}


def gpu_arm(args):
    import torch

    world, rank, local = _dist()
    if args.hash_slots:
        from paper_2601_07048_b200 import search as _js

        _js.TUNING["hash_slots"] = args.hash_slots
    S = _setup(args, world, rank)
    ests = {"reference": ["reference"], "popcount": ["popcount"], "auto": ["reference", "popcount"]}[args.estimator]
    cal = {e: _calibrate(S, args, world, e) for e in ests}

    runs = {}
    for e in ests:
        Le = cal[e][0]
        ab = _alg_bytes(S, Le, e)
        T = _timed_steps(S, args, world, Le, local, e)
        T.update(_kernel_times(S, args, Le, e))
        runs[e] = (Le, ab, T, args.nq * world * args.steps / (T["total_ms"] / 1e3))
        log(f"[{e}] L={Le} value={runs[e][3]:.0f} queries/s, search kernel {T['search_ms']:.3f} ms, "
            f"evals/query ref {ab['evals_ref']:.0f} device {ab['evals_dev']:.0f}")
    est = max(runs, key=lambda e: runs[e][3])
    L, ab, T, value = runs[est]
    sweep_pts = cal[est][1]
    e2e = _e2e(S, args, world, L, est)
    peak, peak_kind = _peaks()
    search_s = T["search_ms"] / 1e3
    achieved = ab["search_bytes"] / search_s / 1e9
    out = _json_base(args, world, L)
    wl_key = out["config"]["workload"] + f" L={L} {est}"
    ncu = _ncu_record(wl_key)
    clk = T["clocks"].get("sm_mhz") or 1965.0
    issue = None
    if ncu.get("warp_inst_per_launch"):
        # issue roofline: 4 warp-instruction issues per clock per SM x 148 SMs
        ipl = ncu["warp_inst_per_launch"]
        rate = ipl / search_s
        issue = {"warp_inst_per_launch": int(ipl), "achieved_ginst_s": round(rate / 1e9, 1),
                 "peak_ginst_s": round(4 * 148 * clk * 1e6 / 1e9, 1),
                 "frac": round(rate / (4 * 148 * clk * 1e6), 4), "source": ncu.get("source")}
    out.update({
        "impl": "b200", "estimator": est,
        "value": round(value, 1),
        "ms_per_step": round(T["total_ms"] / args.steps, 3),
        "e2e": e2e,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "traffic": ncu.get("dram_bytes_per_launch"),
                     "traffic_source": ncu.get("source"),
                     "kernel": f"beam_search_kernel<{'RABITQ_FAST' if est == 'popcount' else 'RABITQ'},{args.bits}>",
                     "alg_bytes_per_launch": int(ab["search_bytes"]), "kernel_ms": round(search_s * 1e3, 4),
                     "evals_counted": "reference |{start} U N(expanded)| per query (device re-evaluations excluded)",
                     "issue": issue},
        "gpu_launches": T["launches"],
        "clocks": T["clocks"],
        "recall_at_10": next(p["recall"] for p in sweep_pts if p["L"] == L),
        "sweep": sweep_pts,
        "per_query": {"hops": round(ab["hops"], 2), "evals_reference": round(ab["evals_ref"], 1),
                      "evals_device": round(ab["evals_dev"], 1),
                      "reevaluated_frac": round(ab["evals_dev"] / ab["evals_ref"] - 1.0, 4),
                      "lossy_queries": ab["lossy"]},
        "kernel_ms": {"bind": round(T["bind_ms"], 4), "search": round(search_s * 1e3, 4),
                      "rerank": round(T["rerank_ms"], 4),
                      "note": "each kernel alone on one stream over the full batch (the step runs two lanes)"},
        "build": {"inserts_per_s": round(args.n / S["t_build"], 1), "build_s": round(S["t_build"], 2),
                  "rabitq_fit_s": round(S["t_fit"], 3), "gen_s": round(S["t_gen"], 2),
                  "graph_sha": _graph_sha(S["graph"].adjacency, S["graph"].degrees, S["graph"].active_count,
                                          S["graph"].entry_point),
                  "roofline": _insert_roofline(S, args, peak),
                  "search_kernel_roofline": _insert_search_roofline(S, args, peak)},
        "estimators": {e: {"L": runs[e][0], "value": round(runs[e][3], 1),
                           "recall_at_10": next(p["recall"] for p in cal[e][1] if p["L"] == runs[e][0]),
                           "search_kernel_ms": round(runs[e][2]["search_ms"], 4),
                           "bit_exact": e == "reference"} for e in runs},
    })
    if rank == 0 and world == 1 and not args.no_cpu:
        Lr = cal["reference"][0] if "reference" in cal else L
        cb, cg = _cpu_search_baseline(S, args, Lr)
        out["cpu_baseline"] = cb
        if args.stream:
            out["build"]["stream_batch"] = _stream_insert(S, args, cg)
    if rank == 0:
        line = json.dumps(out)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(line + "\n")
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main():
    args = _args()
    if args.impl == "reference":
        reference_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
