"""Interleaved A/B of env-selected build variants in one process (dev tool).

    python tools/exp_build_ab.py "JB_CLOSED_PASS=0" "JB_CLOSED_PASS=1,JB_CLOSED_EXTRA=2" ...
Each variant is a comma list of VAR=VALUE read per batch by the library; 1M x 128
bulk builds, variants interleaved over reps; prints min / median per variant and
whether every variant's graph hash matches the first."""
import hashlib
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

n = int(os.environ.get("JB_AB_N", "1000000"))
d = int(os.environ.get("JB_AB_D", "128"))
reps = int(os.environ.get("JB_AB_REPS", "4"))
variants = [dict(kv.split("=", 1) for kv in v.split(",") if kv) for v in sys.argv[1:]] or [{}]
x = jb.gen_lowrank(n, d, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
ds.device()
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000)
jb.build(jb.VectorDataset(x[:250_000]), p)
times = [[] for _ in variants]
hashes = [None for _ in variants]
for r in range(reps):
    for i, v in enumerate(variants):
        old = {k: os.environ.get(k) for k in v}
        os.environ.update(v)
        torch.cuda.synchronize()
        t = time.perf_counter()
        g = jb.build(ds, p)
        torch.cuda.synchronize()
        times[i].append(time.perf_counter() - t)
        for k, o in old.items():
            if o is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = o
        if r == 0:
            hashes[i] = hashlib.sha256(g.host_adjacency()[: g.active_count].tobytes()).hexdigest()[:16]
for i, v in enumerate(variants):
    print(f"{v}: min {min(times[i]):.3f} s median {statistics.median(times[i]):.3f} s "
          f"({n / min(times[i]):.0f} inserts/s) graph {hashes[i]} same={hashes[i] == hashes[0]}")
