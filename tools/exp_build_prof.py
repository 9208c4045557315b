"""Bulk-build phase profile (dev tool): JB_PROFILE=1 per-batch phase timings."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb
import importlib; jbuild = importlib.import_module("paper_2601_07048_b200.build")

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 128
x = jb.gen_lowrank(n, d, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
ds.device()
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000)
jb.build(jb.VectorDataset(x[:250_000]), p)  # warm-up (pool grown to 100K batches)
torch.cuda.synchronize()
os.environ["JB_PROFILE"] = os.environ.get("JB_EXP_PROFILE", "0")
for rep in range(int(os.environ.get("JB_EXP_REPS", "1"))):
    jbuild.WORK[:] = 0
    t = time.perf_counter()
    g = jb.build(ds, p)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    print(f"build {n}x{d}: {el:.3f} s, {n / el:.0f} inserts/s; work {dict(zip(jbuild.WORK_FIELDS, jbuild.WORK.tolist()))}",
          file=sys.stderr)
