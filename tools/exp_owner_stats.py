"""Owner-merge statistics of one 100K batch (dev tool): needs a library built with
JB_NVCC_EXTRA=-DJB_OWNER_STATS (touch csrc/build.cu first).
    python tools/exp_owner_stats.py N"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import _lib

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
x = jb.gen_lowrank(n + 100_000, 96, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
p = jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2, max_batch=100_000)
g = jb.GraphIndex(capacity=n + 100_000, degree_cap=32)
jb.insert_stream(g, ds, range(0, n), p)
lib = _lib.lib()
buf = (C.c_ulonglong * 16)()
lib.jb_debug_owner_stats(buf)
jb.insert_stream(g, ds, range(n, n + 100_000), p)
torch.cuda.synchronize()
lib.jb_debug_owner_stats(buf)
s = np.array(buf[:], dtype=np.int64)
print("pruned targets", s[0], "candidates", s[1], "mean n", s[1] / max(1, s[0]))
print("unstaged targets", s[2], "their candidates", s[3])
print("histogram of n (bins of 16):", s[4:].tolist())
print("graph degree mean", float(np.asarray(g.degrees[: g.active_count]).mean()))
