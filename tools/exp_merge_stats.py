"""Merge statistics of the search kernel (dev tool). Needs a library built with
JB_NVCC_EXTRA=-DJB_MERGE_STATS (rebuild in place: touch csrc/search.cu first)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import _lib
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(10_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qd = torch.from_numpy(q).cuda()
buf = (C.c_ulonglong * 66)()
lib = _lib.lib()
lib.jb_debug_merge_stats(buf)
for est in ("popcount",):
    b = js._Bound(idx, qd, est)
    js._launch(g, b, 128, None, 0)
    torch.cuda.synchronize()
    lib.jb_debug_merge_stats(buf)
    h = np.array(buf[:33], dtype=np.float64)
    e = np.array(buf[33:66], dtype=np.float64)
    print(est, "merges", int(h.sum()), "per query", h.sum() / 10000)
    print("after filter: fraction with 0..32 candidates", np.round(h / h.sum(), 3).tolist())
    print("mean after filter", (h * np.arange(33)).sum() / h.sum(), " mean evaluated", (e * np.arange(33)).sum() / e.sum())
