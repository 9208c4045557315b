"""Owner-merge (phase 3) candidate statistics of a 1M x 128 build (dev tool; needs
JB_NVCC_EXTRA=-DJB_OWNER_STATS)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import _lib

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
buf = (C.c_ulonglong * 16)()
lib = _lib.lib()
lib.jb_debug_owner_stats(buf)
jb.build(jb.VectorDataset(x), jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
lib.jb_debug_owner_stats(buf)
v = np.array(buf[:], dtype=np.int64)
print(f"pruned targets {v[0]}, mean candidates {v[1] / max(v[0], 1):.1f}; unstaged {v[2]} "
      f"({100 * v[2] / max(v[0], 1):.2f}%), their candidates {v[3]} ({100 * v[3] / max(v[1], 1):.1f}% of all)")
print("histogram of n by 16s:", v[4:16].tolist())
