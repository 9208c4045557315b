"""Build time with beamann's default BuildParams (R=64, L=128) at 200K x 128 and 100K x 960 (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb

for n, d in ((200_000, 128), (100_000, 960)):
    x = jb.gen_lowrank(n, d, seed=1, d_int=16, noise=0.05, basis_seed=0)
    ds = jb.VectorDataset(x)
    p = jb.BuildParams()  # defaults: degree_cap=64, build_beam_width=128
    jb.build(jb.VectorDataset(x[: n // 4]), p)
    torch.cuda.synchronize()
    t = time.perf_counter()
    jb.build(ds, p)
    torch.cuda.synchronize()
    print(f"default params {n}x{d}: {time.perf_counter() - t:.3f} s", flush=True)
