"""Int8 screen of the exact search (dev tool): phase-1-shaped traced search of 100K
dataset rows at L=64 on a 1M x 128 graph, with and without screen records
(interleaved CUDA-event timings; identical outputs asserted)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

n = int(os.environ.get("JB_EXP_N", "1000000"))
d = int(os.environ.get("JB_EXP_D", "128"))
x = jb.gen_lowrank(n, d, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
q = ds.device().x[n - 100_000:].contiguous()
os.environ.setdefault("JB_SCREEN_FORCE", "1")  # measure the screen even where the library's policy skips it
on = js._Bound(ds, q)
off = js._Bound(ds, q)
off.screen = None
cap = 4 * 64 + 512
res = {}
ts = {"off": [], "on": []}
for rep in range(5):
    for name, b in (("off", off), ("on", on)):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = js._launch(g, b, 64, None, cap)
        e1.record()
        torch.cuda.synchronize()
        ts[name].append(e0.elapsed_time(e1))
        res[name] = [t.cpu() for t in out[:5]]
for i in range(5):
    assert torch.equal(res["off"][i], res["on"][i]), i
if os.environ.get("JB_EXP_NCU"):  # one launch each inside the profiler range
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    js._launch(g, off, 64, None, cap)
    js._launch(g, on, 64, None, cap)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
for k, v in ts.items():
    print(f"screen {k}: median {np.median(v[1:]):.3f} ms per 100K queries")
