"""Search-kernel tail study (dev tool): hop-count spread and batch-size scaling on the bench index."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(40_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qd = torch.from_numpy(q).cuda()


def t_launch(b, L, reps=7):
    for _ in range(2):
        js._launch(g, b, L, None, 0)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, e in ev:
        a.record()
        js._launch(g, b, L, None, 0)
        e.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(e) for a, e in ev]))


b = js._Bound(idx, qd[:10_000], "popcount")
_, hops, evals, *_ = js._launch(g, b, 128, None, 0)
h = hops.cpu().numpy()
print(f"hops: mean {h.mean():.1f} sd {h.std():.1f} p50 {np.percentile(h, 50):.0f} p99 {np.percentile(h, 99):.0f} max {h.max()}")
qa = b.qadd.cpu().numpy()
print(f"corr(hops, |q-c|^2) = {np.corrcoef(h, qa)[0, 1]:.3f}")
for nq in (5_000, 10_000, 20_000, 40_000):
    bb = js._Bound(idx, qd[:nq].contiguous(), "popcount")
    ms = t_launch(bb, 128)
    print(f"nq={nq}: {ms:.3f} ms  {nq / ms / 1e3:.2f} MQPS", flush=True)
# longest-first order (by the previous run's hops) for 10K
order = torch.from_numpy(np.argsort(-h, kind="stable")).cuda()
bo = js._Bound(idx, qd[:10_000][order].contiguous(), "popcount")
print(f"10K sorted by hops desc: {t_launch(bo, 128):.3f} ms")
