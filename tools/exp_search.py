"""Search-kernel experiments on the bench index (not part of the product or the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(40_000, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qd = torch.from_numpy(q).cuda()

def t_search(nq, L, est, hs=0, reps=5):
    js.TUNING["hash_slots"] = hs
    b = js._Bound(idx, qd[:nq].contiguous(), est)
    for _ in range(2):
        js._launch(g, b, L, None, 0)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, e in ev:
        a.record(); js._launch(g, b, L, None, 0); e.record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(e) for a, e in ev]))

for est in ("reference", "popcount"):
    for nq in (2368, 4736, 10000, 20000, 40000):
        ms = t_search(nq, 128, est)
        print(f"{est:9s} nq={nq:6d} L=128 {ms:7.3f} ms  {nq / ms * 1e3 / 1e6:6.2f} MQPS  {ms / nq * 1e6:7.1f} ns/query", flush=True)
for hs in (512, 1024, 2048):
    print("hash", hs, f"{t_search(10000, 128, 'popcount', hs):.3f} ms", flush=True)
