"""One search launch on the bench index inside an NVTX range "prof/" (dev tool, for ncu).

    ncu --nvtx --nvtx-include "prof/" ... python tools/exp_prof_search.py [L] [estimator]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2601_07048_b200 as jb
from paper_2601_07048_b200 import search as js

L = int(sys.argv[1]) if len(sys.argv) > 1 else 128
est = sys.argv[2] if len(sys.argv) > 2 else "popcount"
nq = int(os.environ.get("JB_EXP_NQ", "5000"))
x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
q = jb.gen_lowrank(nq, 128, seed=1_000_003, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
idx = jb.rabitq_fit(ds, bits=1, seed=1)
qd = torch.from_numpy(q).cuda()
b = js._Bound(idx, qd, est)
js._launch(g, b, L, None, 0)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("prof")
js._launch(g, b, L, None, 0)
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("done")
