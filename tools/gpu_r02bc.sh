python - <<'PY' 2>&1 | grep -E "^\[jb\] batch \[|total" | tail -3
import os, time
os.environ["JB_PROFILE"] = "1"
import torch, paper_2601_07048_b200 as jb
x = jb.gen_lowrank(1_000_000, 128, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
t0 = time.perf_counter()
g = jb.build(ds, jb.BuildParams())
torch.cuda.synchronize()
print("total", time.perf_counter() - t0)
PY
timeout 900 python tools/exp_defaults_1m.py 2>&1 | tail -8
