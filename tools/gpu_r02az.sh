python - <<'PY' 2>&1 | grep -E "^\[jb\] batch|total" | tail -4
import os, time
os.environ["JB_PROFILE"] = "1"
import torch, paper_2601_07048_b200 as jb
x = jb.gen_lowrank(1_000_000, 960, seed=1, d_int=16, noise=0.05, basis_seed=0)
ds = jb.VectorDataset(x)
t0 = time.perf_counter()
g = jb.build(ds, jb.BuildParams(degree_cap=32, build_beam_width=64, alpha=1.2))
torch.cuda.synchronize()
print("total", time.perf_counter() - t0)
PY
