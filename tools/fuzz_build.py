"""Randomized build parity vs the oracle over R / D / alpha / batch / option combinations (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import paper_2601_07048_b200 as jb
from conftest import gaussian, lowrank
from oracle import vamana

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
cases = int(sys.argv[2]) if len(sys.argv) > 2 else 20
bad = 0
for c in range(cases):
    n = int(rng.integers(200, int(os.environ.get("FUZZ_NMAX", "2500"))))
    D = int(rng.choice([int(v) for v in os.environ.get("FUZZ_DIMS", "3,8,20,33,64,96,128").split(",")]))
    R = int(rng.choice([int(v) for v in os.environ.get("FUZZ_R", "4,9,24,33,40,64,100").split(",")]))
    L = int(max(R, rng.choice([8, 16, 48, 100, 160])))
    alpha = float(rng.choice([1.0, 1.1, 1.2, 1.5]))
    mb = int(rng.choice([50, 300, 1000, 100_000]))
    tp = bool(rng.random() < 0.25)
    x = gaussian(n, D, c) if rng.random() < 0.5 else lowrank(n, D, min(D, 8), 0.05, c)
    if os.environ.get("FUZZ_KIND") == "u8":  # u8 rows (integer distances)
        x = np.clip(np.rint((x - x.min()) / (x.max() - x.min()) * 255.0), 0, 255).astype(np.uint8)
    t = time.time()
    oerr = None
    try:
        og = vamana.build(x, R=R, L=L, alpha=alpha, max_batch=mb, two_pass=tp)
    except RuntimeError as e:  # the reference's own repair failure (no donor)
        oerr = str(e)
    to = time.time() - t
    p = jb.BuildParams(degree_cap=R, build_beam_width=L, alpha=alpha, max_batch=mb, two_pass=tp)
    if oerr is not None:
        try:
            jb.build(jb.VectorDataset(x), p)
            ok = False
        except RuntimeError as e:
            ok = str(e) == oerr
    else:
        g = jb.build(jb.VectorDataset(x), p)
        ok = (g.entry_point == og.entry and np.array_equal(g.degrees[:n], og.deg[:n])
              and np.array_equal(g.adjacency[:n], og.adj[:n]))
    ap = ra = False
    bad += not ok
    print(f"case {c}: n={n} D={D} R={R} L={L} a={alpha} mb={mb} ap={ap} ra={ra} tp={tp}: "
          f"{'OK' if ok else 'MISMATCH'}{' (both raise: ' + oerr + ')' if oerr else ''} (oracle {to:.1f}s)", flush=True)
print("mismatches", bad)
