"""CPU simulation (dev tool): share of phase-1 evaluations a rigorous lower bound
would drop once the beam is full, for bf16 / int8 centred rows and a half-row
partial sum, on the C port's 200K x 128 graph at L=64 (150 queries)."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import cref
import paper_2601_07048_b200 as jb
n, D = 200_000, 128
x = jb.gen_lowrank(n, D, seed=1, d_int=16, noise=0.05, basis_seed=0)
t = time.time()
g = cref.build(x, 32, 64, 1.2)
print('build', time.time() - t, file=sys.stderr)
adj = g.adj; deg = g.deg; entry = g.entry
c = x.mean(0)
xc = (x - c).astype(np.float32)
import torch
xb = torch.from_numpy(xc).to(torch.bfloat16).float().numpy()
eps = np.sqrt(((xb.astype(np.float64) - xc) ** 2).sum(1)) * (1 + 1e-6)
nx = (x.astype(np.float64) ** 2).sum(1)
rng = np.random.default_rng(0)
qs = x[rng.choice(n, 150, replace=False)] + rng.standard_normal((150, D)).astype(np.float32) * 0.02
L = 64
sc = np.abs(xc).max(1) / 127.0
x8 = (np.rint(xc / sc[:, None]).clip(-127, 127) * sc[:, None]).astype(np.float64)
eps8 = np.sqrt(((x8 - xc) ** 2).sum(1)) * (1 + 1e-6)
drop8 = 0
drop88 = 0
tot = 0; full = 0; drop_tri = 0; drop_half = 0; drop_cs = 0
xbu = torch.from_numpy(x).to(torch.bfloat16).float().numpy()
for q in qs:
    d_all = lambda ids: ((x[ids].astype(np.float64) - q) ** 2).sum(1)
    qc = q - c
    nq = float((q.astype(np.float64) ** 2).sum())
    beam = [(float(d_all([entry])[0]), entry)]
    seen = {entry}; expanded = set()
    while True:
        cand = [b for b in beam if b[1] not in expanded]
        if not cand: break
        u = cand[0][1]; expanded.add(u)
        nb = [int(v) for v in adj[u][:deg[u]] if v not in seen]
        if not nb: continue
        for v in nb: seen.add(v)
        nb = np.array(nb)
        d = d_all(nb)
        tot += len(nb)
        if len(beam) == L:
            worst = beam[-1][0]
            full += len(nb)
            # triangle bound on centered bf16 rows
            r = np.sqrt(((xb[nb].astype(np.float64) - qc) ** 2).sum(1)) - eps[nb]
            lb = np.where(r > 0, r * r, 0) * (1 - 1e-4)
            drop_tri += int((lb > worst).sum())
            r8 = np.sqrt(((x8[nb] - qc) ** 2).sum(1)) - eps8[nb]
            sq = np.abs(qc).max() / 127.0
            q8 = np.rint(qc / sq).clip(-127, 127) * sq
            eq = np.sqrt(((q8 - qc) ** 2).sum()) * (1 + 1e-6)
            r88 = np.sqrt(((x8[nb] - q8) ** 2).sum(1)) - eps8[nb] - eq
            drop88 += int((np.where(r88 > 0, r88 * r88, 0) * (1 - 1e-4) > worst).sum())
            drop8 += int((np.where(r8 > 0, r8 * r8, 0) * (1 - 1e-4) > worst).sum())
            # partial (first half) squared distance
            ph = ((x[nb, :64].astype(np.float64) - q[:64]) ** 2).sum(1) * (1 - 1e-4)
            drop_half += int((ph > worst).sum())
            # uncentered bf16 cauchy-schwarz
            s = (xbu[nb].astype(np.float64) @ q.astype(np.float64))
            lbc = nx[nb] + nq - 2 * s - 2 * 2 ** -9 * np.sqrt(nx[nb] * nq) * 1.01
            drop_cs += int((lbc > worst).sum())
        beam = sorted(beam + list(zip(d.tolist(), nb.tolist())))[:L]
print(f"evals {tot}, with full beam {full} ({full/tot:.2f}); screened out: triangle-bf16-centered {drop_tri/tot:.3f}, half-row {drop_half/tot:.3f}, cs-bf16 {drop_cs/tot:.3f} int8-centered {drop8/tot:.3f} int8xint8 {drop88/tot:.3f}")
