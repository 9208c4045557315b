"""Synthetic workload generators shared by both arms of bench.py (numpy only).

Neither arm's data depends on the product package: the reference arm
(`bench.py --impl reference`) must run without importing
paper_2601_07048_b200 or touching the GPU, and both arms must see identical
rows, so the generator lives here. `lowrank` is byte-identical to the
package's `gen_lowrank` (SURVEY.md Appendix B recipe with a shared basis).
"""

from __future__ import annotations

import numpy as np


def lowrank(count: int, dims: int, seed: int, d_int: int = 16, noise: float = 0.05,
            basis_seed: int | None = 0) -> np.ndarray:
    """Low-intrinsic-dimension f32 rows: z @ A + noise * N(0, 1), A from default_rng(basis_seed)
    (shared by shards and held-out queries), z and the noise from default_rng(seed)."""
    if basis_seed is None:
        g = np.random.default_rng(seed)
        a = g.standard_normal((d_int, dims)) / np.sqrt(d_int)
    else:
        a = np.random.default_rng(basis_seed).standard_normal((d_int, dims)) / np.sqrt(d_int)
        g = np.random.default_rng(seed)
    out = np.empty((count, dims), dtype=np.float32)
    z_all = g.standard_normal((count, d_int))
    step = 262_144
    for lo in range(0, count, step):  # chunked noise draws continue the same stream
        hi = min(count, lo + step)
        out[lo:hi] = z_all[lo:hi] @ a + noise * g.standard_normal((hi - lo, dims))
    return out


def gaussian(count: int, dims: int, seed: int) -> np.ndarray:
    """The reference's gen_synthetic(count, dims, seed) 'gaussian' rows (core.py:209-233)."""
    return np.random.default_rng(seed).standard_normal((count, dims)).astype(np.float32)
