"""ORACLE — test infrastructure only. RaBitQ restated in numpy.

  * seeded rotation: PCG64 normals -> QR -> column sign fix     rabitq.py:59-68
  * code packing, m-bit codes LSB-first                        rabitq.py:78-101
  * fit (centroid, per-4096-row blocks, metadata)              rabitq.py:257-301
  * bind (rotated query, query_add, query_sumq)                rabitq.py:170-181
  * estimator est = qadd + add + rescale*(<u,q> - sumq), >= 0  rabitq.py:235-244
"""

from __future__ import annotations

import functools

import numpy as np

BLOCK = 4096  # rabitq.py:56


@functools.lru_cache(maxsize=8)
def rotation(seed: int, dims: int) -> np.ndarray:
    g = np.random.default_rng(seed)
    q, r = np.linalg.qr(g.standard_normal((dims, dims)))
    return q * np.where(np.diag(r) >= 0, 1.0, -1.0)


def pack(u: np.ndarray, bits: int) -> np.ndarray:
    n, d = u.shape
    per = 8 // bits
    nbytes = (d * bits + 7) // 8
    padded = np.zeros((n, nbytes * per), dtype=np.uint16)
    padded[:, :d] = u
    lanes = padded.reshape(n, nbytes, per) << (bits * np.arange(per, dtype=np.uint16))
    return lanes.sum(axis=2, dtype=np.uint16).astype(np.uint8)


def unpack(codes: np.ndarray, bits: int, dims: int) -> np.ndarray:
    per = 8 // bits
    sh = (bits * np.arange(per)).astype(np.uint8)
    vals = (codes[..., :, None] >> sh) & np.uint8((1 << bits) - 1)
    return vals.reshape(*codes.shape[:-1], -1)[..., :dims]


def fit(x: np.ndarray, bits: int, seed: int):
    """Returns (centroid f32[D], codes u8[n, cb], meta f32[n, 2])."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, dims = x.shape
    centroid = x.astype(np.float64).mean(axis=0).astype(np.float32)
    rot = rotation(seed, dims)
    levels = 2 ** bits - 1
    mid = levels / 2.0
    codes = np.empty((n, (dims * bits + 7) // 8), dtype=np.uint8)
    meta = np.empty((n, 2), dtype=np.float32)
    for lo in range(0, n, BLOCK):
        hi = min(n, lo + BLOCK)
        res = (x[lo:hi] - centroid).astype(np.float64)
        norm = np.sqrt(np.einsum("bd,bd->b", res, res))
        nz = norm > 0.0
        o = (res / np.where(nz, norm, 1.0)[:, None]) @ rot.T
        delta = 2.0 * np.abs(o).max(axis=1) / levels
        sd = np.where(delta > 0.0, delta, 1.0)
        u = np.clip(np.round(o / sd[:, None] + mid), 0, levels).astype(np.uint8)
        u[~nz] = 1 << (bits - 1)
        ip = np.einsum("bd,bd->b", o, sd[:, None] * (u.astype(np.float64) - mid))
        good = nz & (ip > 1e-12)
        meta[lo:hi, 0] = np.where(nz, norm * norm, 0.0).astype(np.float32)
        meta[lo:hi, 1] = np.where(good, -2.0 * norm * delta / np.where(good, ip, 1.0), 0.0).astype(np.float32)
        codes[lo:hi] = pack(u, bits)
    return centroid, codes, meta


def bind(queries: np.ndarray, centroid: np.ndarray, bits: int, seed: int):
    q = np.atleast_2d(np.asarray(queries, dtype=np.float32))
    qc = q - centroid[None, :]
    rotated = (qc.astype(np.float64) @ rotation(seed, q.shape[1]).T).astype(np.float32)
    qadd = np.einsum("qd,qd->q", qc, qc)
    sumq = (rotated.sum(axis=1) * np.float32((2 ** bits - 1) / 2.0)).astype(np.float32)
    return rotated, qadd, sumq


class QuantSource:
    """Bound estimator with the call shape of ExactSource (rabitq.py:225-244)."""

    def __init__(self, codes, meta, bits, dims, rotated, qadd, sumq):
        self.codes, self.meta, self.bits, self.dims = codes, meta, bits, dims
        self.rotated, self.qadd, self.sumq = rotated, qadd, sumq

    def __call__(self, qrows, ids):
        u = unpack(self.codes[ids], self.bits, self.dims).astype(np.float32)
        dots = np.einsum("md,md->m", u, self.rotated[qrows])
        est = self.qadd[qrows] + self.meta[ids, 0] + self.meta[ids, 1] * (dots - self.sumq[qrows])
        return np.maximum(est, np.float32(0))
