"""Vector datasets and synthetic generators (mirror of the reference's core.py).

`VectorDataset` keeps the reference contract (core.py:55-107): an immutable,
finite, C-contiguous (count, dims) f32 (or u8) array. The B200 path adds a
lazily created device mirror — the f32 rows in HBM plus their A1-order
squared norms — that every kernel reads; it is built once per dataset.
"""

from __future__ import annotations

import enum
import threading
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib

__all__ = ["ElementKind", "DistanceKind", "VectorDataset", "AugmentedDataset", "mips_augment", "sq_l2", "dot",
           "gen_synthetic", "gen_lowrank", "row_sq_norms"]


class ElementKind(enum.Enum):
    U8 = "u8"
    F32 = "f32"

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.uint8) if self is ElementKind.U8 else np.dtype(np.float32)

    @property
    def itemsize(self) -> int:
        return self.dtype.itemsize


class DistanceKind(enum.Enum):
    SQUARED_EUCLIDEAN = "sq_l2"
    INNER_PRODUCT = "ip"


@dataclass
class DeviceRows:
    """HBM mirror of a dataset: rows [n, D] (f32, or u8) and their squared norms
    [n] (f32 in A1 order, or exact u32 integers held in an int32 tensor)."""
    x: object
    norms: object
    count: int
    dims: int
    kind: ElementKind = ElementKind.F32


class VectorDataset:
    """Immutable row-major store of `count` vectors of `dims` elements (core.py:55-107)."""

    def __init__(self, data: np.ndarray):
        arr = np.asarray(data)
        if arr.ndim != 2:
            raise ValueError(f"dataset array must be 2-D, got shape {arr.shape}")
        if arr.shape[1] < 1:
            raise ValueError("dims must be >= 1")
        if arr.dtype == np.uint8:
            self._kind = ElementKind.U8
        elif arr.dtype == np.float32:
            self._kind = ElementKind.F32
        else:
            raise ValueError(f"unsupported element dtype {arr.dtype}; use uint8 or float32")
        arr = np.ascontiguousarray(arr)
        if self._kind is ElementKind.F32 and arr.size and not np.isfinite(arr).all():
            raise ValueError("dataset contains non-finite values")
        arr.setflags(write=False)
        self._data = arr
        self._dev: DeviceRows | None = None
        self._dev_lock = threading.Lock()

    @classmethod
    def from_device(cls, x_dev, host: np.ndarray | None = None) -> "VectorDataset":
        """Wrap rows already resident in HBM (torch f32 [n, D] CUDA tensor).

        The host copy is materialized lazily only if a host-side caller asks
        for `.data`; the kernels read the device rows directly.
        """
        torch = _lib.require_cuda()
        if x_dev.dtype != torch.float32 or x_dev.dim() != 2 or not x_dev.is_cuda:
            raise ValueError("from_device expects a CUDA float32 (n, D) tensor")
        obj = cls.__new__(cls)
        obj._kind = ElementKind.F32
        obj._data = host
        obj._dev_lock = threading.Lock()
        x_dev = x_dev.contiguous()
        norms = torch.empty(x_dev.shape[0], dtype=torch.float32, device=x_dev.device)
        _lib.check(_lib.lib().jb_row_sq_norms(_lib.ptr(x_dev), x_dev.shape[0], x_dev.shape[1],
                                             _lib.ptr(norms), _lib.stream_ptr()))
        obj._dev = DeviceRows(x_dev, norms, x_dev.shape[0], x_dev.shape[1])
        obj._shape = tuple(x_dev.shape)
        return obj

    @property
    def data(self) -> np.ndarray:
        if self._data is None:
            arr = self._dev.x.cpu().numpy()
            arr.setflags(write=False)
            self._data = arr
        return self._data

    @property
    def element_kind(self) -> ElementKind:
        return self._kind

    @property
    def dims(self) -> int:
        return self._data.shape[1] if self._data is not None else self._dev.dims

    @property
    def count(self) -> int:
        return self._data.shape[0] if self._data is not None else self._dev.count

    def row(self, i: int) -> np.ndarray:
        return self.data[i]

    def slice_rows(self, start: int, stop: int) -> "VectorDataset":
        return VectorDataset(self.data[start:stop])

    def __len__(self) -> int:
        return self.count

    def __repr__(self) -> str:
        return f"VectorDataset(count={self.count}, dims={self.dims}, kind={self._kind.value})"

    # ---- device mirror -------------------------------------------------
    def device(self) -> DeviceRows:
        """Upload once (rows + norms computed on device) and cache."""
        if self._dev is not None:
            return self._dev
        torch = _lib.require_cuda()
        with self._dev_lock:
            if self._dev is None:
                with warnings.catch_warnings():  # read-only numpy -> torch view, copied to HBM at once
                    warnings.simplefilter("ignore", UserWarning)
                    x = torch.from_numpy(np.ascontiguousarray(self._data)).to("cuda", non_blocking=False)
                if self._kind is ElementKind.U8:
                    if x.shape[1] * 255 ** 2 >= 1 << 32:
                        raise ValueError("u8 dims too large for 32-bit packed distances")
                    norms = torch.empty(x.shape[0], dtype=torch.int32, device=x.device)
                    if x.shape[0]:
                        _lib.check(_lib.lib().jb_row_sq_norms_u8(_lib.ptr(x), x.shape[0], x.shape[1], _lib.ptr(norms),
                                                                _lib.stream_ptr()))
                else:
                    norms = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
                    if x.shape[0]:
                        _lib.check(_lib.lib().jb_row_sq_norms(_lib.ptr(x), x.shape[0], x.shape[1], _lib.ptr(norms),
                                                             _lib.stream_ptr()))
                self._dev = DeviceRows(x, norms, x.shape[0], x.shape[1], self._kind)
        return self._dev

    def device_f32(self):
        """Exact f32 copy of u8 rows on the device (for the f64 medoid / ground-truth
        paths, which the reference runs on x.astype(f64)); the f32 rows otherwise."""
        dev = self.device()
        if self._kind is not ElementKind.U8:
            return dev.x
        cached = getattr(self, "_dev_f32", None)
        if cached is not None:
            return cached
        torch = _lib.require_cuda()
        out = torch.empty(dev.x.shape, dtype=torch.float32, device=dev.x.device)
        _lib.check(_lib.lib().jb_u8_to_f32(_lib.ptr(dev.x), dev.x.numel(), _lib.ptr(out), _lib.stream_ptr()))
        self._dev_f32 = out  # kept: the rerank reads it asynchronously
        return out

    def device_screen(self):
        """(records [n, jb_screen_record_bytes(D)] u8, centre [D] f32) on the device:
        int8 screen records of the f32 rows (extension, jb_search_args.screen),
        built once per dataset; None for u8 rows or D > 1040."""
        dev = self.device()
        if self._kind is ElementKind.U8 or dev.dims > 1040 or dev.count == 0:
            return None
        cached = getattr(self, "_dev_screen", None)
        if cached is not None:
            return cached
        torch = _lib.require_cuda()
        L = _lib.lib()
        st = _lib.stream_ptr()
        # any centre keeps the bound rigorous (eps is measured against it); the mean of
        # the first 64K rows is close enough and its sequential f64 chain is 16x shorter
        center = torch.empty(dev.dims, dtype=torch.float32, device=dev.x.device)
        _lib.check(L.jb_column_mean_f32(_lib.ptr(dev.x), min(dev.count, 65536), dev.dims, _lib.ptr(center), st))
        rb = int(L.jb_screen_record_bytes(dev.dims))
        rec = torch.empty((dev.count, rb), dtype=torch.uint8, device=dev.x.device)
        _lib.check(L.jb_screen_records(_lib.ptr(dev.x), _lib.ptr(dev.norms), dev.count, dev.dims, _lib.ptr(center),
                                       _lib.ptr(rec), st))
        self._dev_screen = (rec, center)
        return self._dev_screen


@dataclass(frozen=True)
class AugmentedDataset:
    """A dataset lifted into dims+1 space so inner-product ranking becomes L2
    ranking (core.py:111-130): data rows carry sqrt(M^2 - ||x||^2) in the last
    coordinate, query rows carry 0."""

    dataset: VectorDataset
    base_dims: int
    max_norm: float
    role: str  # "data" or "query"

    def __post_init__(self):
        if self.dataset.dims != self.base_dims + 1:
            raise ValueError("augmented dims must equal base dims + 1")
        if self.role not in ("data", "query"):
            raise ValueError(f"role must be 'data' or 'query', got {self.role!r}")


def mips_augment(data, queries) -> tuple[AugmentedDataset, AugmentedDataset]:
    """core.py:169-206 on the device (jb_mips_augment): [x, sqrt(M^2 - ||x||^2)] and
    [q, 0] written straight into HBM; the returned datasets wrap those rows."""
    data, queries = as_dataset(data), as_dataset(queries)
    if data.element_kind is not ElementKind.F32 or queries.element_kind is not ElementKind.F32:
        raise ValueError("mips_augment requires f32 datasets")
    if data.count == 0:
        raise ValueError("mips_augment requires non-empty data")
    if data.dims != queries.dims:
        raise ValueError(f"dimension mismatch: data dims {data.dims}, query dims {queries.dims}")
    torch = _lib.require_cuda()
    x, q = data.device().x, queries.device().x if queries.count else None
    D = data.dims
    ad = torch.empty((data.count, D + 1), dtype=torch.float32, device=x.device)
    aq = torch.empty((queries.count, D + 1), dtype=torch.float32, device=x.device)
    m2 = np.zeros(1, dtype=np.float64)
    _lib.check(_lib.lib().jb_mips_augment(_lib.ptr(x), data.count, D, _lib.ptr(q), queries.count, _lib.ptr(ad),
                                          _lib.ptr(aq), m2.ctypes.data, _lib.stream_ptr()))
    max_sq = float(m2[0])
    if not np.isfinite(max_sq):
        raise ValueError("non-finite norms in data")
    m = float(np.sqrt(max_sq))
    return (AugmentedDataset(VectorDataset.from_device(ad), D, m, "data"),
            AugmentedDataset(VectorDataset.from_device(aq), D, m, "query"))


def as_dataset(obj) -> VectorDataset:
    """Accept this package's VectorDataset or any object with a 2-D `.data` array
    (e.g. the reference's beamann.VectorDataset) — the drop-in path."""
    if isinstance(obj, VectorDataset):
        return obj
    if isinstance(obj, AugmentedDataset) or (hasattr(obj, "dataset") and hasattr(obj, "base_dims")):
        return as_dataset(obj.dataset)
    data = getattr(obj, "data", None)
    if isinstance(data, np.ndarray) and data.ndim == 2:
        cache = getattr(obj, "_jb_dataset", None)
        if cache is None:
            cache = VectorDataset(data)
            try:
                object.__setattr__(obj, "_jb_dataset", cache)
            except Exception:
                pass
        return cache
    raise TypeError(f"unsupported dataset {type(obj).__name__}")


def _require_same_shape(a: np.ndarray, b: np.ndarray) -> None:
    if a.shape != b.shape:
        raise ValueError(f"dimension mismatch: {a.shape} vs {b.shape}")


def row_sq_norms(x) -> np.ndarray:
    """core.py:161-166 on the device: per-row squared norms, integer-exact (int64) for
    u8 rows, f32 in einsum('nd,nd->n') order for f32 rows (jb_row_sq_norms_u8 /
    jb_row_sq_norms). Other dtypes: ValueError (the device path has the two element
    kinds of the reference's datasets)."""
    torch = _lib.require_cuda()
    a = np.asarray(x)
    if a.ndim != 2:
        raise ValueError("row_sq_norms expects a 2-D array")
    if a.dtype not in (np.float32, np.uint8):
        raise ValueError(f"row_sq_norms: f32 or u8 rows expected, got {a.dtype}")
    n, d = a.shape
    if n == 0:
        return np.zeros(0, dtype=np.int64 if a.dtype == np.uint8 else np.float32)
    xd = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    st = _lib.stream_ptr()
    if a.dtype == np.uint8:
        out = torch.empty(n, dtype=torch.int32, device="cuda")
        _lib.check(_lib.lib().jb_row_sq_norms_u8(_lib.ptr(xd), n, d, _lib.ptr(out), st))
        return out.cpu().numpy().view(np.uint32).astype(np.int64)
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().jb_row_sq_norms(_lib.ptr(xd), n, d, _lib.ptr(out), st))
    return out.cpu().numpy()


def sq_l2(a, b) -> float:
    """core.py:119-133 (scalar helper, host)."""
    a, b = np.asarray(a), np.asarray(b)
    _require_same_shape(a, b)
    if a.dtype == np.uint8 and b.dtype == np.uint8:
        d = a.astype(np.int64) - b.astype(np.int64)
        return int(np.dot(d, d))
    diff = a.astype(np.float32, copy=False) - b.astype(np.float32, copy=False)
    return float(np.dot(diff, diff))


def dot(a, b) -> float:
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    _require_same_shape(a, b)
    return float(np.dot(a, b))


def gen_synthetic(count: int, dims: int, seed: int, distribution: str = "gaussian") -> VectorDataset:
    """Same seeded draws as the reference (core.py:209-233)."""
    if count < 1 or dims < 1:
        raise ValueError("count and dims must be >= 1")
    rng = np.random.default_rng(seed)
    if distribution == "gaussian":
        x = rng.standard_normal((count, dims))
    elif distribution == "clustered":
        centers = rng.standard_normal((16, dims)) * 4.0
        assign = rng.integers(0, 16, size=count)
        x = centers[assign] + rng.standard_normal((count, dims))
    else:
        raise ValueError(f"unknown distribution {distribution!r}")
    return VectorDataset(x.astype(np.float32))


def gen_lowrank(count: int, dims: int, seed: int, d_int: int = 16, noise: float = 0.05,
                basis_seed: int | None = None) -> np.ndarray:
    """Low-intrinsic-dimension synthetic rows: SIFT/DEEP/GIST-shaped
    data on which recall@10 >= 0.95 is reachable. Returns f32 (count, dims).

    With basis_seed=None this is exactly the Appendix B recipe (one generator draws
    the basis, then the latent rows, then the noise). With basis_seed set, the
    basis comes from default_rng(basis_seed) and the rows from default_rng(seed),
    so disjoint shards and held-out queries share one subspace.
    """
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
