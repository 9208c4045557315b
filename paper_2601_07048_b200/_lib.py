"""ctypes binding of libjasper_b200.so (the C ABI declared in include/jasper_b200.h).

The product has exactly one compute path: the sm_100a kernels in this library.
Loading fails loudly if the library is missing or no CUDA device is present —
there is no CPU fallback anywhere in the package.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libjasper_b200.so")

JB_OK, JB_EINVAL, JB_ECUDA, JB_ENODONOR, JB_EOVERFLOW = 0, 1, 2, 3, 4
SRC_EXACT, SRC_RABITQ, SRC_RABITQ_FAST, SRC_EXACT_U8 = 0, 1, 2, 3
KIND_F32, KIND_U8 = 0, 1

p = C.c_void_p
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


class SearchArgs(C.Structure):
    _fields_ = [
        ("adjacency", p), ("degree_cap", i32), ("active_count", i64),
        ("source", i32), ("dims", i32), ("data", p), ("data_norms", p),
        ("records", p), ("record_bytes", i32), ("bits", i32),
        ("queries", p), ("query_add", p), ("query_sumq", p), ("nq", i64),
        ("starts", p), ("start_vertex", i64),
        ("beam_width", i32), ("hash_slots", i32), ("trace_cap", i32),
        ("frontier_keys", p), ("hops", p), ("evals", p), ("trace_ids", p), ("trace_dists", p),
        ("flags", p),
        ("data_u8", p), ("norms_u32", p), ("queries_u8", p), ("query_norms_u32", p),
        ("screen", p), ("screen_center", p),
    ]


class KnnPlan(C.Structure):
    _fields_ = [("search", SearchArgs), ("centroid", p), ("rotation", p), ("rerank_data", p), ("k", i32),
                ("chunk", i32)]


class InsertArgs(C.Structure):
    _fields_ = [
        ("adjacency", p), ("degrees", p), ("degree_cap", i32), ("capacity", i64),
        ("data", p), ("data_norms", p), ("dims", i32), ("count", i64),
        ("build_beam_width", i32), ("alpha", f64), ("always_prune", i32), ("reverse_all_visited", i32),
        ("start", i64), ("stop", i64), ("entry_point", i64),
        ("entry_point_out_host", p), ("bridges_out_host", p), ("stats_out_host", p),  # int64 [8]
        ("active_count", i64),
        ("element_kind", i32), ("data_u8", p), ("norms_u32", p),
        ("quantized", i32), ("records", p), ("record_bytes", i32), ("bits", i32),
        ("bound_rotated", p), ("bound_qadd", p), ("bound_qsumq", p),
        ("repair_beam_width", i32),
        ("closure", p), ("screen", p), ("screen_center", p),
    ]


_SIGS = {
    "jb_last_error": (C.c_char_p, []),
    "jb_abi_version": (C.c_int, []),
    "jb_sm_count": (C.c_int, [C.c_int, p]),
    "jb_row_sq_norms": (C.c_int, [p, i64, i32, p, p]),
    "jb_medoid": (C.c_int, [p, i64, i32, p, p]),
    "jb_row_sq_norms_u8": (C.c_int, [p, i64, i32, p, p]),
    "jb_medoid_u8": (C.c_int, [p, i64, i32, p, p]),
    "jb_u8_to_f32": (C.c_int, [p, i64, p, p]),
    "jb_beam_search": (C.c_int, [C.POINTER(SearchArgs), p]),
    "jb_frontier_topk": (C.c_int, [p, i64, i32, i32, p, p, p]),
    "jb_frontier_topk_u8": (C.c_int, [p, i64, i32, i32, p, p, p]),
    "jb_rerank_topk": (C.c_int, [p, i32, p, i64, p, i32, i32, p, p, p]),
    "jb_count_evals": (C.c_int, [p, i32, p, i32, p, p, i64, p, i64, p, p]),
    "jb_search_knn_host": (C.c_int, [C.POINTER(KnnPlan), p, i64, p, p, p]),
    "jb_search_knn_device": (C.c_int, [C.POINTER(KnnPlan), p, i64, p, p, p]),
    "jb_rabitq_record_bytes": (i32, [i32, i32]),
    "jb_rabitq_plane_record_bytes": (i32, [i32, i32]),
    "jb_rabitq_pack_planes": (C.c_int, [p, p, i64, i32, i32, p, p]),
    "jb_rabitq_pack_records": (C.c_int, [p, p, i64, i32, i32, p, p]),
    "jb_rabitq_encode": (C.c_int, [p, i64, i32, i32, p, p, p, p, p]),
    "jb_column_mean_f32": (C.c_int, [p, i64, i32, p, p]),
    "jb_screen_record_bytes": (i32, [i32]),
    "jb_screen_records": (C.c_int, [p, p, i64, i32, p, p, p]),
    "jb_rabitq_bind": (C.c_int, [p, i64, i32, i32, p, p, p, p, p, p]),
    "jb_batch_insert": (C.c_int, [C.POINTER(InsertArgs), p]),
    "jb_repair_connectivity": (C.c_int, [C.POINTER(InsertArgs), p]),
    "jb_refine_batch": (C.c_int, [C.POINTER(InsertArgs), p]),
    "jb_robust_prune": (C.c_int, [p, p, i32, p, i64, p, p, p, f64, i32, p, p, p, p]),
    "jb_exact_knn": (C.c_int, [p, i64, i32, p, i64, i32, p, p, p]),
    "jb_exact_knn_kind": (C.c_int, [p, i64, i32, p, i64, i32, i32, p, p, p]),
    "jb_mips_augment": (C.c_int, [p, i64, i32, p, i64, p, p, p, p]),
    "jb_merge_shard_topk": (C.c_int, [p, p, i32, i64, i32, p, p, p, p]),
    "jb_pack_shard_topk": (C.c_int, [p, p, i64, i32, i64, p, p]),
    "jb_bound_distances": (C.c_int, [C.POINTER(SearchArgs), i64, p, p, i64, p, p]),
    "jb_robust_prune_matrix": (C.c_int, [p, p, p, i32, f64, i32, p, p, p]),
    "jb_merge_shard_records": (C.c_int, [p, i32, i64, i32, p, p, p]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


def load_library() -> C.CDLL:
    """Load (without requiring a GPU) and type every exported symbol."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2601_07048_b200._build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def lib() -> C.CDLL:
    return _lib if _lib is not None else load_library()


class NoDonorError(RuntimeError):
    pass


def check(status: int) -> None:
    if status == JB_OK:
        return
    msg = (lib().jb_last_error() or b"").decode(errors="replace")
    if status == JB_EINVAL:
        raise ValueError(msg)
    if status == JB_ENODONOR:
        raise NoDonorError(msg)
    raise RuntimeError(f"jasper_b200 error {status}: {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2601_07048_b200 needs a CUDA device (B200, sm_100a); none is visible")
    return torch


def stream_ptr(stream=None) -> int:
    torch = require_cuda()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    """Device (or host) address of a torch tensor / numpy array; None passes NULL."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return int(t.data_ptr())
