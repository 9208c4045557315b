"""paper_2601_07048_b200 — B200-native hot paths of Jasper (arXiv 2601.07048).

Drop-in for the reference package `beamann`'s index API (build / insert /
search with R, L, alpha and k): the same names, argument meanings, error
behaviour and return types, with every hot loop running as hand-written
sm_100a CUDA kernels in libjasper_b200.so (C ABI: include/jasper_b200.h).
There is no CPU fallback: without the library or a CUDA device, calls raise.
"""

from .build import BuildParams, EdgeBuffer, batch_insert, build, insert_stream
from .core import (AugmentedDataset, DistanceKind, ElementKind, VectorDataset, dot, gen_lowrank, gen_synthetic,
                   mips_augment, row_sq_norms, sq_l2)
from .graph import Candidate, FormatError, GraphIndex, medoid, robust_prune
from .rabitq import QueryPrep, RaBitQIndex, estimate_sq_dist, prep_query, rotate
from .rabitq import fit as rabitq_fit
from .search import (SearchParams, SearchResult, SearchStats, beam_search, run_beam_searches, search_knn,
                     search_knn_batch, search_knn_batch_device)

from . import measure, shard  # noqa: E402
from .measure import GroundTruth, SweepPoint, exact_knn, recall_at_k, run_queries, sweep  # noqa: E402

__version__ = "0.1.0"

__all__ = [
    "BuildParams", "EdgeBuffer", "batch_insert", "build", "insert_stream",
    "AugmentedDataset", "mips_augment", "Candidate", "DistanceKind", "ElementKind", "FormatError", "GraphIndex", "QueryPrep", "RaBitQIndex",
    "SearchParams", "SearchResult", "SearchStats", "VectorDataset", "beam_search", "dot", "estimate_sq_dist",
    "gen_lowrank", "gen_synthetic", "medoid", "prep_query", "rabitq_fit", "robust_prune", "rotate",
    "run_beam_searches", "search_knn", "GroundTruth", "exact_knn", "SweepPoint", "recall_at_k", "run_queries", "sweep", "search_knn_batch", "search_knn_batch_device", "sq_l2", "row_sq_norms",
]
