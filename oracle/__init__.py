"""ORACLE — TEST INFRASTRUCTURE ONLY. Not part of the product.

A plain numpy restatement of the reference package `beamann`'s hot path
(/root/reference/pkg/src/beamann, "the reference"), used as the checker for
the CUDA path and as the CPU baseline in bench.py. Only tests/, the
`smoke()` of __graft_entry__.py and bench.py's CPU-baseline leg may import it.
The product package (paper_2601_07048_b200) never imports anything here.

Parity pinning: every function here is checked against fixtures produced by
running the live reference in this container (tests/golden/make_golden.py,
committed with its outputs) and against the SPEC.md known-answer tests.
The arithmetic uses the same numpy primitives the reference uses (einsum,
pairwise sum, lexsort, f64 GEMM) so its rounding is the reference's rounding.
"""

from . import knn, rabitq, search, vamana  # noqa: F401
