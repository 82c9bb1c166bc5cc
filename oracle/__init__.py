"""CPU oracle for the spectral-partition hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in numpy/scipy, the algorithm of the reference package
``specpart`` (``/root/reference/pkg/src/specpart``) for the path BASELINE.json
names: edge list -> directed CSR -> W = A + A' and degrees -> matrix-free
Laplacian -> soft-locked LOBPCG -> gap detection -> QRCP assignment. Every
function cites the reference file:line it follows.

It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
it. The product package ``paper_1708_07481_b200`` never imports it and has no
CPU fallback.

Pinning: ``tests/golden/make_golden.py`` runs the real reference (importable in
the build container from /root/reference/pkg/src) on seeded inputs and commits
the outputs (CSR hashes, Ritz/residual histories, labels) as fixtures;
``tests/test_oracle_golden.py`` checks this restatement against them.
"""

from .graph_ref import (  # noqa: F401
    coerce_edges,
    directed_csr,
    symmetrize_csr,
    directed_degrees,
    laplacian_apply,
    LaplacianRef,
)
from .lobpcg_ref import SolverCfg, lobpcg_ref, orthonormalize_ref, small_gen_eigh_ref, random_init  # noqa: F401
from .spectral_ref import (  # noqa: F401
    block_size_for,
    detect_gap_ref,
    qrcp_assign_ref,
    partition_static_ref,
)
from .streaming_ref import partition_stream_ref, warm_start_ref  # noqa: F401
from .metrics_ref import contingency_counts, partition_match, pairwise_recall, pairwise_precision  # noqa: F401
