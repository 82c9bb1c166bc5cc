"""B200-native spectral partitioning hot path (arXiv 1708.07481 / specpart).

Drop-in for the reference package's hot path: ``from_edges`` ->
``partition_static`` (LOBPCG on the graph Laplacian + QRCP assignment), with
every numeric kernel in hand-written CUDA for sm_100a (``csrc/``) reached
through the C ABI in ``include/specpart_b200.h``.
"""

__version__ = "0.1.0"

from .errors import (  # noqa: F401
    AssignmentError,
    ConditioningError,
    ContractError,
    DomainError,
    NativeError,
    ParseError,
    SolverError,
    SpecpartError,
    StreamStageError,
    UndefinedMetricError,
)
from .graph import (  # noqa: F401
    LaplacianOperator,
    SparseGraph,
    apply_delta,
    degrees,
    empty_graph,
    from_edges,
    laplacian_apply,
    load_edge_list,
    symmetrize,
    write_edge_list,
)
