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
from .lobpcg import (  # noqa: F401,E402
    DenseOperator,
    EigenState,
    SolverConfig,
    lobpcg_solve,
    orthonormalize,
    random_init,
    rayleigh_ritz,
    residual_norms,
)
from .spectral import (  # noqa: F401,E402
    GapResult,
    Partition,
    assign_clusters_kmeans,
    assign_clusters_qrcp,
    block_size_for,
    detect_gap,
    partition_static,
    read_labels,
    write_labels,
)
from .metrics import (  # noqa: F401,E402
    ContingencyTable,
    contingency,
    pair_counts,
    pairwise_precision,
    pairwise_recall,
    partition_match,
    stage_record,
)
from .streaming import (  # noqa: F401,E402
    StageResult,
    StreamStage,
    load_manifest,
    partition_stream,
    warm_start,
    write_manifest,
)
