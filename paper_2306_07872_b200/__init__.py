"""B200-native weighted DAWN (arXiv 2306.07872): GOVM/GSVM shortest paths.

Drop-in for the hot path of the reference package ``sparsepath``: the same
solver names, signatures, return types and error behaviour, executed by
hand-written sm_100a CUDA kernels behind the C ABI in ``include/dawn.h``
(``libdawn.so``, loaded through ctypes).  There is no CPU fallback.
"""

from .device import (
    DeviceGraph,
    clear_cache,
    device_graph,
    get_default_precision,
    get_default_schedule,
    set_default_precision,
    set_default_schedule,
    set_tuning,
)
from .graph import (
    CsrGraph,
    EdgeList,
    WeightMode,
    apply_weight_mode,
    build_csr,
    csr_from_arrays,
    generate_random_graph,
    to_edge_list,
)
from .solver import (
    SOLVERS,
    AggregateStats,
    DistanceVector,
    FrontierFlags,
    PredecessorVector,
    SolveStats,
    aggregate_stats,
    apsp,
    format_distance_row,
    format_distance_rows,
    govm_sssp,
    gsvm_sssp,
    mssp,
    mssp_stats,
    read_distance_rows,
    seed_source,
    write_distance_rows,
)

from .errors import (
    GraphParseError,
    GraphSizeError,
    NegativeWeightError,
    SparsepathError,
    UnsupportedFormatError,
)
from .experiments import MuReport, run_mu_experiment
from .graphio import (
    load_edge_list,
    load_matrix_market,
    read_graph,
    write_edge_list,
    write_graph,
    write_matrix_market,
)
from .oracles import (
    DEFAULT_FLOYD_CAP,
    FloydResult,
    OracleResult,
    bellman_ford_sssp,
    dijkstra_sssp,
    floyd_warshall_apsp,
)

__version__ = "0.1.0"

__all__ = [
    "CsrGraph",
    "EdgeList",
    "WeightMode",
    "apply_weight_mode",
    "build_csr",
    "csr_from_arrays",
    "generate_random_graph",
    "to_edge_list",
    "DistanceVector",
    "PredecessorVector",
    "FrontierFlags",
    "SolveStats",
    "AggregateStats",
    "seed_source",
    "gsvm_sssp",
    "govm_sssp",
    "mssp",
    "mssp_stats",
    "apsp",
    "aggregate_stats",
    "format_distance_row",
    "format_distance_rows",
    "write_distance_rows",
    "read_distance_rows",
    "SOLVERS",
    "DeviceGraph",
    "device_graph",
    "clear_cache",
    "set_default_precision",
    "get_default_precision",
    "set_tuning",
    "set_default_schedule",
    "get_default_schedule",
    "MuReport",
    "run_mu_experiment",
    "SparsepathError",
    "GraphParseError",
    "UnsupportedFormatError",
    "NegativeWeightError",
    "GraphSizeError",
    "OracleResult",
    "FloydResult",
    "dijkstra_sssp",
    "bellman_ford_sssp",
    "floyd_warshall_apsp",
    "DEFAULT_FLOYD_CAP",
    "load_edge_list",
    "load_matrix_market",
    "write_edge_list",
    "write_matrix_market",
    "read_graph",
    "write_graph",
]
