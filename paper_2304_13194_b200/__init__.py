"""B200-native Jet multilevel k-way graph partitioner (arXiv 2304.13194).

Drop-in for the hot path of the reference package `jetpart`:
`partition(graph, RefinerConfig(k=...)) -> PartitionResult`, plus the
per-kernel functions of coarsening and Jet refinement under the reference's
names. All compute runs in hand-written sm_100a CUDA kernels in libjet.so.
"""

from .config import RefinerConfig, rebalance_thresholds
from .driver import PartitionResult, partition, project
from .errors import (BalanceInfeasibleError, JetpartError, ParseError, PreprocessError,
                     RebalanceInfeasibleError)
from .graph import (
    Graph,
    PartitionState,
    cutsize,
    from_edge_arrays,
    imbalance_of,
    is_balanced,
    part_weight_limit,
)
from .moves import MoveList
from .ops import (
    ConnectivityTable,
    Hierarchy,
    LockTable,
    afterburner,
    build_conn,
    build_hierarchy,
    contract,
    initial_partition,
    jet_refine,
    jetlp_pass,
    match_vertices,
    select_destinations,
    strong_rebalance_pass,
    update_conn,
    weak_rebalance_pass,
)
from ._lib import Context, DeviceGraph

__version__ = "0.1.0"

__all__ = [
    "BalanceInfeasibleError", "ConnectivityTable", "Context", "DeviceGraph", "Graph", "Hierarchy", "JetpartError",
    "LockTable", "MoveList", "ParseError", "PreprocessError", "PartitionResult", "PartitionState", "RebalanceInfeasibleError",
    "RefinerConfig", "afterburner", "build_conn", "build_hierarchy", "contract", "cutsize",
    "from_edge_arrays", "imbalance_of", "initial_partition", "is_balanced", "jet_refine",
    "jetlp_pass", "match_vertices", "part_weight_limit", "partition", "project",
    "rebalance_thresholds", "select_destinations", "strong_rebalance_pass",
    "update_conn", "weak_rebalance_pass",
]
