"""B200-native fcLSH engine (Fast CoveringLSH, arXiv 1602.02620).

The compute path is libfclsh_b200.so (sm_100a kernels + C++ host behind the
C-ABI in include/fclsh_gpu.h); this package is the Python mirror of the
reference library's API over it (``fclsh``), the BASELINE workload
definitions (``configs``) and the multi-GPU sharded cluster (``cluster``).
"""
from . import fclsh  # noqa: F401
from .fclsh import (  # noqa: F401
    M31, M61, ConstructionKind, CoveringFamily, DataError, IndexSet, PlanKind, PlanOverride, PreprocessPlan,
    ResourceError, UsageError, build_covering_family, build_index, hash_batch, make_covering_family, make_plan,
)
