"""B200-native hot path of the multigrid-in-time KKT preconditioner of
arXiv 2405.04808, behind the reference package's (``tempokkt``) solver and
preconditioner API.

Host code is Python; every operator application, block-Jacobi sweep,
block Gauss-Seidel substitution, time transfer and Krylov vector operation
is a hand-written sm_100a CUDA kernel in ``libtempokkt_b200.so`` reached
through the C-ABI in ``include/tempokkt_b200.h``.  There is no CPU
fallback: without the library (or a GPU) the compute entry points raise.
"""

__version__ = "0.1.0"

from .errors import (Breakdown, ConfigError, DimensionMismatch, IndivisibleSteps,
                     NativeLibraryError, NewtonDivergence, NonFiniteValue, SingularBlock,
                     SingularMatrix, TempoKktError, UnsupportedStructure)
from .timedisc import ProblemSpec, TimeGrid, Trajectory, forward_solve
from .problems import (BurgersConfig, HeatNeumannConfig, VanDerPolConfig, build_burgers,
                       build_heat_neumann, build_vanderpol)
from .kkt import (BlockTriKKT, DiagonalSolver, KktLayout, StageBlocks, assemble_kkt,
                  assemble_rhs, build_stage_blocks, check_theorem1, clustered_permutation,
                  dump_matrix_market, factor_diagonal, from_clustered, split_parts,
                  stage_blocks_from_arrays, to_clustered)
from .krylov import LinearOperator, Preconditioner, SolveReport, fgmres, gmres
from .smoothers import (bgs_apply, fgs_apply, jacobi_apply, sgs_apply,
                        smoother_preconditioner)
from .multigrid import (MgHierarchy, TransferOps, build_hierarchy, coarse_solve, cycle,
                        default_levels, mg_preconditioner)
from .pipeline import HostPipeline

__all__ = [
    "Breakdown", "ConfigError", "DimensionMismatch", "IndivisibleSteps", "NativeLibraryError",
    "NewtonDivergence", "NonFiniteValue", "SingularBlock", "SingularMatrix", "TempoKktError",
    "UnsupportedStructure",
    "ProblemSpec", "TimeGrid", "Trajectory", "forward_solve",
    "BurgersConfig", "HeatNeumannConfig", "VanDerPolConfig", "build_burgers",
    "build_heat_neumann", "build_vanderpol",
    "BlockTriKKT", "DiagonalSolver", "KktLayout", "StageBlocks", "assemble_kkt",
    "build_stage_blocks", "stage_blocks_from_arrays", "assemble_rhs", "check_theorem1",
    "clustered_permutation", "dump_matrix_market", "factor_diagonal", "from_clustered",
    "split_parts", "to_clustered",
    "LinearOperator", "Preconditioner", "SolveReport", "fgmres", "gmres",
    "bgs_apply", "fgs_apply", "jacobi_apply", "sgs_apply", "smoother_preconditioner",
    "MgHierarchy", "TransferOps", "build_hierarchy", "coarse_solve", "cycle",
    "default_levels", "mg_preconditioner", "HostPipeline",
]
