"""B200-native block ILU(k) preconditioner (arXiv 1703.01325) -- drop-in for the
reference package ``blockiluk``'s factor / apply / Krylov entry points.

Host code here is thin: index containers, argument checks and exception
mapping.  Every numeric step of the path runs as hand-written sm_100a CUDA in
``_lib/libbiluk.so`` (C ABI: ``include/biluk.h``); torch tensors are used as
device buffers only.  There is no CPU fallback.
"""

from .errors import FactorizationError, MatrixMarketError, SingularBlockError, StructuralError
from .factor import (BlockIlukFactors, block_ilu0_factorize, block_invert, build_preconditioner, materialize,
                     point_ilu0_factorize, split_ldu, symbolic_phase)
from .krylov import SolverConfig, SolveStats, bicgstab, bicgstab_batched, gmres
from .sparse import (BcsrMatrix, CsrMatrix, PatternMatrix, assemble_csr, bcsr_from_csr, block_diagonal,
                     csr_expand, csr_from_triplets, extract_point_pattern)
from .matrix_market import read_matrix_market
from .symbolic import coupled_iluk_oracle
from .trisolve import (LevelSchedule, TriangularOperand, apply_block_diagonal, apply_preconditioner,
                       apply_preconditioner_many, build_level_schedule, solve_unit_triangular, strict_triangle)
from .device import DeviceOperator
from .synthetic import gen_poisson_3d, reservoir_block_grid

__version__ = "0.1.0"


def spmv(a, x, workers=1):
    """y = a @ x on the GPU (reference sparse.py:278-301); numpy in -> numpy out."""
    import numpy as np
    from .device import operator_for, torch
    t = torch()
    y = operator_for(a).matvec(x)
    if isinstance(x, t.Tensor) and x.is_cuda:
        return y
    return y.cpu().numpy()


__all__ = [
    "BcsrMatrix", "BlockIlukFactors", "CsrMatrix", "DeviceOperator", "FactorizationError", "LevelSchedule",
    "MatrixMarketError", "PatternMatrix", "SingularBlockError", "SolveStats", "SolverConfig", "StructuralError",
    "TriangularOperand", "apply_block_diagonal", "apply_preconditioner", "apply_preconditioner_many",
    "assemble_csr", "bcsr_from_csr", "bicgstab", "bicgstab_batched", "block_diagonal", "block_ilu0_factorize",
    "block_invert", "build_level_schedule", "build_preconditioner", "coupled_iluk_oracle", "csr_expand",
    "csr_from_triplets", "extract_point_pattern", "gen_poisson_3d", "gmres", "materialize",
    "point_ilu0_factorize", "read_matrix_market", "reservoir_block_grid", "solve_unit_triangular", "split_ldu",
    "spmv", "strict_triangle", "symbolic_phase", "__version__",
]
