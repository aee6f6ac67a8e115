"""B200-native fp64 Schwarz smoothers for SIPG Laplacians (arXiv 1910.11239).

Drop-in for the hot path of the reference package `dgmg`: the matrix-free
SIPG operator, the cell / vertex-patch fast-diagonalisation solver sets and
the additive / coloured-multiplicative smoothing steps, computed by
hand-written sm_100a CUDA kernels behind a C ABI (include/dgmg_b200.h).
"""

from . import basis, dgop, distorted, experiment, fastdiag, flops, krylov, mesh, multigrid, smoothers, tables  # noqa: F401
from .basis import Basis1D  # noqa: F401
from .dgop import apply_operator, make_context, residual  # noqa: F401
from .fastdiag import CellSolverSet, PatchSolverSet, SingularLocalSolverError  # noqa: F401
from .flops import FlopCounter  # noqa: F401
from .krylov import pcg, pgmres  # noqa: F401
from .mesh import build_hierarchy, box_level  # noqa: F401
from .multigrid import LevelTransfer, MultigridConfig, VCycle, build_transfer  # noqa: F401
from .smoothers import (LevelSmoother, SmootherConfig, make_level_smoother,  # noqa: F401
                        smooth_additive, smooth_multiplicative)

__version__ = "0.1.0"
