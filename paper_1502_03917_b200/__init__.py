"""B200-native all-at-once multigrid for Poisson and Stokes control.

Drop-in for the hot path of the reference package ``ocmg`` (arXiv
1502.03917, Takacs): the same assemble / smoother / cycle / solve entry
points (``ocmg/__init__.py:13-50``, hot-path subset), backed by hand-written
sm_100a CUDA kernels behind the C ABI in ``include/ocmg_b200.h``.  Vectors
are CUDA fp64 tensors in the reference's global layout; numpy arrays are
accepted and copied through.  There is no CPU fallback.
"""
from ._lib import SingularMatrixError, build
from .assembly import (BlockSystem, FieldLayout, assemble_p1,
                       assemble_taylor_hood, build_poisson_system,
                       build_stokes_system, p1_class_tables,
                       pressure_mean_projection)
from .mesh import StructuredMesh
from .multigrid import (CoarseSolver, CycleConfig, Multigrid, SolveReport,
                        assemble_hierarchy, baseline_rhs, build_solver)
from .smoothers import (SmootherKind, SmootherState, cgs_sweep, lsgs_sweep,
                        make_smoother, normal_equation_sweep, slsgs_sweep,
                        vanka_sweep)
from .transfer import (TransferPair, p1_prolongation, p2_prolongation,
                       system_transfer)
from .vanka import VankaPatches, build_vanka_patches

__version__ = "0.1.0"

__all__ = [
    "BlockSystem", "CoarseSolver", "CycleConfig", "FieldLayout", "Multigrid",
    "SingularMatrixError", "SmootherKind", "SmootherState", "SolveReport",
    "StructuredMesh", "TransferPair", "assemble_hierarchy", "assemble_p1",
    "assemble_taylor_hood", "baseline_rhs", "build", "build_poisson_system",
    "build_solver", "build_stokes_system", "cgs_sweep", "lsgs_sweep",
    "make_smoother",
    "normal_equation_sweep", "p1_class_tables", "p1_prolongation",
    "p2_prolongation", "pressure_mean_projection", "slsgs_sweep",
    "system_transfer", "VankaPatches", "build_vanka_patches", "vanka_sweep",
]
