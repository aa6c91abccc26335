"""B200-native matrix-free phase-field-fracture hot path (arXiv 2005.00331).

Drop-in for the operator / multigrid / Krylov API of the reference package
fracturekit 0.1.0: the same names and signatures, computed by hand-written
sm_100a CUDA kernels in ``libpff_b200.so`` (C ABI: include/pff_b200.h).
"""

from ._lib import PffError
from .active_set import (ActiveSetParams, ActiveSetSolver, SolveReport, SolverFailure,
                         converged, determine_active_set, lumped_mass_diagonal)
from .basis import LANE_WIDTHS, MaterialParams, ShapeData, shape_data
from .krylov import GmresResult, KrylovConfig, gmres_solve
from .mesh import ConstraintSet, DofMap, MeshHierarchy, MeshLevel, build_hierarchy
from .multigrid import (ChebyshevConfig, GmgPreconditioner, TransferOperator,
                        build_prolongation, chebyshev_apply, estimate_lambda_max,
                        estimate_lambda_range)
from .operator import (AssemblyMemoryError, BlockVector, JacobianOperator, SparseOracle, assemble_oracle,
                       cell_matrices, LinearizationState, StaleCacheError,
                       apply_block_phiphi, apply_block_uu, apply_jacobian, apply_phi_row,
                       block_diagonal, block_diagonals, extrapolate_phase, residual, restrict_state_to_level)

from .simulation import (BenchRecord, LoadRecord, MemoryReport, ScenarioConfig, SimulationResult,
                         apply_boundary_values, benchmark_vmult, boundary_program, memory_report,
                         reaction_load, run_simulation)

__version__ = "0.1.0"
