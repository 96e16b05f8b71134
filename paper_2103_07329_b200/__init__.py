"""mrsolve-b200: B200-native solve phase of multi-RHS AMG-preconditioned Krylov.

Drop-in for the solve path of the reference package ``mrsolve``
(/root/reference/pkg/src/mrsolve): the same ``ParamTree`` configuration,
``prepare(config, A).run(B, X) -> SolveStats`` call and exception types,
executed by hand-written sm_100a CUDA kernels behind a C ABI
(include/mrsolve_b200.h, built into libmrsolve_b200.so).

Layout:
  core      host data model (CsrBlock, BlockVector, partitions)
  params    ParamTree configuration (roles, schemas, legality)
  amg       hierarchy: native bitwise restatement of the reference RS setup
  kernels   the kernel-plugin interface on CUDA tensors (csr_spmv, axpby, ...)
  solvers   prepare / ConfiguredSolver / SolveStats (device-driven solve)
  team      multi-GPU row partition over NCCL (halo exchange, allreduce)
  io        seeded generators for the BASELINE.json configurations
  sysfile   XAMGBIN1 system files and YAML run configurations
  cli       the batch driver (python -m paper_2103_07329_b200.cli)
"""

from .core import (SUPPORTED_NRHS, BlockVector, CsrBlock, IndexWidth, PrecisionTag,
                   VectorFlags, choose_width, compress_indices, make_partition)
from .errors import (BreakdownError, CapacityError, ConfigurationError, DeviceError,
                     FormatError, InstabilityError, InvalidArgumentError, MrSolveError,
                     SetupDegeneracyError, ShapeMismatchError, SingularDiagonalError,
                     SingularMatrixError)
from .io import gen_poisson3d, gen_random_sdd, gen_stencil27_aniso, seeded_rhs
from .sysfile import parse_run_config, read_system, write_system
from .params import ParamList, ParamTree
from .amg import AmgParams, Hierarchy, Level, estimate_eig_bounds, setup

__version__ = "0.1.0"


def __getattr__(name):
    # solver/kernels pull in torch + the CUDA library: import on first use
    if name in ("prepare", "solve", "SolveStats", "ConfiguredSolver"):
        from . import solvers
        return getattr(solvers, name)
    if name in ("kernels", "solvers", "team", "cli"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
