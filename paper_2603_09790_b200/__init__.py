"""paper_2603_09790_b200 -- B200-native Chebyshev-basis s-step PCG with FGS
Gram solves (arXiv 2603.09790), a drop-in for the reference chebstep solve
path. The compute path is libchebstep_gpu.so (hand-written sm_100a CUDA
behind include/chebstep_gpu.h); this package is the Python mirror of the
reference API on top of that C ABI. Importing it fails if the library has
not been built -- there is no CPU fallback.
"""
from .chebstep import *  # noqa: F401,F403
from .chebstep import (  # noqa: F401
    BasisBreakdownError, ChebyshevParams, Context, CsrMatrix, DeviceProblem, DimensionError,
    Error, FgsConfig, FgsResult, GramSolverKind, GramSystem, IdentityPreconditioner,
    InvalidArgumentError, InvalidMatrixError, JacobiPreconditioner, MpkResult, NotSpdError,
    PcgConfig, PoissonSpec, PoissonSystem, SolveReport, SolveResult, SolverBreakdownError,
    SolverConfig, SpectrumEstimate, assemble_gram, block_gram, block_update, default_context,
    device_count, estimate_interval, fgs_solve, gram_from_matrix, halo_map_csr, monitor_inexact,
    mpk_chebyshev, partition_rows, pcg_s_solve, pcg_solve, poisson27, random_vector,
    small_cholesky_solve, spmv, spmv_into, stencil7, tridiag_eigvals, read_matrix_market,
    write_matrix_market, validate_structure, validate_symmetric, validate_spd_diagonal, ParseError,
    normalize_gram, fgs_rate, FgsRate, kappa_sym, BlockJacobiPreconditioner,
    DevicePreconditioner)
from ._lib import LIB_PATH  # noqa: F401
