"""B200-native ChFSI: the hot path of `spectral_chain` (arXiv:1206.3768)
rebuilt on sm_100a.

Drop-in import surface for the reference's solver path
(`spectral_chain/__init__.py:15-80`): same names and signatures; arrays
live in HBM as CUDA tensors; all n-sized arithmetic runs in libchfsi.so
(hand-written CUDA + cuBLAS/cuSOLVER), loaded lazily on first use.
"""

from .linalg_errors import (
    EigenSolverError,
    NotHermitianError,
    NotPositiveDefiniteError,
    RankDeficientError,
)
from .linalg import (
    cholesky,
    gemm,
    hermitian_eig,
    hermitian_view,
    qr_orthonormalize,
    triangular_solve,
)
from .reduction import (
    EigenPencil,
    EigenSolution,
    StandardProblem,
    back_transform,
    forward_transform,
    residual,
    to_standard,
)
from .chfsi import (
    ChfsiConfig,
    ChfsiGuess,
    FilterWindow,
    SolveReport,
    chebyshev_filter,
    chebyshev_response,
    chfsi_solve,
    filter_flops,
    lanczos_upper_bound,
    rayleigh_ritz,
)
from .harness import OracleMismatchError, oracle_solve, solve_sequence
from .sequence import BASELINE_CONFIGS, BaselineConfig, iter_baseline_sequence
from .pencil_io import FormatError, load_sequence, read_pencil, save_sequence, write_pencil
from .analysis import AngleReport, angle_report, match_eigenvectors
from ._lib import BackendUnavailable

__version__ = "0.1.0"
