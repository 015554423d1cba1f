"""B200-native ChFSI: the hot path of `spectral_chain` (arXiv:1206.3768)
rebuilt on sm_100a.

Drop-in import surface for the reference's solver path
(`spectral_chain/__init__.py:15-80`): same names and signatures. All n-sized
arithmetic runs in libchfsi.so (hand-written CUDA + cuBLAS/cuSOLVER), loaded
lazily on first use; results come back as numpy arrays for numpy inputs (as
the reference's) and stay in HBM as CUDA tensors for CUDA-tensor inputs
(`set_array_output` / `array_output` override that policy).
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
from .harness import (
    REPORT_FIELDS,
    SOLVERS,
    BaselineSource,
    ExperimentReport,
    ExperimentRow,
    ExperimentSpec,
    GenerateSource,
    LoadSource,
    OracleMismatchError,
    emit_report,
    oracle_solve,
    run_experiment,
    solve_sequence,
)
from .sequence import (
    BASELINE_CONFIGS,
    BaselineConfig,
    CorrelationSchedule,
    PencilSequence,
    generate_sequence,
    iter_baseline_sequence,
)
from ._device import array_output, get_array_output, set_array_output
from .pencil_io import FormatError, load_sequence, read_pencil, save_sequence, write_pencil
from .analysis import AngleReport, angle_report, match_eigenvectors
from ._lib import BackendUnavailable

__version__ = "0.1.0"
