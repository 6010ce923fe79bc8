"""B200-native mixed-precision Sylvester / Lyapunov solver (arXiv 2503.03456).

Drop-in for the hot path of the reference package ``mpsylv``: the solver
entry points ``mp_orth`` / ``mp_inv`` / ``solve_pert_sylv_tri_stat`` with the
reference's ``SylvesterProblem`` / ``RefinementConfig`` / ``SolveReport`` and
exception types, backed by hand-written sm_100a CUDA kernels behind the C ABI
in ``include/mpsylv_b200.h``.  ``solve`` is the torch-native entry.
"""

import os as _os

# one hardware work queue per stream for the batched lane executor (C4): must be in the
# environment before the CUDA context exists, i.e. before torch touches the device
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

from .costmodel import FlopCount, flops
from .errors import (DeviceError, DimensionError, FormatOverflowError, IterationLimitError, MpsylvError,
                     NotHermitianError, NumericBreakdownError, PrecisionOverflowWarning, RankDeficiencyError,
                     SingularEquationError, SingularMatrixError, UnsupportedPrecisionError)
from .precision import (B24, BFLOAT16, BINARY16, BINARY32, BINARY64, FORMATS, TF32, FlopCounter, FpFormat,
                        PrecisionContext, format_from_name, parse_format)
from .refinement import RefinementConfig, SolveReport, mp_inv, mp_orth, solve, solve_pert_sylv_tri_stat
from .batch import gather_solutions, shard_range, solve_batched
from .sylvester import DirectSolveReport, SylvesterProblem, bartels_stewart, residual, solve_sylv_tri
from .linalg import QrFactors, SchurFactors, gemm, mgs_qr, schur
from .condition import KappaEstimate, kappa_sylv, kappa_sylv_tensor
from .hermitian import hermitian_eig, solve_hermitian
from .split2 import mp_inv_split2, mp_orth_split2, solve_factored
from .gmresir import GmresConfig, GmresIrReport, apply_preconditioner, gmres_ir_sylv

__version__ = "0.1.0"
