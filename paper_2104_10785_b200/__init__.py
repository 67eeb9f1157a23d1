"""B200-native Golub-Kahan bidiagonalization path of arXiv 2104.10785.

Drop-in for the hot-path API of the reference package `krysvd`
(reference __init__.py:5-41): same names, arguments, return types and
exceptions for bidiagonalize / fsvd / estimate_rank and their helpers.
Computation runs in libksvd.so (hand-written sm_100a CUDA + NCCL); there is
no CPU fallback.
"""

from .bidiag import (BidiagConfig, BidiagState, GKRun, bidiagonal_matrix,
                     bidiagonalize, run_gk, with_k_max)
from .errors import ConfigError, NumericalError, ShapeMismatchError
from .fsvd import SymTridiag, fsvd, gram_tridiag, symtridiag_eig
from .linops import (GK_START, DeviceMatrix, FactoredOperator, LinearOperator, PartialSvd,
                     as_operator, row_partition, substream)
from .matrixio import (read_csv_matrix, read_matrix, read_matrix_device, write_matrix,
                       write_matrix_device)
from .rank import RankReport, count_above, estimate_rank
from .restart import RestartInfo, fsvd_restarted

__version__ = "0.1.0"

__all__ = [
    "BidiagConfig", "BidiagState", "GKRun", "bidiagonal_matrix", "bidiagonalize",
    "run_gk", "with_k_max",
    "ConfigError", "NumericalError", "ShapeMismatchError",
    "SymTridiag", "fsvd", "gram_tridiag", "symtridiag_eig",
    "GK_START", "DeviceMatrix", "FactoredOperator", "LinearOperator", "PartialSvd", "as_operator",
    "row_partition", "substream",
    "RankReport", "count_above", "estimate_rank", "RestartInfo", "fsvd_restarted",
    "read_csv_matrix", "read_matrix", "read_matrix_device", "write_matrix", "write_matrix_device",
    "__version__",
]
