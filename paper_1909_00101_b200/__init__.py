"""B200-native blocked one-sided (implicit) Hari-Zimmermann GSVD.

Drop-in for the reference package's GSVD entry point (hzgsvd.solve,
pkg/src/hzgsvd/blocked.py:640-663): same inputs, same GsvdResult, same
configuration and exceptions, with the hot path in hand-written sm_100a
CUDA (libhzg.so, C ABI in include/hzg.h).
"""

from .accuracy import AccuracyReport, accuracy_report, invert_via_lu
from .config import EPS, SolverConfig, SweepStats
from .core import GsvdResult, MatrixPlanePair, ProblemPair, border_pair
from .errors import (DeviceError, FileFormatError, HzgsvdError, NotPositiveDefiniteError,
                     ProtocolError, RankError)
from .ops import (cholesky_upper, form_grammians, postmultiply, preprocess_tall, qr_shorten, rescale_z,
                  run_distributed)
from .solver import DeviceGsvd, clear_cache, gsvd_1x1, gsvd_blocked, solve, upload_bordered
from .planes_io import read_matrix, read_sigma_tsv, write_matrix, write_result, write_sigma_tsv
from .stripes import StripeState, exchange_step, partition_stripes
from .strategies import (CommMapping, StrategyTable, block_moves, circle_positions, comm_mapping,
                         dump_table, gen_table, validate_table)

__version__ = "0.1.0"

__all__ = [
    "EPS", "SolverConfig", "SweepStats", "GsvdResult", "MatrixPlanePair", "ProblemPair", "border_pair",
    "DeviceError", "FileFormatError", "HzgsvdError",
    "NotPositiveDefiniteError", "ProtocolError", "RankError", "DeviceGsvd", "gsvd_1x1", "gsvd_blocked",
    "solve", "upload_bordered", "CommMapping", "StrategyTable", "block_moves", "circle_positions",
    "comm_mapping", "dump_table", "gen_table", "validate_table", "cholesky_upper", "form_grammians",
    "postmultiply", "qr_shorten", "rescale_z", "run_distributed", "clear_cache", "preprocess_tall",
    "StripeState", "exchange_step", "partition_stripes", "AccuracyReport", "accuracy_report", "invert_via_lu",
    "read_matrix", "write_matrix", "read_sigma_tsv", "write_sigma_tsv", "write_result",
]
