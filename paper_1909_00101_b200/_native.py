"""ctypes binding of libhzg.so (the C ABI declared in include/hzg.h).

There is no fallback: if the library is missing or no CUDA device is
present, every entry point raises DeviceError.
"""

import ctypes
import os
import threading

from .errors import DeviceError, NotPositiveDefiniteError, RankError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HZG_LIB") or os.path.join(HERE, "_lib", "libhzg.so")

HZG_OK, HZG_RANK, HZG_NOT_PD, HZG_CUDA, HZG_INVALID = 0, 1, 2, 3, 4


class HzgConfig(ctypes.Structure):
    _fields_ = [("variant_id", ctypes.c_int32), ("outer_mm", ctypes.c_int32), ("inner_mm", ctypes.c_int32),
                ("max_inner_sweeps", ctypes.c_int32), ("max_outer_sweeps", ctypes.c_int32),
                ("block_width", ctypes.c_int32), ("sorting", ctypes.c_int32), ("fallback_qr", ctypes.c_int32),
                ("shorten_qr", ctypes.c_int32), ("gate_eps", ctypes.c_double), ("exact", ctypes.c_int32),
                ("split_rows", ctypes.c_int32), ("approx_2x2", ctypes.c_int32)]


EXPORTS = ("hzg_create", "hzg_workspace_bytes", "hzg_bind", "hzg_set_schedule", "hzg_set_z_rows", "hzg_init_fgz", "hzg_sweep", "hzg_sweep_launch", "hzg_sweep_wait",
           "hzg_run_steps", "hzg_run_pairs", "hzg_wave_step", "hzg_wave_join", "hzg_collect", "hzg_rescale_z", "hzg_finalize", "hzg_test_block", "hzg_set_timing", "hzg_kernel_times",
           "hzg_step_counters", "hzg_debug_phases", "hzg_launch_counts", "hzg_op_grammian",
           "hzg_op_cholesky_upper", "hzg_op_qr_shorten", "hzg_op_qr_rfactor", "hzg_op_postmultiply", "hzg_op_rescale", "hzg_test_fastmath", "hzg_comm_unique_id", "hzg_comm_unique_id_bytes", "hzg_comm_attach",
           "hzg_comm_set_moves", "hzg_dist_sweep", "hzg_dist_sweep_launch", "hzg_dist_sweep_wait",
           "hzg_comm_attach_all", "hzg_comm_exchange_all", "hzg_comm_exchange", "hzg_comm_detach", "hzg_lu_workspace_bytes",
           "hzg_lu_complete", "hzg_gemm_comp", "hzg_sumsq_comp", "hzg_last_error",
           "hzg_destroy")

_lib = None
_lock = threading.Lock()


def load(path=LIB_PATH):
    """Load libhzg.so and declare its signatures (no device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError("libhzg.so not built (%s); run __graft_entry__.build()" % path)
        L = ctypes.CDLL(path)
        P, I32, I64, D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.hzg_create.argtypes = [ctypes.POINTER(P), ctypes.c_int, I64, I64, I64, I32,
                                 ctypes.POINTER(HzgConfig), D]
        L.hzg_create.restype = ctypes.c_int
        L.hzg_workspace_bytes.argtypes = [P]
        L.hzg_workspace_bytes.restype = ctypes.c_size_t
        L.hzg_bind.argtypes = [P] + [P] * 6 + [P, P]
        L.hzg_bind.restype = ctypes.c_int
        L.hzg_set_schedule.argtypes = [P, P, I32, I32]
        L.hzg_set_schedule.restype = ctypes.c_int
        L.hzg_set_z_rows.argtypes = [P, I64]
        L.hzg_set_z_rows.restype = ctypes.c_int
        L.hzg_init_fgz.argtypes = [P]
        L.hzg_init_fgz.restype = ctypes.c_int
        L.hzg_sweep.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hzg_sweep_launch.argtypes = [P]
        L.hzg_sweep_launch.restype = ctypes.c_int
        L.hzg_sweep_wait.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hzg_sweep_wait.restype = ctypes.c_int
        L.hzg_sweep.restype = ctypes.c_int
        L.hzg_run_steps.argtypes = [P, I32, I32]
        L.hzg_run_steps.restype = ctypes.c_int
        L.hzg_run_pairs.argtypes = [P, I32, I32, I32, P]
        L.hzg_run_pairs.restype = ctypes.c_int
        L.hzg_wave_step.argtypes = [P, I32, I32, P, P]
        L.hzg_wave_step.restype = ctypes.c_int
        L.hzg_wave_join.argtypes = [P, P, P]
        L.hzg_wave_join.restype = ctypes.c_int
        L.hzg_collect.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hzg_collect.restype = ctypes.c_int
        L.hzg_rescale_z.argtypes = [P]
        L.hzg_rescale_z.restype = ctypes.c_int
        L.hzg_finalize.argtypes = [P, I64, I64, I64, I32] + [P] * 9
        L.hzg_finalize.restype = ctypes.c_int
        L.hzg_test_block.argtypes = [I32, I32, ctypes.POINTER(HzgConfig), D] + [P] * 6 + [P]
        L.hzg_test_block.restype = ctypes.c_int
        L.hzg_set_timing.argtypes = [P, I32]
        L.hzg_set_timing.restype = ctypes.c_int
        L.hzg_kernel_times.argtypes = [P, P, P, I32]
        L.hzg_kernel_times.restype = ctypes.c_int
        L.hzg_step_counters.argtypes = [P, P, I64, ctypes.POINTER(I64)]
        L.hzg_step_counters.restype = ctypes.c_int
        L.hzg_debug_phases.argtypes = [P, I32, P]
        L.hzg_debug_phases.restype = ctypes.c_int
        L.hzg_launch_counts.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hzg_launch_counts.restype = ctypes.c_int
        L.hzg_op_grammian.argtypes = [I64, I32, I32, I32, P, P, P, P, P]
        L.hzg_op_grammian.restype = ctypes.c_int
        L.hzg_op_cholesky_upper.argtypes = [I32, I32, P, P, P]
        L.hzg_op_cholesky_upper.restype = ctypes.c_int
        L.hzg_op_qr_shorten.argtypes = [I64, I32, I32, P, P, P, P, P]
        L.hzg_op_qr_shorten.restype = ctypes.c_int
        L.hzg_op_qr_rfactor.argtypes = [I64, I32, I32, I32, ctypes.c_double, P, P, P, P, P]
        L.hzg_op_qr_rfactor.restype = ctypes.c_int
        L.hzg_op_postmultiply.argtypes = [I64, I32, I32, P, P, P, P, P]
        L.hzg_op_postmultiply.restype = ctypes.c_int
        L.hzg_op_rescale.argtypes = [I64, I64, I64, I32, I32, I32] + [P] * 6 + [I64, P, P, P, P]
        L.hzg_op_rescale.restype = ctypes.c_int
        L.hzg_test_fastmath.argtypes = [I64, ctypes.c_uint64, P]
        L.hzg_test_fastmath.restype = ctypes.c_int
        L.hzg_comm_unique_id.argtypes = [P]
        L.hzg_comm_unique_id.restype = ctypes.c_int
        L.hzg_comm_unique_id_bytes.argtypes = []
        L.hzg_comm_unique_id_bytes.restype = ctypes.c_size_t
        L.hzg_comm_attach.argtypes = [P, I32, I32, P]
        L.hzg_comm_attach.restype = ctypes.c_int
        L.hzg_comm_set_moves.argtypes = [P, P, P, I32]
        L.hzg_comm_set_moves.restype = ctypes.c_int
        L.hzg_dist_sweep.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hzg_dist_sweep.restype = ctypes.c_int
        L.hzg_dist_sweep_launch.argtypes = [P]
        L.hzg_dist_sweep_launch.restype = ctypes.c_int
        L.hzg_dist_sweep_wait.argtypes = [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]
        L.hzg_dist_sweep_wait.restype = ctypes.c_int
        L.hzg_comm_attach_all.argtypes = [P, I32]
        L.hzg_comm_attach_all.restype = ctypes.c_int
        L.hzg_comm_exchange_all.argtypes = [P, I32, P, I32]
        L.hzg_comm_exchange_all.restype = ctypes.c_int
        L.hzg_comm_exchange.argtypes = [P, P, I32]
        L.hzg_comm_exchange.restype = ctypes.c_int
        L.hzg_comm_detach.argtypes = [P]
        L.hzg_comm_detach.restype = ctypes.c_int
        L.hzg_lu_workspace_bytes.argtypes = [I64]
        L.hzg_lu_workspace_bytes.restype = ctypes.c_size_t
        L.hzg_lu_complete.argtypes = [I64, I32, P, P, I64, P, P, P, P, P]
        L.hzg_lu_complete.restype = ctypes.c_int
        L.hzg_gemm_comp.argtypes = [I64, I64, I64, I32, I32, P, P, I64, P, P, I64, P, P, I64, P]
        L.hzg_gemm_comp.restype = ctypes.c_int
        L.hzg_sumsq_comp.argtypes = [I64, I64, P, P, I64, P, P, I64, I32, P, I32, P]
        L.hzg_sumsq_comp.restype = ctypes.c_int
        L.hzg_last_error.argtypes = [P]
        L.hzg_last_error.restype = ctypes.c_char_p
        L.hzg_destroy.argtypes = [P]
        L.hzg_destroy.restype = None
        _lib = L
        return L


def make_config(cfg):
    """Decode a SolverConfig into the C struct."""
    return HzgConfig(cfg.variant_id, int(cfg.outer_kind == "mm"), int(cfg.inner_kind == "mm"),
                     cfg.max_inner_sweeps, cfg.max_outer_sweeps, cfg.block_width, int(bool(cfg.sorting)),
                     int(bool(cfg.fallback_qr)), int(cfg.shorten == "qr"), float(cfg.gate_eps),
                     int(bool(getattr(cfg, "exact", False))), int(getattr(cfg, "split_rows", 0)),
                     int(bool(getattr(cfg, "approx_2x2", True)) and not getattr(cfg, "exact", False)))


def check(code, ctx=None, what=""):
    """Map a C status to the reference's exceptions."""
    if code == HZG_OK:
        return
    msg = what
    if ctx is not None:
        try:
            m = load().hzg_last_error(ctx)
            if m:
                msg = "%s: %s" % (what, m.decode()) if what else m.decode()
        except Exception:
            pass
    if code == HZG_NOT_PD:
        raise NotPositiveDefiniteError(msg)
    if code == HZG_RANK:
        raise RankError(msg)
    if code == HZG_INVALID:
        raise ValueError(msg or "invalid argument to the device solver")
    raise DeviceError(msg or "CUDA failure")
