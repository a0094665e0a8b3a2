"""ctypes binding of the C-ABI in include/ssfm.h.

The shared library is built in-tree (`python __graft_entry__.py` or
`make -C paper_2510_13310_b200/csrc`) into `paper_2510_13310_b200/_lib/`.
There is no fallback: if the library or a CUDA device is missing, every
solver entry point raises.
"""

from __future__ import annotations

import ctypes as ct
import os

from .errors import NativeError, raise_for_status

LIB_PATH = os.environ.get("SSFM_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                                                         "libssfm_b200.so")   # override: kernel-variant experiments

# Functions the header declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "ssfm_last_error", "ssfm_version", "ssfm_create_ba", "ssfm_create_gp",
    "ssfm_destroy", "ssfm_num_params", "ssfm_num_residuals", "ssfm_device_bytes",
    "ssfm_cost", "ssfm_linearize", "ssfm_solve_normal", "ssfm_post_step",
    "ssfm_lm_solve", "ssfm_export_pattern", "ssfm_profile_get", "ssfm_profile_enable",
    "ssfm_operator_info", "ssfm_comm_init", "ssfm_comm_connect", "ssfm_check_jacobian",
    "ssfm_bench_operator", "ssfm_reproj_stats", "ssfm_block_jtj", "ssfm_block_jtr",
    "ssfm_block_scale_diag", "ssfm_dense_scatter", "ssfm_dense_solve",
    "ssfm_rotation_auc", "ssfm_center_moments", "ssfm_apply_sim3",
    "ssfm_bal_read", "ssfm_bal_take", "ssfm_bal_free", "ssfm_make_rays", "ssfm_schur_solve",
    "ssfm_trim_cache", "ssfm_cache_bytes", "ssfm_arena_create", "ssfm_arena_destroy", "ssfm_arena_info",
    "ssfm_create_ba_in", "ssfm_create_gp_in", "ssfm_lm_mode", "ssfm_prune", "ssfm_handle_device", "ssfm_enable_peer_access",
)

TERMINATIONS = {0: "max_iter", 1: "converged_cost", 2: "converged_grad", 3: "solver_failure"}


class LMConfigC(ct.Structure):
    _fields_ = [
        ("max_iterations", ct.c_int32),
        ("lambda0", ct.c_double), ("lambda_up", ct.c_double), ("lambda_down", ct.c_double),
        ("lambda_min", ct.c_double), ("lambda_max", ct.c_double),
        ("rel_cost_tol", ct.c_double), ("grad_tol", ct.c_double),
        ("cg_max_iters", ct.c_int32),
        ("cg_tol", ct.c_double),
    ]


class IterRecordC(ct.Structure):
    _fields_ = [
        ("iteration", ct.c_int32), ("step_accepted", ct.c_int32),
        ("cg_iters", ct.c_int32), ("status", ct.c_int32),
        ("cost_before", ct.c_double), ("cost_after", ct.c_double), ("lam", ct.c_double),
        ("wall_time_ns", ct.c_int64), ("device_ms", ct.c_double),
    ]


class BADescC(ct.Structure):
    _fields_ = [
        ("num_cameras", ct.c_int32), ("num_points", ct.c_int32), ("num_obs", ct.c_int64),
        ("model", ct.c_int32), ("optimize_focal", ct.c_int32), ("shared_focal", ct.c_int32),
        ("loss_kind", ct.c_int32), ("loss_delta", ct.c_double),
        ("cam_idx", ct.c_void_p), ("pt_idx", ct.c_void_p), ("pixels", ct.c_void_p),
        ("pps", ct.c_void_p), ("dists", ct.c_void_p), ("focals", ct.c_void_p),
    ]


class GPDescC(ct.Structure):
    _fields_ = [
        ("num_cameras", ct.c_int32), ("num_points", ct.c_int32), ("num_obs", ct.c_int64),
        ("depth_mode", ct.c_int32), ("gauge_fixed", ct.c_int32),
        ("loss_kind", ct.c_int32), ("loss_delta", ct.c_double),
        ("cam_idx", ct.c_void_p), ("pt_idx", ct.c_void_p), ("rays", ct.c_void_p),
        ("depths", ct.c_void_p),
    ]


# ssfm_schur_plan (include/ssfm.h): sizes, then device pointers in header order
SCHUR_PLAN_SIZES = ("n_params", "n_ret", "n_rblk", "n_pt", "n_u", "n_slots", "n_sc", "n_direct")
SCHUR_PLAN_ARRAYS = (
    ("ret_s_off", "i8"), ("ret_theta", "i8"), ("pre_off", "i8"), ("direct_dst", "i8"), ("direct_src", "i8"),
    ("pt_diag", "i8"), ("pt_theta", "i8"), ("u_w", "i4"), ("u_ret", "i4"), ("u_pt", "i4"), ("u_off", "i8"),
    ("u_gather", "i8"), ("u_by_ret", "i4"), ("ret_useg", "i8"), ("u_by_pt", "i4"), ("pt_useg", "i8"),
    ("slot_seg", "i8"), ("slot_ra", "i4"), ("slot_rb", "i4"), ("con_ua", "i4"), ("con_ub", "i4"),
    ("sc_diag", "i8"), ("sc_theta", "i8"), ("sc_uc", "i8"), ("sc_up", "i8"), ("sc_c", "i4"), ("sc_p", "i4"),
    ("sc_u", "i4"), ("sc_by_c", "i4"), ("c_scseg", "i8"), ("sc_by_p", "i4"), ("p_scseg", "i8"),
    ("sc_by_u", "i4"), ("u_scseg", "i8"),
)


class SchurPlanC(ct.Structure):
    _fields_ = [(n, ct.c_int64) for n in SCHUR_PLAN_SIZES] + [(n, ct.c_void_p) for n, _ in SCHUR_PLAN_ARRAYS]


_lib = None


def load(required: bool = True):
    """Load the library once. Raises NativeError when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if required:
            raise NativeError(f"native library not built: {LIB_PATH} (run __graft_entry__.build())")
        return None
    lib = ct.CDLL(LIB_PATH)
    P, I32, I64, D = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_double
    lib.ssfm_last_error.restype = ct.c_char_p
    lib.ssfm_version.restype = ct.c_char_p
    lib.ssfm_handle_device.argtypes = [P]
    lib.ssfm_handle_device.restype = I32
    lib.ssfm_enable_peer_access.argtypes = [I32, I32]
    lib.ssfm_lm_mode.argtypes = [P]
    lib.ssfm_lm_mode.restype = I32
    lib.ssfm_prune.argtypes = [I64, P, P, I32, I32, P, P, P, ct.POINTER(I32), ct.POINTER(I32), ct.POINTER(I64), P]
    lib.ssfm_create_ba.argtypes = [ct.POINTER(BADescC), P, ct.POINTER(P)]
    lib.ssfm_create_gp.argtypes = [ct.POINTER(GPDescC), P, ct.POINTER(P)]
    lib.ssfm_destroy.argtypes = [P]
    for fn in ("ssfm_num_params", "ssfm_num_residuals", "ssfm_device_bytes"):
        getattr(lib, fn).argtypes = [P]
        getattr(lib, fn).restype = I64
    lib.ssfm_cost.argtypes = [P, P, ct.POINTER(D), P]
    lib.ssfm_linearize.argtypes = [P, P, P, P, P, ct.POINTER(D), P]
    lib.ssfm_solve_normal.argtypes = [P, D, ct.POINTER(LMConfigC), P, ct.POINTER(I32), P]
    lib.ssfm_post_step.argtypes = [P, P, P]
    lib.ssfm_lm_solve.argtypes = [P, P, ct.POINTER(LMConfigC), ct.POINTER(IterRecordC), I32,
                                  ct.POINTER(I32), ct.POINTER(I32), P]
    lib.ssfm_export_pattern.argtypes = [P, P, P, P, I64, ct.POINTER(I64), P, I64, ct.POINTER(I64), P]
    lib.ssfm_profile_get.argtypes = [P, I32, ct.POINTER(D), ct.POINTER(I64), ct.POINTER(D)]
    lib.ssfm_profile_enable.argtypes = [P, I32]
    lib.ssfm_rotation_auc.argtypes = [P, P, I32, P, I32, P, P]
    lib.ssfm_center_moments.argtypes = [P, P, I32, P, P]
    lib.ssfm_apply_sim3.argtypes = [P, P, D, P, P, P, I32, P, I64, P]
    lib.ssfm_bal_read.argtypes = [ct.c_char_p, ct.POINTER(P), P]
    lib.ssfm_bal_take.argtypes = [P, P, P, P, P, P]
    lib.ssfm_make_rays.argtypes = [I64, P, P, P, P, P, P, P, P, P]
    lib.ssfm_bal_free.argtypes = [P]
    lib.ssfm_trim_cache.argtypes = [I32, ct.POINTER(I64)]
    lib.ssfm_arena_create.argtypes = [I32, I64, ct.POINTER(P)]
    lib.ssfm_arena_destroy.argtypes = [P]
    lib.ssfm_arena_info.argtypes = [P, ct.POINTER(I64), ct.POINTER(I64), ct.POINTER(I32), ct.POINTER(I64)]
    lib.ssfm_create_ba_in.argtypes = [ct.POINTER(BADescC), P, P, ct.POINTER(P)]
    lib.ssfm_create_gp_in.argtypes = [ct.POINTER(GPDescC), P, P, ct.POINTER(P)]
    lib.ssfm_cache_bytes.argtypes = []
    lib.ssfm_cache_bytes.restype = I64
    lib.ssfm_schur_solve.argtypes = [ct.POINTER(SchurPlanC), P, P, ct.POINTER(LMConfigC), P, ct.POINTER(I32), P]
    lib.ssfm_bal_free.restype = None
    for fn in EXPORTS:
        if fn not in ("ssfm_last_error", "ssfm_version", "ssfm_num_params", "ssfm_num_residuals",
                      "ssfm_device_bytes", "ssfm_bal_free", "ssfm_cache_bytes"):
            getattr(lib, fn).restype = ct.c_int
    _lib = lib
    return lib


def check(code: int) -> None:
    if code != 0:
        msg = load().ssfm_last_error().decode(errors="replace")
        raise_for_status(code, msg)


def lm_config_c(cfg) -> LMConfigC:
    return LMConfigC(int(cfg.max_iterations), float(cfg.lambda0), float(cfg.lambda_up),
                     float(cfg.lambda_down), float(cfg.lambda_min), float(cfg.lambda_max),
                     float(cfg.rel_cost_tol), float(cfg.grad_tol), int(cfg.cg_max_iters),
                     float(cfg.cg_tol))


def trim_cache(device: int = -1) -> int:
    """Free the device blocks that destroyed handles left in the library's
    reuse cache (ssfm_trim_cache); returns the bytes freed."""
    lib = load(required=False)
    if lib is None:
        return 0
    freed = ct.c_int64(0)
    check(lib.ssfm_trim_cache(int(device), ct.byref(freed)))
    return int(freed.value)


class Arena:
    """A grow-only device arena (ssfm_arena_*): native problems created in it
    share its HBM stage after stage (the Workspace's device side)."""

    def __init__(self, reserve_bytes: int = 0):
        out = ct.c_void_p(0)
        check(load().ssfm_arena_create(-1, int(reserve_bytes), ct.byref(out)))
        self.ptr = out.value

    def info(self) -> dict:
        cap, hw, nm = ct.c_int64(0), ct.c_int64(0), ct.c_int64(0)
        live = ct.c_int32(0)
        check(load().ssfm_arena_info(ct.c_void_p(self.ptr), ct.byref(cap), ct.byref(hw), ct.byref(live),
                                     ct.byref(nm)))
        return {"capacity": cap.value, "high_water": hw.value, "live_handles": live.value,
                "chunk_mallocs": nm.value}

    def close(self) -> None:
        if self.ptr and _lib is not None:
            check(_lib.ssfm_arena_destroy(ct.c_void_p(self.ptr)))
        self.ptr = 0

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                _lib.ssfm_arena_destroy(ct.c_void_p(self.ptr))
        except Exception:
            pass
        self.ptr = 0


class Handle:
    """Owns one native problem handle (device arena) on the current CUDA device."""

    def __init__(self, ptr: int, keepalive=()):
        self.ptr = ptr
        self._keepalive = keepalive  # input tensors must outlive creation only

    def __del__(self):
        try:
            if self.ptr and _lib is not None:
                _lib.ssfm_destroy(ct.c_void_p(self.ptr))
        except Exception:
            pass
        self.ptr = 0
