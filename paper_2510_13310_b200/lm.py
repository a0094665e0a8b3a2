"""Levenberg-Marquardt driver types and entry points (drop-in for sparsesfm/lm.py).

`lm_solve(problem, theta0, config, workspace)` keeps the reference signature
and semantics (lm.py:727-800): same damping schedule, accept/reject rule,
termination strings and `SolveReport` records. For BAProblem / GPProblem the
whole iteration runs in the native library (csrc/ssfm.cu: ssfm_lm_solve); the
host only reads one small status block per iteration. Problems that are not
B200 problems (the reference's duck-typed provider protocol) go through the
generic device path in `sparse_block` (GPU J^T J / J^T r / Schur-PCG on the
explicit block system); there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as ct
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import (CGStall, SingularBlock, SolverFailure, ZeroQuaternion)


@dataclass(slots=True)
class LMConfig:
    """lm.py:36-58 (same defaults and validation)."""
    max_iterations: int = 100
    lambda0: float = 1e-4
    lambda_up: float = 10.0
    lambda_down: float = 2.0
    lambda_min: float = 1e-10
    lambda_max: float = 1e10
    rel_cost_tol: float = 1e-6
    grad_tol: float = 1e-10
    cg_max_iters: int = 500
    cg_tol: float = 1e-8
    solver: str = "schur_pcg"          # "schur_pcg" | "dense"

    def __post_init__(self):
        for name in ("lambda0", "lambda_up", "lambda_down", "lambda_min",
                     "lambda_max", "rel_cost_tol", "grad_tol", "cg_tol"):
            if not getattr(self, name) > 0:
                raise ValueError(f"{name} must be positive")
        if not (self.lambda_min < self.lambda0 < self.lambda_max):
            raise ValueError("need lambda_min < lambda0 < lambda_max")
        if self.solver not in ("schur_pcg", "dense"):
            raise ValueError(f"unknown solver {self.solver!r}")


@dataclass(slots=True)
class IterationRecord:
    """lm.py:61-69 (+ device_ms: CUDA-event time of the iteration)."""
    iteration: int
    cost_before: float
    cost_after: float
    lam: float
    step_accepted: bool
    cg_iters: int
    wall_time_ns: int
    device_ms: float = 0.0
    status: int = 0           # ssfm_status of an in-step failure (rejection), else 0


@dataclass(slots=True)
class SolveReport:
    iterations: list = field(default_factory=list)
    termination: str = "max_iter"

    @property
    def accepted_costs(self) -> list:
        return [it.cost_after for it in self.iterations if it.step_accepted]

    @property
    def num_accepted(self) -> int:
        return sum(1 for it in self.iterations if it.step_accepted)


class Workspace:
    """Grow-only scratch arena shared across solver stages (lm.py:86-101).

    Host arrays handed out by `take` mirror the reference. The device side is
    a grow-only HBM arena (`device_arena`, csrc: ssfm_arena): a native problem
    whose handle is first created through lm_solve / run_ba / run_gp with this
    workspace allocates from it, and once that problem is released the next
    stage's problem (GP -> BA) reuses the same HBM without cudaMalloc.
    """

    def __init__(self):
        self._arrays: dict = {}
        self.caches: dict = {}
        self._arena = None

    def device_arena(self):
        if self._arena is None:
            from . import _native
            self._arena = _native.Arena()
        return self._arena

    def release_device(self) -> None:
        """Free the device arena (every problem created in it must be released)."""
        if self._arena is not None:
            self._arena.close()
            self._arena = None

    def take(self, name: str, shape, dtype=np.float64) -> np.ndarray:
        if isinstance(shape, (int, np.integer)):
            shape = (int(shape),)
        size = int(np.prod(shape, dtype=np.int64))
        arr = self._arrays.get(name)
        if arr is None or arr.size < size or arr.dtype != np.dtype(dtype):
            arr = np.empty(max(size, 1), dtype=dtype)
            self._arrays[name] = arr
        return arr[:size].reshape(shape)


def renormalize(theta, layout):
    """Unit-normalise every camera_pose quaternion (lm.py:104-117)."""
    from .sparse_block import KIND_CODE
    out = np.array(theta, dtype=np.float64, copy=True)
    ids = np.nonzero(layout.kind_codes == KIND_CODE["camera_pose"])[0]
    if len(ids) == 0:
        return out
    idx = layout.param_offsets[ids][:, None] + np.arange(4)
    q = out[idx]
    nrm = np.linalg.norm(q, axis=1)
    if (nrm < 1e-12).any():
        raise ZeroQuaternion("quaternion norm below 1e-12 during renormalization")
    out[idx] = q / nrm[:, None]
    return out


def _torch():
    import torch
    if not torch.cuda.is_available():
        from .errors import NativeError
        raise NativeError("no CUDA device available: the B200 solver has no CPU path")
    return torch


def _stream(torch):
    return ct.c_void_p(torch.cuda.current_stream().cuda_stream)


def _to_device_theta(torch, theta0):
    is_t = isinstance(theta0, torch.Tensor)
    t = theta0.detach().to(device="cuda", dtype=torch.float64).clone() if is_t else \
        torch.as_tensor(np.asarray(theta0, dtype=np.float64)).to("cuda")
    return t.contiguous(), is_t


def lm_solve(problem, theta0, config: LMConfig | None = None,
             workspace: Workspace | None = None):
    """Levenberg-Marquardt with accept/reject damping control (lm.py:727-800).

    Returns (theta, SolveReport); theta is a numpy array for numpy input and a
    CUDA tensor for tensor input.
    """
    config = config or LMConfig()
    native = getattr(problem, "_native_handle", None)
    if native is None:
        from .sparse_block import generic_lm_solve
        return generic_lm_solve(problem, theta0, config, workspace)
    if config.solver != "schur_pcg":
        from .sparse_block import generic_lm_solve
        return generic_lm_solve(problem, theta0, config, workspace)
    torch = _torch()
    theta, was_tensor = _to_device_theta(torch, theta0)
    if theta.numel() != problem.layout.total_params:
        from .errors import DimensionMismatch
        raise DimensionMismatch("theta0 length does not match the problem layout")
    if not bool(torch.isfinite(theta).all()):
        raise ValueError("theta0 must be finite")
    h = native(workspace) if workspace is not None else native()
    lib = _native.load()
    cap = max(1, int(config.max_iterations))
    recs = (_native.IterRecordC * cap)()
    nrec = ct.c_int32(0)
    term = ct.c_int32(0)
    cfg = _native.lm_config_c(config)
    getattr(problem, "_enter_collective", lambda: None)()
    rc = lib.ssfm_lm_solve(ct.c_void_p(h.ptr), ct.c_void_p(theta.data_ptr()), ct.byref(cfg), recs,
                           cap, ct.byref(nrec), ct.byref(term), _stream(torch))
    report = SolveReport(termination=_native.TERMINATIONS.get(term.value, "max_iter"))
    for k in range(nrec.value):
        r = recs[k]
        report.iterations.append(IterationRecord(
            int(r.iteration), float(r.cost_before), float(r.cost_after), float(r.lam),
            bool(r.step_accepted), int(r.cg_iters), int(r.wall_time_ns), float(r.device_ms),
            int(r.status)))
    if rc == 3:
        msg = lib.ssfm_last_error().decode(errors="replace")
        report.termination = "solver_failure"
        raise SolverFailure(msg, report)
    _native.check(rc)
    if was_tensor:
        return theta, report
    return theta.cpu().numpy(), report


def solve_normal(sys, layout, config: LMConfig, workspace: Workspace | None = None,
                 info: dict | None = None):
    """Solve the damped normal equations (lm.py:707-720) on the device.

    `sys` is a BlockNormalSystem (already damped, gradient = -J^T r). Raises
    SingularBlock or CGStall like the reference.
    """
    from .sparse_block import generic_solve_normal
    return generic_solve_normal(sys, layout, config, workspace, info)


__all__ = ["LMConfig", "IterationRecord", "SolveReport", "Workspace", "renormalize",
           "lm_solve", "solve_normal", "CGStall", "SingularBlock"]


def _now_ns() -> int:
    return time.perf_counter_ns()
