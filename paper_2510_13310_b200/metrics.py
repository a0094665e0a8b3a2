"""Accuracy metrics of a reconstruction on the device.

Same names, arguments, results and errors as the reference's
`synth_metrics.align` / `center_rmse` / `rotation_auc` (synth_metrics.py:
199-309); the O(C^2) pairwise AUC, the Umeyama moments and the Sim(3)
transform of every point run as CUDA kernels (csrc/metrics.cuh). The 3x3 SVD
and its sign fix stay host logic, as in the reference.

The `*_device` variants take CUDA tensors and leave the scene on the device
(for the GP -> BA pipeline); the Scene / SceneArrays variants copy the arrays
host -> device once.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import InsufficientCameras
from .lm import _stream, _torch
from .scene import SceneArrays, arrays_to_scene, as_arrays, quat_from_matrix


@dataclass(slots=True)
class Alignment:
    """y ~ s R x + t (synth_metrics.py:199-207)"""
    kind: str
    rotation: np.ndarray
    translation: np.ndarray
    scale: float

    def apply(self, x: np.ndarray) -> np.ndarray:
        return self.scale * (np.asarray(x) @ self.rotation.T) + self.translation


def _dev(torch, a, width):
    if isinstance(a, torch.Tensor):
        if not a.is_cuda or a.dtype != torch.float64:
            raise ValueError("expected a float64 CUDA tensor")
        return a.contiguous().view(-1, width)
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64).reshape(-1, width), device="cuda")


def _ptr(t) -> ct.c_void_p:
    return ct.c_void_p(t.data_ptr())


def center_moments_device(x, y) -> np.ndarray:
    """[mx(3), my(3), cov(9), var_x, sum|x-y|^2] of the [n][3] centres x (estimate), y (truth)."""
    torch = _torch()
    xd, yd = _dev(torch, x, 3), _dev(torch, y, 3)
    out = np.zeros(17)
    _native.check(_native.load().ssfm_center_moments(_ptr(xd), _ptr(yd), len(xd), out.ctypes.data_as(ct.c_void_p),
                                                     _stream(torch)))
    return out


def _alignment(m: np.ndarray, n: int, kind: str) -> Alignment:
    mx, my, cov, var_x = m[0:3], m[3:6], m[6:15].reshape(3, 3), float(m[15])
    u, d, vt = np.linalg.svd(cov)
    s3 = np.ones(3)
    if np.linalg.det(u) * np.linalg.det(vt) < 0:
        s3[2] = -1.0
    rot = u @ np.diag(s3) @ vt
    scale = 1.0
    if kind == "sim3":
        scale = float((d * s3).sum()) / var_x
        if scale <= 0:
            raise InsufficientCameras("degenerate similarity (non-positive scale)")
    return Alignment(kind, rot, my - scale * rot @ mx, scale)


def _check_align(kind: str, n: int, m: int) -> None:
    if kind not in ("sim3", "se3"):
        raise ValueError(f"unknown alignment kind {kind!r}")
    if n != m:
        raise InsufficientCameras("camera counts differ")
    if kind == "sim3" and n < 3:
        raise InsufficientCameras("sim3 alignment needs at least 3 cameras")
    if n < 2:
        raise InsufficientCameras("alignment needs at least 2 cameras")


def align_device(quats, centers, points, true_centers, kind: str = "sim3") -> Alignment:
    """Register the estimate's camera centres onto the truth's and transform
    the estimate (quats [C][4], centers [C][3], points [P][3] float64 CUDA
    tensors) IN PLACE (synth_metrics.py:210-257)."""
    torch = _torch()
    _check_align(kind, len(centers), len(true_centers))
    al = _alignment(center_moments_device(centers, true_centers), len(centers), kind)
    rq = quat_from_matrix(al.rotation)
    rqc = np.array([rq[0], -rq[1], -rq[2], -rq[3]])
    rot = np.ascontiguousarray(al.rotation, dtype=np.float64).reshape(-1)
    tr = np.ascontiguousarray(al.translation, dtype=np.float64)
    for t, w in ((quats, 4), (centers, 3), (points, 3)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("align_device transforms contiguous float64 CUDA tensors in place")
    _native.check(_native.load().ssfm_apply_sim3(
        rot.ctypes.data_as(ct.c_void_p), tr.ctypes.data_as(ct.c_void_p), al.scale, rqc.ctypes.data_as(ct.c_void_p),
        _ptr(quats), _ptr(centers), len(centers), _ptr(points), points.numel() // 3, _stream(torch)))
    return al


def align(estimate, truth, kind: str = "sim3"):
    """Closed-form least-squares registration of camera centres; returns the
    transform (y ~ s R x + t) and the transformed estimate
    (synth_metrics.py:210-257)."""
    torch = _torch()
    est, tru = as_arrays(estimate), as_arrays(truth)
    _check_align(kind, est.num_cameras, tru.num_cameras)
    q, c, p = (_dev(torch, est.quats, 4).clone(), _dev(torch, est.centers, 3).clone(),
               _dev(torch, est.points, 3).clone())
    al = align_device(q, c, p, _dev(torch, tru.centers, 3), kind)
    out = est.copy()
    out.quats, out.centers, out.points = q.cpu().numpy(), c.cpu().numpy(), p.cpu().numpy()
    return al, (out if isinstance(estimate, SceneArrays) else arrays_to_scene(out))


def center_rmse(estimate, truth) -> float:
    """sqrt(mean |c_est - c_true|^2) over cameras (synth_metrics.py:260-263)."""
    a, b = as_arrays(estimate).centers, as_arrays(truth).centers
    return center_rmse_device(a, b)


def center_rmse_device(a, b) -> float:
    n = len(a)
    m = center_moments_device(a, b)
    return float(np.sqrt(m[16] / n))


def rotation_auc_device(q_est, q_true, thresholds_deg) -> dict[float, float]:
    """Pairwise relative-rotation AUC (0-100) of [C][4] quaternion arrays or
    CUDA tensors: for every unordered camera pair the error is the angle of
    R_est_rel R_true_rel^T; AUC@tau = mean max(0, 1 - err/tau) * 100
    (synth_metrics.py:281-309)."""
    torch = _torch()
    c = len(q_est)
    if c < 2 or c != len(q_true):
        raise InsufficientCameras("need two scenes with >= 2 matching cameras")
    taus = [float(t) for t in thresholds_deg]
    out: dict[float, float] = {}
    qe, qt = _dev(torch, q_est, 4), _dev(torch, q_true, 4)
    for k in range(0, len(taus), 16):
        chunk = np.ascontiguousarray(taus[k:k + 16], dtype=np.float64)
        res = np.zeros(len(chunk))
        _native.check(_native.load().ssfm_rotation_auc(_ptr(qe), _ptr(qt), c, chunk.ctypes.data_as(ct.c_void_p),
                                                       len(chunk), res.ctypes.data_as(ct.c_void_p), _stream(torch)))
        out.update({t: float(v) for t, v in zip(chunk.tolist(), res.tolist())})
    return out


def rotation_auc(estimate, truth, thresholds_deg) -> dict[float, float]:
    return rotation_auc_device(as_arrays(estimate).quats, as_arrays(truth).quats, thresholds_deg)
