"""Global SfM solve stage: GP then BA on the device.

The reference has no pipeline function; SPEC's global SfM loop runs global
positioning (gp.py:204-218, rotations fixed) and then bundle adjustment
(ba.py:264-271) on the GP output, sharing one workspace. Here both stages
stay on the device: GP writes its centres and points into a copy of the scene
(rotations and focals untouched, exactly run_gp), BA starts from it. Both
handles live in one Workspace device arena: the GP handle is released before
the BA handle is created, so the two stages reuse the same HBM (the "unified
memory pool" of PAPER.md:165), and the hand-off never leaves the device.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from . import _native
from .ba import BAProblem
from .gp import fix_gauge, make_rays_device
from .lm import LMConfig, SolveReport, Workspace, _stream, _torch, lm_solve
from .scene import RobustLoss, SceneArrays, as_arrays


@dataclass
class PipelineReport:
    gp: SolveReport
    ba: SolveReport
    rmse_after_gp: float
    rmse_after_ba: float
    # with `truth`: Sim(3)-aligned camera-centre RMSE and pairwise rotation AUC
    # (synth_metrics.align / center_rmse / rotation_auc, on the device)
    center_rmse: float | None = None
    rotation_auc: dict | None = None


def reproj_stats(problem: BAProblem, theta) -> tuple[float, int]:
    """(sum of squared pixel errors, number of observations in front of their
    camera) on the device (the numerator / denominator of synth_metrics
    reproj_rmse, synth_metrics.py:312-325)."""
    torch = _torch()
    t = problem._theta_dev(torch, theta)
    s, n = ct.c_double(0.0), ct.c_int64(0)
    _native.check(_native.load().ssfm_reproj_stats(ct.c_void_p(problem._native_handle().ptr),
                                                   ct.c_void_p(t.data_ptr()), ct.byref(s), ct.byref(n),
                                                   _stream(torch)))
    return float(s.value), int(n.value)


def reproj_rmse_device(problem: BAProblem, theta) -> float:
    s, n = reproj_stats(problem, theta)
    return float(np.sqrt(s / n)) if n else float("nan")


def run_global_sfm(scene, gp_loss: RobustLoss | None = None, ba_loss: RobustLoss | None = None,
                   gp_config: LMConfig | None = None, ba_config: LMConfig | None = None, seed: int = 0,
                   optimize_focal: bool = True, truth=None, auc_thresholds=(1.0, 3.0, 5.0, 10.0),
                   workspace: Workspace | None = None):
    """GP (Huber 0.1 by default, seeded init, gauge fixed) then BA (Huber 1.0)
    on the GP output. Returns (scene, PipelineReport); with `truth` the report
    carries the aligned centre RMSE and the rotation AUC (metrics.py).

    Device-resident hand-off: the observations are uploaded once (the GP rays
    are built from them on the device), both stages share one Workspace arena
    (the GP handle is released before the BA handle is created in the same
    HBM), and BA starts from the GP solution without leaving the device; only
    the final parameters come back to the host."""
    torch = _torch()
    arr = as_arrays(scene)
    gp_loss = gp_loss or RobustLoss("huber", 0.1)
    ba_loss = ba_loss or RobustLoss("huber", 1.0)
    ws = workspace or Workspace()
    gp = fix_gauge(make_rays_device(arr, depth_mode=False, loss=gp_loss, seed=seed))
    cam32, pt32 = gp._dev_inputs["cam"], gp._dev_inputs["pt"]
    pix = torch.as_tensor(np.ascontiguousarray(arr.pixels, dtype=np.float64)).to("cuda", non_blocking=True)
    th0 = torch.as_tensor(gp.initial_theta()).to("cuda")
    th_gp, rep_gp = lm_solve(gp, th0, gp_config or LMConfig(max_iterations=20), ws)
    C, P = arr.num_cameras, arr.num_points
    # BA start: rotations and focals of the input, centres and points from GP
    ba = BAProblem(arr, ba_loss, optimize_focal)
    th_ba0 = torch.empty(ba.layout.total_params, dtype=torch.float64, device="cuda")
    pose = th_ba0[:7 * C].view(C, 7)
    pose[:, :4] = torch.as_tensor(np.ascontiguousarray(arr.quats, dtype=np.float64)).to("cuda")
    pose[:, 4:] = th_gp[:3 * C].view(C, 3)
    th_ba0[7 * C:7 * C + 3 * P] = th_gp[3 * C:3 * (C + P)]
    if optimize_focal:
        th_ba0[7 * C + 3 * P:] = torch.as_tensor(np.ascontiguousarray(arr.focals, dtype=np.float64)).to("cuda")
    gp.release()                      # the arena resets: BA takes the same HBM
    del th_gp
    ba.set_device_inputs(cam=cam32, pt=pt32, pixels=pix)
    ba._native_handle(ws)
    rm0 = reproj_rmse_device(ba, th_ba0)
    th_ba, rep_ba = lm_solve(ba, th_ba0, ba_config or LMConfig(max_iterations=10), ws)
    rm1 = reproj_rmse_device(ba, th_ba)
    out = ba.decode(th_ba)
    ba.release()
    rep = PipelineReport(rep_gp, rep_ba, rm0, rm1)
    if truth is not None:
        from . import metrics
        _, aligned = metrics.align(out, truth, "sim3")
        rep.center_rmse = metrics.center_rmse(aligned, truth)
        rep.rotation_auc = metrics.rotation_auc(aligned, truth, auc_thresholds)
    return out, rep
