"""Bundle adjustment problem (drop-in for sparsesfm/ba.py).

Residual of observation (i, j): r = sqrt(w) (project(camera_i, X_j) - x_ij),
w the Huber IRLS weight frozen per linearization; observations behind the
camera are masked (ba.py:1-11). Everything per observation is evaluated on
the device (csrc/ba.cuh, csrc/ba_kernels.cuh); `linearize` materialises the
reference-layout BlockSparseJacobian only as a parity / inspection path.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import EmptyProblem
from .lm import LMConfig, SolveReport, Workspace, lm_solve
from .scene import (MODEL_CODE, RobustLoss, SceneArrays, arrays_to_scene, as_arrays)
from .sparse_block import BlockLayout, BlockSparseJacobian


def _torch():
    from .lm import _torch as t
    return t()


def _index_dev(torch, idx):
    """int32 device copy of an index array: integer inputs are copied as they
    are and narrowed on the device (a host-side astype of 20M indices costs
    more than moving the wider type)."""
    x = np.asarray(idx)
    if x.dtype.kind in "iu" and x.flags.c_contiguous:
        return torch.from_numpy(x).to("cuda").to(torch.int32)
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int32)).to("cuda")


class _DeviceProblem:
    """Common plumbing of the native problems: lazy handle creation on the
    current CUDA device, theta transfer, cost / linearize / post_step."""

    _native_ptr = None

    def _create(self, arena=None):  # pragma: no cover - abstract
        raise NotImplementedError

    def _enter_collective(self):
        """Hook before each native call (sharded problems synchronise their
        local shards here, dist._Sharded._enter_collective)."""

    def _native_handle(self, workspace=None):
        """The device problem, created on first use; with a Workspace (lm_solve,
        run_ba / run_gp) it is created in the workspace's device arena."""
        if self._native_ptr is None:
            self._native_ptr = self._create(workspace.device_arena() if workspace is not None else None)
        return self._native_ptr

    def _device_input(self, torch, key, make):
        """a device copy of an input array: the caller's (set_device_inputs) or a fresh upload"""
        d = getattr(self, "_dev_inputs", None)
        if d is not None and d.get(key) is not None:
            return d[key]
        return make()

    def set_device_inputs(self, **tensors) -> None:
        """Hand the problem device-resident copies of its per-observation
        inputs (cam=int32, pt=int32 [N] CUDA tensors; pixels [N,2] / rays [N,3]
        float64) so handle creation copies device to device instead of
        uploading from the host (the GP -> BA pipeline)."""
        self._dev_inputs = dict(tensors)

    @staticmethod
    def _create_call(lib, kind, desc, arena, stream, out):
        if arena is None:
            fn = lib.ssfm_create_ba if kind == "ba" else lib.ssfm_create_gp
            return fn(ct.byref(desc), stream, ct.byref(out))
        fn = lib.ssfm_create_ba_in if kind == "ba" else lib.ssfm_create_gp_in
        return fn(ct.byref(desc), ct.c_void_p(arena.ptr), stream, ct.byref(out))

    @staticmethod
    def _theta_dev(torch, theta):
        if isinstance(theta, torch.Tensor):
            return theta.detach().to(device="cuda", dtype=torch.float64).contiguous()
        return torch.as_tensor(np.ascontiguousarray(theta, dtype=np.float64)).to("cuda")

    def cost(self, theta) -> float:
        torch = _torch()
        from .lm import _stream
        t = self._theta_dev(torch, theta)
        out = ct.c_double(0.0)
        self._enter_collective()
        _native.check(_native.load().ssfm_cost(ct.c_void_p(self._native_handle().ptr),
                                               ct.c_void_p(t.data_ptr()), ct.byref(out),
                                               _stream(torch)))
        return float(out.value)

    def _linearize_dev(self, theta, want_J=True):
        torch = _torch()
        from .lm import _stream
        t = self._theta_dev(torch, theta)
        h = self._native_handle()
        r = torch.empty(self.layout.total_residuals, dtype=torch.float64, device="cuda")
        J = torch.empty(self.jac_width * self.num_obs if want_J else 1, dtype=torch.float64, device="cuda")
        g = torch.empty(self.layout.total_params, dtype=torch.float64, device="cuda")
        gmax = ct.c_double(0.0)
        self._enter_collective()
        _native.check(_native.load().ssfm_linearize(
            ct.c_void_p(h.ptr), ct.c_void_p(t.data_ptr()), ct.c_void_p(r.data_ptr()),
            ct.c_void_p(J.data_ptr()) if want_J else None, ct.c_void_p(g.data_ptr()),
            ct.byref(gmax), _stream(torch)))
        return r, J, g, float(gmax.value)

    def linearize(self, theta):
        """(weighted residuals, BlockSparseJacobian) in the reference layout."""
        r, J, _, _ = self._linearize_dev(theta)
        jac = self.jac
        jac.data[:] = J.cpu().numpy()
        self._residuals = r.cpu().numpy()
        return self._residuals, jac

    def gradient(self, theta) -> np.ndarray:
        """J^T r in theta layout (jtr of the reference linearization)."""
        _, _, g, _ = self._linearize_dev(theta, want_J=False)
        return g.cpu().numpy()

    def post_step(self, theta):
        torch = _torch()
        from .lm import _stream
        is_t = isinstance(theta, torch.Tensor)
        t = self._theta_dev(torch, theta).clone()
        self._enter_collective()
        _native.check(_native.load().ssfm_post_step(ct.c_void_p(self._native_handle().ptr),
                                                    ct.c_void_p(t.data_ptr()), _stream(torch)))
        return t if is_t else t.cpu().numpy()

    @property
    def jac(self) -> BlockSparseJacobian:
        if getattr(self, "_jac", None) is None:
            self._jac = BlockSparseJacobian.allocate(self.layout, self._res_ids(), self._param_ids())
        return self._jac

    def release(self, trim: bool = False) -> None:
        """Destroy the device handle now (instead of at garbage collection).
        Its device blocks go to the library's reuse cache (ssfm_destroy), so
        the next problem of the same shape skips cudaMalloc; trim=True returns
        them to the CUDA allocator instead (also: _native.trim_cache())."""
        h = self._native_ptr
        self._native_ptr = None
        if h is not None and h.ptr:
            _native.load().ssfm_destroy(ct.c_void_p(h.ptr))
            h.ptr = 0
        if trim:
            _native.trim_cache()

    def device_bytes(self) -> int:
        return int(_native.load().ssfm_device_bytes(ct.c_void_p(self._native_handle().ptr)))

    def export_pattern(self):
        """Reference-equivalent integer structures computed on the device:
        dict(obs_pt_order, obs_cam_order, off_keys, schur_slots)."""
        torch = _torch()
        from .lm import _stream
        h = self._native_handle()
        lib = _native.load()
        n = self.num_obs
        pt = torch.empty(n, dtype=torch.int32, device="cuda")
        cm = torch.empty(n, dtype=torch.int32, device="cuda")
        nk, ns = ct.c_int64(0), ct.c_int64(0)
        _native.check(lib.ssfm_export_pattern(ct.c_void_p(h.ptr), ct.c_void_p(pt.data_ptr()),
                                              ct.c_void_p(cm.data_ptr()), None, 0, ct.byref(nk),
                                              None, 0, ct.byref(ns), _stream(torch)))
        keys = torch.empty(max(nk.value, 1) * 2, dtype=torch.int32, device="cuda")
        slots = torch.empty(max(ns.value, 1) * 2, dtype=torch.int32, device="cuda")
        _native.check(lib.ssfm_export_pattern(ct.c_void_p(h.ptr), None, None,
                                              ct.c_void_p(keys.data_ptr()), nk.value, ct.byref(nk),
                                              ct.c_void_p(slots.data_ptr()), ns.value, ct.byref(ns),
                                              _stream(torch)))
        return {"obs_pt_order": pt.cpu().numpy(), "obs_cam_order": cm.cpu().numpy(),
                "off_keys": keys[:2 * nk.value].view(-1, 2).cpu().numpy(),
                "schur_slots": slots[:2 * ns.value].view(-1, 2).cpu().numpy()}


class BAProblem(_DeviceProblem):
    """Reprojection residual/Jacobian provider (ba.py:27-197).

    Parameter layout: per camera a 7-wide pose block (q, t), one 3-wide block
    per point, then the focal blocks (one per camera, one shared, or none).
    """

    def __init__(self, scene, loss: RobustLoss | None = None, optimize_focal: bool = True,
                 shared_focal: bool = False):
        arr = as_arrays(scene)
        if arr.num_observations == 0:
            raise EmptyProblem("scene has no observations")
        self._scene_is_arrays = isinstance(scene, SceneArrays)
        self.loss = loss or RobustLoss("trivial")
        self.optimize_focal = bool(optimize_focal)
        self.shared_focal = bool(shared_focal)
        self.arr = arr
        c, p, n = arr.num_cameras, arr.num_points, arr.num_observations
        self.num_cameras, self.num_points, self.num_obs = c, p, n
        runs = [("camera_pose", c), ("point", p)]
        if optimize_focal:
            runs.append(("focal", 1 if shared_focal else c))
        self.layout = BlockLayout.from_runs(runs, 2, n)
        self.per_obs = 2 + int(optimize_focal)
        self.jac_width = 20 + 2 * int(optimize_focal)
        self._jac = None
        self._native_ptr = None

    def _res_ids(self):
        return np.repeat(np.arange(self.num_obs, dtype=np.int32), self.per_obs)

    def _param_ids(self):
        c, p = self.num_cameras, self.num_points
        ids = np.empty((self.num_obs, self.per_obs), dtype=np.int32)
        ids[:, 0] = self.arr.cam_idx
        ids[:, 1] = c + self.arr.pt_idx
        if self.optimize_focal:
            ids[:, 2] = c + p if self.shared_focal else c + p + self.arr.cam_idx
        return ids.ravel()

    def _create(self, arena=None):
        torch = _torch()
        from .lm import _stream
        a = self.arr
        dev = lambda x, dt: torch.as_tensor(np.ascontiguousarray(x, dtype=dt)).to("cuda")  # noqa: E731
        cam = self._device_input(torch, "cam", lambda: _index_dev(torch, a.cam_idx))
        pt = self._device_input(torch, "pt", lambda: _index_dev(torch, a.pt_idx))
        pix = self._device_input(torch, "pixels", lambda: dev(a.pixels, np.float64))
        pps = dev(a.pps, np.float64)
        dists = dev(a.dists, np.float64)
        foc = dev(a.focals, np.float64)
        desc = _native.BADescC(
            a.num_cameras, a.num_points, a.num_observations, MODEL_CODE.get(a.model_tag, 0),
            int(self.optimize_focal), int(self.shared_focal), self.loss.code, float(self.loss.delta),
            cam.data_ptr(), pt.data_ptr(), pix.data_ptr(), pps.data_ptr(), dists.data_ptr(),
            foc.data_ptr())
        out = ct.c_void_p(0)
        _native.check(self._create_call(_native.load(), "ba", desc, arena, _stream(torch), out))
        torch.cuda.current_stream().synchronize()
        return _native.Handle(out.value, keepalive=(arena,) if arena is not None else ())

    # -- theta packing (ba.py:68-107) ----------------------------------------
    def encode(self) -> np.ndarray:
        c, p = self.num_cameras, self.num_points
        theta = np.empty(self.layout.total_params)
        pose = theta[:7 * c].reshape(c, 7)
        pose[:, :4] = self.arr.quats
        pose[:, 4:] = self.arr.centers
        theta[7 * c:7 * c + 3 * p] = self.arr.points.ravel()
        if self.optimize_focal:
            off = 7 * c + 3 * p
            if self.shared_focal:
                theta[off] = self.arr.focals[0]
            else:
                theta[off:off + c] = self.arr.focals
        return theta

    def _views(self, theta):
        c, p = self.num_cameras, self.num_points
        theta = np.asarray(theta, dtype=np.float64)
        pose = theta[:7 * c].reshape(c, 7)
        pts = theta[7 * c:7 * c + 3 * p].reshape(p, 3)
        if self.optimize_focal:
            off = 7 * c + 3 * p
            foc = np.full(c, theta[off]) if self.shared_focal else theta[off:off + c]
        else:
            foc = self.arr.focals
        return pose[:, :4], pose[:, 4:], pts, foc

    def decode(self, theta):
        if not isinstance(theta, np.ndarray):
            theta = theta.detach().cpu().numpy()
        q, t, x, f = self._views(theta)
        out = self.arr.copy()
        out.quats = q / np.linalg.norm(q, axis=1, keepdims=True)
        out.centers = t.copy()
        out.points = x.copy()
        out.focals = np.array(f, dtype=np.float64)
        return out if self._scene_is_arrays else arrays_to_scene(out)


def ba_residuals(problem: BAProblem, theta) -> np.ndarray:
    """Weighted, masked reprojection residuals (ba.py:200-203)."""
    r, _, _, _ = problem._linearize_dev(theta, want_J=False)
    return r.cpu().numpy()


def ba_jacobian(problem: BAProblem, theta) -> BlockSparseJacobian:
    _, j = problem.linearize(theta)
    return j


@dataclass(slots=True)
class PruneRemap:
    camera_map: np.ndarray
    point_map: np.ndarray
    observation_mask: np.ndarray


def _prune_device(cam, pt, c, p):
    """(camera_map, point_map, observation mask) from ssfm_prune (the fixed
    point of ba.py:234-243 on the device, bit-identical); None without a GPU."""
    try:
        import torch
    except ImportError:   # pragma: no cover
        return None
    if not torch.cuda.is_available() or _native.load(required=False) is None:
        return None
    from .lm import _stream
    n = len(cam)
    cam_d = torch.as_tensor(cam.astype(np.int32)).cuda()
    pt_d = torch.as_tensor(pt.astype(np.int32)).cuda()
    cmap = torch.empty(max(c, 1), dtype=torch.int32, device="cuda")
    pmap = torch.empty(max(p, 1), dtype=torch.int32, device="cuda")
    mask = torch.empty(max(n, 1), dtype=torch.uint8, device="cuda")
    nc, npt, no = ct.c_int32(0), ct.c_int32(0), ct.c_int64(0)
    _native.check(_native.load().ssfm_prune(n, ct.c_void_p(cam_d.data_ptr()), ct.c_void_p(pt_d.data_ptr()), c, p,
                                            ct.c_void_p(cmap.data_ptr()), ct.c_void_p(pmap.data_ptr()),
                                            ct.c_void_p(mask.data_ptr()), ct.byref(nc), ct.byref(npt),
                                            ct.byref(no), _stream(torch)))
    return (cmap[:c].cpu().numpy().astype(np.int64), pmap[:p].cpu().numpy().astype(np.int64),
            mask[:n].cpu().numpy().astype(bool))


def prune(scene):
    """Drop points seen by < 2 cameras and cameras left without observations,
    to a fixed point (ba.py:223-261). On the device (ssfm_prune) when a GPU is
    present; the host restatement below serves CPU-only use."""
    arr = as_arrays(scene)
    c, p = arr.num_cameras, arr.num_points
    cam, pt = arr.cam_idx.astype(np.int64), arr.pt_idx.astype(np.int64)
    dev = _prune_device(cam, pt, c, p)
    if dev is not None:
        cmap, pmap, obs_ok = dev
        cam_ok, pt_ok = cmap >= 0, pmap >= 0
    else:
        cmap, pmap, obs_ok, cam_ok, pt_ok = _prune_host(cam, pt, c, p)
    return _prune_apply(scene, arr, cmap, pmap, obs_ok, cam_ok, pt_ok)


def _prune_host(cam, pt, c, p):
    cam_ok = np.ones(c, dtype=bool)
    pt_ok = np.ones(p, dtype=bool)
    while True:
        obs_ok = cam_ok[cam] & pt_ok[pt] if len(cam) else np.zeros(0, dtype=bool)
        drop_pt = pt_ok & (np.bincount(pt[obs_ok], minlength=p) < 2)
        drop_cam = cam_ok & (np.bincount(cam[obs_ok], minlength=c) == 0)
        if not drop_pt.any() and not drop_cam.any():
            break
        pt_ok &= ~drop_pt
        cam_ok &= ~drop_cam
    if not obs_ok.any():
        raise EmptyProblem("pruning removed every observation")
    cmap = np.full(c, -1, dtype=np.int64)
    cmap[cam_ok] = np.arange(int(cam_ok.sum()))
    pmap = np.full(p, -1, dtype=np.int64)
    pmap[pt_ok] = np.arange(int(pt_ok.sum()))
    return cmap, pmap, obs_ok, cam_ok, pt_ok


def _prune_apply(scene, arr, cmap, pmap, obs_ok, cam_ok, pt_ok):
    cam, pt = arr.cam_idx.astype(np.int64), arr.pt_idx.astype(np.int64)
    c, p = arr.num_cameras, arr.num_points
    out = SceneArrays(arr.quats[cam_ok], arr.centers[cam_ok], arr.focals[cam_ok], arr.pps[cam_ok],
                      arr.dists[cam_ok], arr.model_tag, arr.points[pt_ok], cmap[cam[obs_ok]],
                      pmap[pt[obs_ok]], arr.pixels[obs_ok],
                      None if arr.depths is None else arr.depths[obs_ok])
    remap = PruneRemap(cmap, pmap, obs_ok)
    if isinstance(scene, SceneArrays):
        return out, remap
    # keep the caller's Camera/Point objects (the reference reuses them)
    from .scene import Observation, Scene
    obs = [Observation(int(cmap[o.camera_id]), int(pmap[o.point_id]), o.pixel, o.depth)
           for k, o in enumerate(scene.observations) if obs_ok[k]]
    return Scene([scene.cameras[i] for i in range(c) if cam_ok[i]],
                 [scene.points[j] for j in range(p) if pt_ok[j]], obs), remap


def run_ba(scene, loss: RobustLoss | None = None, config: LMConfig | None = None,
           optimize_focal: bool = True, shared_focal: bool = False,
           workspace: Workspace | None = None):
    """Encode, optimise on the device, decode (ba.py:264-271)."""
    problem = BAProblem(scene, loss, optimize_focal, shared_focal)
    theta, report = lm_solve(problem, problem.encode(), config, workspace)
    return problem.decode(theta), report
