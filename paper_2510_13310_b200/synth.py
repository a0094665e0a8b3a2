"""Synthetic scenes, perturbation, alignment and accuracy metrics.

Array-native replay of the reference harness (sparsesfm/synth_metrics.py):
`generate_arrays` / `perturb_arrays` consume the seeded numpy generator in
exactly the reference's call sequence (synth_metrics.py:80-121, 165-191), so
the produced arrays are bit-identical to `generate()` / `perturb()` (checked
by tests/test_synth.py against committed golden digests) while avoiding one
Python object per observation. The per-point camera selection
(`rng.choice(c, k, replace=False)`, synth_metrics.py:93) is replayed by a
small native helper (csrc/synth_host.cpp) that emulates numpy's PCG64 stream;
it is self-checked against numpy on every call and falls back to the numpy
loop if the emulation ever disagrees.

This module prepares solver INPUTS on the host; it is not on the solve path.
"""

from __future__ import annotations

import ctypes as ct
from dataclasses import dataclass

import numpy as np

from .errors import DegenerateConfig, EmptyProblem, InsufficientCameras
from .scene import (PINHOLE, Camera, Observation, Point3D, Scene, SceneArrays,
                    arrays_to_scene, as_arrays, front_mask, project_many,
                    quat_from_axis_angle, quat_from_matrix, quat_multiply,
                    quat_normalize, quat_to_matrix)


@dataclass(slots=True)
class SynthConfig:
    """synth_metrics.py:16-40"""
    num_cameras: int = 10
    num_points: int = 200
    rig: str = "ring"
    radius: float = 10.0
    focal: float = 500.0
    pixel_noise_sigma: float = 0.0
    visibility_fraction: float = 1.0
    outlier_fraction: float = 0.0
    seed: int = 0

    def validate(self):
        if self.num_cameras < 2:
            raise DegenerateConfig("need at least 2 cameras")
        if self.num_points < 3:
            raise DegenerateConfig("need at least 3 points")
        if self.rig not in ("ring", "sphere"):
            raise DegenerateConfig(f"unknown rig {self.rig!r}")
        if not 0.0 < self.visibility_fraction <= 1.0:
            raise DegenerateConfig("visibility_fraction must be in (0, 1]")
        if not 0.0 <= self.outlier_fraction < 1.0:
            raise DegenerateConfig("outlier_fraction must be in [0, 1)")
        if self.radius <= 0 or self.focal <= 0 or self.pixel_noise_sigma < 0:
            raise DegenerateConfig("radius/focal/sigma out of range")


def rig_centers(cfg: SynthConfig) -> np.ndarray:
    """Ring on z=0 or Fibonacci sphere (synth_metrics.py:56-68)."""
    c = cfg.num_cameras
    if cfg.rig == "ring":
        a = 2.0 * np.pi * np.arange(c) / c
        return cfg.radius * np.stack([np.cos(a), np.sin(a), np.zeros(c)], axis=1)
    k = np.arange(c) + 0.5
    phi = np.arccos(1.0 - 2.0 * k / c)
    th = np.pi * (1.0 + np.sqrt(5.0)) * k
    return cfg.radius * np.stack([np.sin(phi) * np.cos(th), np.sin(phi) * np.sin(th), np.cos(phi)], axis=1)


def look_at_origin(center) -> np.ndarray:
    """World->camera quaternion, camera +z towards the origin (synth_metrics.py:43-53)."""
    fwd = -center / np.linalg.norm(center)
    up = np.array([0.0, 0.0, 1.0])
    if abs(fwd @ up) > 0.999:
        up = np.array([0.0, 1.0, 0.0])
    right = np.cross(up, fwd)
    right /= np.linalg.norm(right)
    return quat_from_matrix(np.stack([right, np.cross(fwd, right), fwd]))


# ---------------------------------------------------------------------------
# numpy stream replay of rng.choice(c, k, replace=False) for many points
# ---------------------------------------------------------------------------

_M64 = (1 << 64) - 1


def _host_lib():
    from . import _native
    try:
        return _native.load(required=False)
    except OSError:
        return None


def _choose_sorted_numpy(rng, c, k, p):
    out = np.stack([rng.choice(c, size=k, replace=False) for _ in range(p)]) if p else np.zeros((0, k), np.int64)
    out.sort(axis=1)
    return out


def _choose_sorted(rng, c: int, k: int, p: int) -> np.ndarray:
    lib = _host_lib()
    floyd = c <= 10000 or k <= c // 50
    if lib is None or not hasattr(lib, "ssfm_synth_choose_sorted") or not floyd or k > 64 or p == 0:
        return _choose_sorted_numpy(rng, c, k, p)
    fn = lib.ssfm_synth_choose_sorted
    fn.argtypes = [ct.POINTER(ct.c_uint64), ct.c_int64, ct.c_int32, ct.c_int32, ct.c_void_p]
    fn.restype = ct.c_int

    def run(gen, npts):
        s = gen.bit_generator.state
        st = (ct.c_uint64 * 6)(s["state"]["state"] >> 64, s["state"]["state"] & _M64,
                               s["state"]["inc"] >> 64, s["state"]["inc"] & _M64,
                               s["has_uint32"], s["uinteger"])
        out = np.empty((npts, k), dtype=np.int32)
        if fn(st, npts, c, k, out.ctypes.data_as(ct.c_void_p)) != 0:
            return None
        s["state"]["state"] = (st[0] << 64) | st[1]
        s["state"]["inc"] = (st[2] << 64) | st[3]
        s["has_uint32"] = int(st[4])
        s["uinteger"] = int(st[5])
        gen.bit_generator.state = s
        return out.astype(np.int64)

    # self-check the emulation on a copy of the stream
    probe = min(p, 8)
    g_np = np.random.Generator(type(rng.bit_generator)())
    g_np.bit_generator.state = rng.bit_generator.state
    g_c = np.random.Generator(type(rng.bit_generator)())
    g_c.bit_generator.state = rng.bit_generator.state
    a = _choose_sorted_numpy(g_np, c, k, probe)
    b = run(g_c, probe)
    if b is None or not np.array_equal(a, b) or g_np.bit_generator.state != g_c.bit_generator.state:
        return _choose_sorted_numpy(rng, c, k, p)
    out = run(rng, p)
    return out if out is not None else _choose_sorted_numpy(rng, c, k, p)


# ---------------------------------------------------------------------------
# generate / perturb
# ---------------------------------------------------------------------------

def generate_arrays(cfg: SynthConfig):
    """(truth, observed) SceneArrays, bit-identical to generate(cfg)
    (synth_metrics.py:71-133). Observations are camera-major."""
    cfg.validate()
    rng = np.random.default_rng(cfg.seed)
    c, p = cfg.num_cameras, cfg.num_points
    dirs = rng.normal(size=(p, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    radii = 0.5 * cfg.radius * rng.uniform(size=p) ** (1.0 / 3.0)
    points = dirs * radii[:, None]
    centers = rig_centers(cfg)
    quats = np.stack([look_at_origin(t) for t in centers])
    k = min(c, max(2, int(round(cfg.visibility_fraction * c))))
    cam_sel = _choose_sorted(rng, c, k, p)
    pt_of_obs = np.repeat(np.arange(p), k)
    cam_of_obs = cam_sel.ravel()
    order = np.lexsort((pt_of_obs, cam_of_obs))
    cam_of_obs = cam_of_obs[order]
    pt_of_obs = pt_of_obs[order]
    focals = np.full(c, float(cfg.focal))
    zeros2 = np.zeros((c, 2))
    n = len(cam_of_obs)
    proto = SceneArrays(quats, centers, focals, zeros2, zeros2.copy(), PINHOLE, points,
                        cam_of_obs, pt_of_obs, np.zeros((n, 2)), None)
    exact, z = project_many(proto)
    if (z <= 0).any():
        raise DegenerateConfig("rig places a point behind a camera")
    pixels = exact.copy()
    if cfg.pixel_noise_sigma > 0:
        pixels += rng.normal(0.0, cfg.pixel_noise_sigma, size=pixels.shape)
    if cfg.outlier_fraction > 0:
        n_out = int(round(cfg.outlier_fraction * n))
        idx = rng.choice(n, size=n_out, replace=False)
        half = 0.5 * cfg.focal
        pixels[idx] = rng.uniform(-half, half, size=(n_out, 2))

    def build(px):
        return SceneArrays(quats.copy(), centers.copy(), focals.copy(), np.zeros((c, 2)),
                           np.zeros((c, 2)), PINHOLE, points.copy(), cam_of_obs.copy(),
                           pt_of_obs.copy(), px, z.copy())

    return build(exact), build(pixels)


def generate(cfg: SynthConfig):
    """Object-based (truth, observed) Scenes, like synth_metrics.generate."""
    t, o = generate_arrays(cfg)
    return arrays_to_scene(t), arrays_to_scene(o)


def scene_diameter(scene) -> float:
    arr = as_arrays(scene)
    stack = np.concatenate([arr.centers.reshape(-1, 3), arr.points.reshape(-1, 3)], axis=0)
    return float(np.linalg.norm(stack.max(axis=0) - stack.min(axis=0)))


def perturb_arrays(arr: SceneArrays, rot_deg=0.0, center_frac=0.0, focal_frac=0.0,
                   point_frac=0.0, seed=0) -> SceneArrays:
    """synth_metrics.py:156-192 on a SceneArrays (bit-identical)."""
    rng = np.random.default_rng(seed)
    diam = scene_diameter(arr)
    c, p = arr.num_cameras, arr.num_points
    axes = rng.normal(size=(c, 3))
    signs = rng.choice([-1.0, 1.0], size=c)
    cdirs = rng.normal(size=(c, 3))
    cdirs /= np.linalg.norm(cdirs, axis=1, keepdims=True)
    pdirs = rng.normal(size=(p, 3))
    pdirs /= np.linalg.norm(pdirs, axis=1, keepdims=True)
    ang = np.deg2rad(rot_deg)
    quats = np.empty((c, 4))
    for i in range(c):      # per-camera loop keeps the reference's rounding
        quats[i] = quat_normalize(quat_multiply(quat_from_axis_angle(axes[i], ang), arr.quats[i]))
    out = arr.copy()
    out.quats = quats
    out.centers = arr.centers + center_frac * diam * cdirs
    out.focals = arr.focals * (1.0 + signs * focal_frac)
    out.points = arr.points + point_frac * diam * pdirs
    return out


def perturb(scene, rot_deg=0.0, center_frac=0.0, focal_frac=0.0, point_frac=0.0, seed=0):
    arr = perturb_arrays(as_arrays(scene), rot_deg, center_frac, focal_frac, point_frac, seed)
    return arr if isinstance(scene, SceneArrays) else arrays_to_scene(arr)


def trim_points_arrays(arr: SceneArrays, keep_full: int) -> SceneArrays:
    """SURVEY.md 8(d) C3 recipe: every point j >= keep_full loses its
    observation with the highest camera id (1700 / 150k / k=5 -> exactly
    680,000 observations, the BAL Ladybug shape). Observation order kept."""
    cam = np.asarray(arr.cam_idx, dtype=np.int64)
    pt = np.asarray(arr.pt_idx, dtype=np.int64)
    top = np.full(arr.num_points, -1, dtype=np.int64)
    np.maximum.at(top, pt, cam)
    keep = ~((pt >= keep_full) & (cam == top[pt]))
    out = arr.copy()
    out.cam_idx, out.pt_idx = arr.cam_idx[keep], arr.pt_idx[keep]
    out.pixels = arr.pixels[keep]
    if arr.depths is not None:
        out.depths = arr.depths[keep]
    return out


def outlier_mask(truth, observed, sigma: float) -> np.ndarray:
    t, o = as_arrays(truth), as_arrays(observed)
    return np.linalg.norm(t.pixels - o.pixels, axis=1) > max(6.0 * sigma, 1.0)


# ---------------------------------------------------------------------------
# alignment and metrics (synth_metrics.py:199-325)
# ---------------------------------------------------------------------------

@dataclass(slots=True)
class Alignment:
    kind: str
    rotation: np.ndarray
    translation: np.ndarray
    scale: float

    def apply(self, x):
        return self.scale * (np.asarray(x) @ self.rotation.T) + self.translation


def align(estimate, truth, kind: str = "sim3"):
    """Umeyama registration of camera centres; returns (Alignment, aligned)."""
    if kind not in ("sim3", "se3"):
        raise ValueError(f"unknown alignment kind {kind!r}")
    est, tru = as_arrays(estimate), as_arrays(truth)
    n = est.num_cameras
    if n != tru.num_cameras:
        raise InsufficientCameras("camera counts differ")
    if kind == "sim3" and n < 3:
        raise InsufficientCameras("sim3 alignment needs at least 3 cameras")
    if n < 2:
        raise InsufficientCameras("alignment needs at least 2 cameras")
    x, y = est.centers, tru.centers
    mx, my = x.mean(axis=0), y.mean(axis=0)
    xc, yc = x - mx, y - my
    u, d, vt = np.linalg.svd(yc.T @ xc / n)
    sgn = np.ones(3)
    if np.linalg.det(u) * np.linalg.det(vt) < 0:
        sgn[2] = -1.0
    rot = u @ np.diag(sgn) @ vt
    scale = 1.0
    if kind == "sim3":
        scale = float((d * sgn).sum()) / (float((xc * xc).sum()) / n)
        if scale <= 0:
            raise InsufficientCameras("degenerate similarity (non-positive scale)")
    al = Alignment(kind, rot, my - scale * rot @ mx, scale)
    rq = quat_from_matrix(rot)
    rq_c = np.array([rq[0], -rq[1], -rq[2], -rq[3]])
    out = est.copy()
    out.quats = np.stack([quat_normalize(quat_multiply(q, rq_c)) for q in est.quats]) if n else est.quats
    out.centers = al.apply(est.centers)
    out.points = al.apply(est.points)
    return al, (out if isinstance(estimate, SceneArrays) else arrays_to_scene(out))


def center_rmse(estimate, truth) -> float:
    a, b = as_arrays(estimate).centers, as_arrays(truth).centers
    return float(np.sqrt(np.mean(np.sum((a - b) ** 2, axis=1))))


def camera_rotation_errors_deg(estimate, truth) -> np.ndarray:
    qe = as_arrays(estimate).quats
    qt = as_arrays(truth).quats
    qe = qe / np.linalg.norm(qe, axis=1, keepdims=True)
    qt = qt / np.linalg.norm(qt, axis=1, keepdims=True)
    return np.rad2deg(2.0 * np.arccos(np.minimum(np.abs(np.sum(qe * qt, axis=1)), 1.0)))


def rotation_auc(estimate, truth, thresholds_deg) -> dict:
    """Pairwise relative-rotation AUC (0-100) over all camera pairs."""
    qe, qt = as_arrays(estimate).quats, as_arrays(truth).quats
    c = len(qe)
    if c < 2 or c != len(qt):
        raise InsufficientCameras("need two scenes with >= 2 matching cameras")
    qe = qe / np.linalg.norm(qe, axis=1, keepdims=True)
    qt = qt / np.linalg.norm(qt, axis=1, keepdims=True)
    ii, jj = np.triu_indices(c, k=1)

    def rel(q):
        aw, av = q[ii, 0], q[ii, 1:]
        bw, bv = q[jj, 0], -q[jj, 1:]
        w = aw * bw - np.sum(av * bv, axis=1)
        v = aw[:, None] * bv + bw[:, None] * av + np.cross(av, bv)
        return np.concatenate([w[:, None], v], axis=1)

    dots = np.clip(np.abs(np.sum(rel(qe) * rel(qt), axis=1)), 0.0, 1.0)
    err = np.rad2deg(2.0 * np.arccos(dots))
    return {float(t): float(np.mean(np.maximum(0.0, 1.0 - err / t)) * 100.0) for t in thresholds_deg}


def reproj_rmse(scene) -> float:
    arr = as_arrays(scene)
    if arr.num_observations == 0:
        raise EmptyProblem("no observations to evaluate")
    uv, z = project_many(arr)
    m = front_mask(arr.model_tag, z)
    if not m.any():
        raise EmptyProblem("every observation is behind its camera")
    d = uv[m] - arr.pixels[m]
    return float(np.sqrt(np.mean(np.sum(d * d, axis=1))))
