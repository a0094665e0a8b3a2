"""Point-sharded multi-GPU bundle adjustment.

One process per GPU (torchrun), or several handles in one process on one
device (tests). The observations are sharded by point ownership:

* points are split into `world` contiguous ranges balanced by observation
  count (`shard_ranges`); rank r owns its points and every observation of
  them, so point elimination, point back-substitution and the point half of
  the gradient are local;
* camera parameters (poses, focals) and the camera-space PCG vectors are
  replicated; the camera-side sums (J^T J camera blocks, J^T r, Schur
  preconditioner blocks and, every CG iteration, the camera half of S*p) and
  the scalar reductions (cost, |g|^2, max|g|, status) are exchanged through
  peer memory by the native library (csrc/comm.cuh) -- in-kernel for S*p.

Replicated values are combined in rank order on every rank, so every rank
holds bitwise-identical camera parameters and takes the same LM decisions;
the LM report is identical on all ranks. Results differ from a single-GPU
solve only by summation order (bitwise stable per GPU count).

The reference (sparsesfm) has no multi-GPU path; this module extends its
`BAProblem` / `GPProblem` / `lm_solve` API (ba.py:35-36, gp.py:33-35,
lm.py:727-728) without changing it: a `ShardedBAProblem` / `ShardedGPProblem`
is a problem over the rank's shard, `lm_solve` is called on every rank with
the rank's local theta.
"""

from __future__ import annotations

import ctypes as ct

import numpy as np

from . import _native
from .ba import BAProblem, _DeviceProblem
from .gp import GPProblem
from .scene import SceneArrays, as_arrays


def shard_ranges(pt_idx, num_points: int, world: int):
    """Contiguous point ranges [(p0, p1)] per rank, balanced by observation
    count: rank r ends at the first point whose prefix observation count
    reaches r+1 / world of the total. Deterministic, empty ranges allowed."""
    if world < 1:
        raise ValueError("world must be >= 1")
    counts = np.bincount(np.asarray(pt_idx, dtype=np.int64), minlength=num_points)
    csum = np.concatenate([[0], np.cumsum(counts)])
    total = int(csum[-1])
    bounds = [0]
    for r in range(1, world):
        target = (r * total) // world
        p = int(np.searchsorted(csum, target, side="left"))
        bounds.append(min(max(p, bounds[-1]), num_points))
    bounds.append(num_points)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


def shard_arrays(arr: SceneArrays, rank: int, world: int):
    """(local SceneArrays, (p0, p1), observation indices) of one rank: every
    camera, points [p0, p1) renumbered from 0, their observations in the
    original observation order."""
    p0, p1 = shard_ranges(arr.pt_idx, arr.num_points, world)[rank]
    pt = np.asarray(arr.pt_idx, dtype=np.int64)
    obs = np.nonzero((pt >= p0) & (pt < p1))[0]
    local = SceneArrays(arr.quats, arr.centers, arr.focals, arr.pps, arr.dists, arr.model_tag,
                        arr.points[p0:p1], np.asarray(arr.cam_idx)[obs], pt[obs] - p0,
                        arr.pixels[obs], None if arr.depths is None else arr.depths[obs])
    return local, (p0, p1), obs


class _Sharded:
    """Connection plumbing shared by the sharded BA and GP problems."""

    def _init_shard(self, rank, world, group, comm):
        if rank is None or world is None:
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        self.rank, self.world, self.group, self.comm = rank, world, group, comm
        self._connected = world == 1
        return rank, world

    def _connect_torch(self, h):
        if self.world > 1 and self.comm == "torch":
            import torch.distributed as dist
            lib = _native.load()
            ih = (ct.c_char * 64)()
            _native.check(lib.ssfm_comm_init(ct.c_void_p(h.ptr), self.rank, self.world, ih, None))
            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(ih), group=self.group)
            _native.check(lib.ssfm_comm_connect(ct.c_void_p(h.ptr), ct.c_char_p(b"".join(handles)), None))
            self._connected = True

    def _create(self, arena=None):
        h = super()._create(arena)
        self._native_ptr = h
        self._connect_torch(h)
        return h

    def _enter_collective(self):
        """Before every native call that exchanges with the peers. Several
        shards on one device (comm="local"): each shard first finishes its
        torch-side work on its stream, then all shards enter together. The
        exchanges spin on the device, and a torch allocation, device-to-device
        copy or memset issued by one shard's thread while a peer's kernel
        already waits in an exchange is an implicit synchronisation point
        between the streams: that shard's kernels would queue behind the
        peer's waiting kernel. (One process per GPU has no such hazard.)"""
        bar = getattr(self, "_local_barrier", None)
        if bar is not None:
            import torch
            torch.cuda.current_stream().synchronize()
            bar.wait(timeout=600)

    def _native_handle(self, workspace=None):
        h = super()._native_handle(workspace)
        if not self._connected:
            raise RuntimeError("sharded problem not connected: call connect_local(problems) first")
        return h

    def _all_gather(self, obj, shards, pick):
        """every rank's `pick(problem, theta)` in rank order: torch collective,
        or from `shards` = [(problem, theta)] for comm='local'."""
        if shards is not None:
            return [pick(p, th if isinstance(th, np.ndarray) else th.detach().cpu().numpy())
                    for p, th in sorted(shards, key=lambda t: t[0].rank)]
        if self.world == 1:
            return [obj]
        import torch.distributed as dist
        out = [None] * self.world
        dist.all_gather_object(out, obj, group=self.group)
        return out


class ShardedBAProblem(_Sharded, BAProblem):
    """BAProblem over this rank's point shard (see module docstring).

    comm="torch": ranks are torch.distributed ranks (one process per GPU);
    the exchange regions are connected on first use via CUDA IPC handles
    all-gathered over `group`. comm="local": several shards in one process
    on one device; call `connect_local(problems)` before solving.
    Every computing call (cost, linearize, lm_solve) is collective.
    """

    def __init__(self, scene, loss=None, optimize_focal: bool = True, shared_focal: bool = False,
                 rank: int | None = None, world: int | None = None, group=None, comm: str = "torch"):
        arr = as_arrays(scene)
        rank, world = self._init_shard(rank, world, group, comm)
        local, (p0, p1), obs = shard_arrays(arr, rank, world)
        if local.num_observations == 0:
            raise ValueError(f"rank {rank} owns no observations (world {world} too large for this scene)")
        BAProblem.__init__(self, local, loss, optimize_focal, shared_focal)
        self._connected = world == 1
        self.global_arr = arr
        self.point_range = (p0, p1)
        self.obs_index = obs

    # -- theta between the global layout and this rank's shard ---------------
    def scatter_theta(self, theta_global) -> np.ndarray:
        """This rank's local theta [7C | 3 P_local | focals] from a global one."""
        th = np.asarray(theta_global, dtype=np.float64)
        c, P = self.num_cameras, self.global_arr.num_points
        p0, p1 = self.point_range
        parts = [th[:7 * c], th[7 * c + 3 * p0:7 * c + 3 * p1]]
        if self.optimize_focal:
            parts.append(th[7 * c + 3 * P:])
        return np.concatenate(parts)

    def gather_theta(self, theta_local, shards=None) -> np.ndarray:
        """Global theta from every rank's local theta (collective for
        comm="torch"; for comm="local" pass `shards` = [(problem, theta)])."""
        if not isinstance(theta_local, np.ndarray):
            theta_local = theta_local.detach().cpu().numpy()
        c = self.num_cameras
        pts = lambda p, th: th[7 * c:7 * c + 3 * p.num_points]  # noqa: E731
        parts = [theta_local[:7 * c], *self._all_gather(pts(self, theta_local), shards, pts)]
        if self.optimize_focal:
            parts.append(theta_local[7 * c + 3 * self.num_points:])
        return np.concatenate(parts)

    def encode_global(self) -> np.ndarray:
        return BAProblem(self.global_arr, self.loss, self.optimize_focal, self.shared_focal).encode()


class ShardedGPProblem(_Sharded, GPProblem):
    """GPProblem over this rank's point shard: every camera (replicated
    centres, camera-0 gauge), points [p0, p1) renumbered, their observations
    and per-observation scales. The mean-scale gauge of post_step
    (gp.py:130-147) is taken over every rank's scales (one exchange of
    (sum, count))."""

    def __init__(self, base: GPProblem, rank: int | None = None, world: int | None = None, group=None,
                 comm: str = "torch"):
        rank, world = self._init_shard(rank, world, group, comm)
        p0, p1 = shard_ranges(base.pt_idx, base.num_points, world)[rank]
        obs = np.nonzero((base.pt_idx >= p0) & (base.pt_idx < p1))[0]
        if len(obs) == 0:
            raise ValueError(f"rank {rank} owns no observations (world {world} too large for this problem)")
        GPProblem.__init__(self, base.rays[obs], base.fixed_rotations, base.cam_idx[obs], base.pt_idx[obs] - p0,
                           p1 - p0, base.loss, base.depth_mode,
                           None if base.depths is None else base.depths[obs], base.seed)
        self._connected = world == 1
        self._gauge_fixed = base.gauge_fixed
        self.base = base
        self.point_range = (p0, p1)
        self.obs_index = obs

    def scatter_theta(self, theta_global) -> np.ndarray:
        th = np.asarray(theta_global, dtype=np.float64)
        c, P = self.num_cameras, self.base.num_points
        p0, p1 = self.point_range
        parts = [th[:3 * c], th[3 * c + 3 * p0:3 * c + 3 * p1]]
        if not self.depth_mode:
            parts.append(th[3 * (c + P):][self.obs_index])
        return np.concatenate(parts)

    def initial_theta(self) -> np.ndarray:
        """The base problem's seeded initial theta (gp.py:71-80), this rank's part."""
        return self.scatter_theta(self.base.initial_theta())

    def gather_theta(self, theta_local, shards=None) -> np.ndarray:
        if not isinstance(theta_local, np.ndarray):
            theta_local = theta_local.detach().cpu().numpy()
        c, P, N = self.num_cameras, self.base.num_points, self.base.num_obs
        pick = lambda p, th: (th[3 * c:3 * (c + p.num_points)],  # noqa: E731
                              None if p.depth_mode else (p.obs_index, th[3 * (c + p.num_points):]))
        got = self._all_gather(pick(self, theta_local), shards, pick)
        parts = [theta_local[:3 * c], *[g[0] for g in got]]
        if not self.depth_mode:
            sc = np.empty(N)
            for _, (idx, vals) in got:
                sc[idx] = vals
            parts.append(sc)
        return np.concatenate(parts)


def connect_local(problems) -> None:
    """Connect several sharded problems (ranks 0..R-1 of one problem) living in
    this process -- on one device, or on several (peer access is enabled
    between them): exchange regions are plain device pointers. Their collective calls must then run concurrently (one host
    thread per problem) and their PCG grids must fit the device together
    (set SSFM_PCG_SMS before the handles are created). The process needs
    CUDA_MODULE_LOADING=EAGER (set before CUDA initialises): a kernel loaded
    lazily at its first launch waits for the device, i.e. for a peer shard's
    kernel spinning in an exchange."""
    import os
    import warnings
    if os.environ.get("CUDA_MODULE_LOADING", "LAZY").upper() != "EAGER":
        warnings.warn("connect_local: set CUDA_MODULE_LOADING=EAGER before CUDA initialises; with lazy "
                      "module loading the first exchange of same-device shards can stall", RuntimeWarning)
    import threading
    lib = _native.load()
    world = len(problems)
    regions = (ct.c_void_p * world)()
    for p in problems:
        if p.world != world or p.comm != "local":
            raise ValueError("connect_local needs comm='local' problems of one world")
    # shards on several devices of this process: direct peer access both ways
    devs = sorted({int(lib.ssfm_handle_device(ct.c_void_p(_DeviceProblem._native_handle(p).ptr))) for p in problems})
    for a in devs:
        for b in devs:
            if a != b:
                _native.check(lib.ssfm_enable_peer_access(a, b))
    for p in problems:
        h = _DeviceProblem._native_handle(p)
        reg = ct.c_void_p(0)
        _native.check(lib.ssfm_comm_init(ct.c_void_p(h.ptr), p.rank, world, None, ct.byref(reg)))
        regions[p.rank] = reg.value
    for p in problems:
        h = _DeviceProblem._native_handle(p)
        _native.check(lib.ssfm_comm_connect(ct.c_void_p(h.ptr), None, regions))
        p._connected = True
    bar = threading.Barrier(world)   # the shards enter each collective call together (_enter_collective)
    for p in problems:
        p._local_barrier = bar


def run_ba_sharded(scene, loss=None, config=None, optimize_focal: bool = True, group=None):
    """run_ba (ba.py:264-271) over the torch.distributed ranks: every rank
    returns the full solved scene (decoded from the gathered theta) and the
    (identical) SolveReport."""
    from .lm import lm_solve
    prob = ShardedBAProblem(scene, loss, optimize_focal, group=group)
    th0 = prob.encode()
    th, rep = lm_solve(prob, th0, config)
    full = prob.gather_theta(th)
    g = BAProblem(prob.global_arr, prob.loss, optimize_focal)
    return g.decode(full), rep


def run_gp_sharded(scene, depth_mode: bool = False, loss=None, config=None, seed: int = 0, group=None):
    """run_gp (gp.py:204-218) over the torch.distributed ranks: every rank
    returns the gathered global theta and the (identical) SolveReport."""
    from .gp import fix_gauge, make_rays
    from .lm import lm_solve
    base = fix_gauge(make_rays(scene, depth_mode, loss, seed))
    prob = ShardedGPProblem(base, group=group)
    th, rep = lm_solve(prob, prob.initial_theta(), config)
    return prob.gather_theta(th), rep
