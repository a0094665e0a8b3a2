"""CPU (no GPU): the host side of the point-sharded solver (dist.py) and the
decomposition it relies on, with a world-size-2 gloo process group.

* shard_ranges / shard_arrays: contiguous, disjoint, balanced by observation
  count, every observation on exactly one rank, order kept, points renumbered;
* scatter_theta / gather_theta round trip over gloo (all_gather_object);
* the exchange is exactly what the native path allreduces: with points
  disjoint between ranks, the damped Schur complement on the cameras, its
  right-hand side and the camera half of S*p are SUMS of per-rank terms
   -- checked with the oracle's dense algebra,
  per-rank terms summed by a gloo all_reduce in rank order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import sparsesfm_port as orc
from paper_2510_13310_b200 import dist as bd
from paper_2510_13310_b200 import synth


def small_scene(seed=0):
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=6, num_points=60, visibility_fraction=0.5,
                                                     pixel_noise_sigma=1.0, seed=seed))
    return synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)


def test_shard_ranges_balanced_disjoint():
    rng = np.random.default_rng(0)
    pt = np.sort(rng.integers(0, 1000, size=20000))
    for world in (1, 2, 3, 4, 8):
        rs = bd.shard_ranges(pt, 1000, world)
        assert rs[0][0] == 0 and rs[-1][1] == 1000
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        counts = [int(((pt >= a) & (pt < b)).sum()) for a, b in rs]
        assert sum(counts) == len(pt)
        assert max(counts) - min(counts) <= 2 * np.bincount(pt).max()


def test_shard_arrays_cover_each_observation_once():
    st = small_scene()
    seen = np.zeros(st.num_observations, dtype=int)
    for r in range(3):
        loc, (p0, p1), obs = bd.shard_arrays(st, r, 3)
        seen[obs] += 1
        assert np.all(np.diff(obs) > 0)                        # observation order kept
        assert np.array_equal(loc.pt_idx + p0, st.pt_idx[obs])  # renumbered points
        assert np.array_equal(loc.points, st.points[p0:p1])
        assert np.array_equal(loc.cam_idx, st.cam_idx[obs])
        assert loc.num_cameras == st.num_cameras
    assert np.all(seen == 1)


def prob_of(arr):
    return dict(C=arr.num_cameras, P=arr.num_points, cam=np.asarray(arr.cam_idx), pt=np.asarray(arr.pt_idx),
                pixels=arr.pixels, pps=arr.pps, dists=arr.dists, focals=arr.focals, model="pinhole",
                focal_mode=1, loss=("huber", 1.0))


def camera_schur(prob, theta, lam):
    """dense damped normal equations -> (S on the 8C camera unknowns, b_red)"""
    r, J = orc.ba_linearize(prob, theta)
    Jd = orc.ba_dense_jacobian(prob, J)
    A = Jd.T @ Jd
    A[np.diag_indices_from(A)] *= 1.0 + lam
    b = -Jd.T @ r
    C, P = prob["C"], prob["P"]
    ret = np.r_[np.arange(7 * C), 7 * C + 3 * P + np.arange(C)]
    pts = 7 * C + np.arange(3 * P)
    App = A[np.ix_(pts, pts)]
    Ainv = np.zeros_like(App)
    for j in range(P):                      # block-diagonal point blocks
        s = slice(3 * j, 3 * j + 3)
        Ainv[s, s] = np.linalg.inv(App[s, s])
    Arp = A[np.ix_(ret, pts)]
    S = A[np.ix_(ret, ret)] - Arp @ Ainv @ Arp.T
    br = b[ret] - Arp @ Ainv @ b[pts]
    return S, br


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = small_scene(seed=4)
        p = bd.ShardedBAProblem(st, rank=rank, world=world)
        th_g = p.encode_global()
        th_l = p.scatter_theta(th_g)
        assert np.array_equal(th_l, p.encode())                  # local layout == local encode
        assert np.array_equal(p.gather_theta(th_l), th_g)        # gloo round trip
        # GP: scatter / gather of centres, points and per-observation scales
        import paper_2510_13310_b200 as b2
        base = b2.fix_gauge(b2.make_rays(st, depth_mode=False, seed=0))
        gp = bd.ShardedGPProblem(base, rank=rank, world=world)
        g0 = base.initial_theta()
        g0[-base.num_obs:] = np.arange(base.num_obs) + 1.0     # distinct scales
        assert np.array_equal(gp.gather_theta(gp.scatter_theta(g0)), g0)
        assert np.array_equal(gp.initial_theta(), gp.scatter_theta(base.initial_theta()))
        loc, _, _ = bd.shard_arrays(st, rank, world)
        S, br = camera_schur(prob_of(loc), th_l, 1e-3)
        t = torch.from_numpy(np.concatenate([S.ravel(), br]))
        dist.all_reduce(t)
        if rank == 0:
            Sf, bf = camera_schur(prob_of(st), th_g, 1e-3)
            n = Sf.size
            q.put((float(np.abs(t[:n].numpy().reshape(Sf.shape) - Sf).max() / np.abs(Sf).max()),
                   float(np.abs(t[n:].numpy() - bf).max() / np.abs(bf).max())))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_schur_is_sum_of_rank_terms(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.spawn(_worker, args=(world, free_port(), q), nprocs=world, join=True)
    es, eb = q.get()
    assert es < 1e-12 and eb < 1e-12
