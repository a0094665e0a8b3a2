"""GPU: the Workspace's device arena (lm.py:86-101 Workspace; csrc ssfm_arena)
and the device-resident GP -> BA hand-off of run_global_sfm.

* problems created through lm_solve(..., workspace) allocate from the arena;
  after the first stage is released the next stage reuses its HBM (no new
  cudaMalloc when it fits; one added chunk when it does not, coalesced on the
  next reset);
* results are bitwise identical to solves outside an arena;
* the arena refuses to be destroyed while a handle lives in it;
* run_global_sfm (one arena, rays and indices on the device, BA started from
  the GP solution on the device) takes the same trajectory as run_gp + run_ba
  from host arrays.
"""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import _native, synth

pytestmark = pytest.mark.gpu


def observed(C=40, P=3000, k=5, seed=4):
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=C, num_points=P, visibility_fraction=k / C,
                                                     pixel_noise_sigma=1.0, seed=seed))
    return obs


def test_arena_reuse_across_stages_is_bitwise_neutral(gpu):
    obs = observed()
    st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    cfg = b2.LMConfig(max_iterations=6)
    ref_gp = b2.fix_gauge(b2.make_rays(obs, loss=b2.RobustLoss("huber", 0.1), seed=0))
    th_g0, rep_g0 = b2.lm_solve(ref_gp, ref_gp.initial_theta(), cfg)
    ref_ba = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
    th_b0, rep_b0 = b2.lm_solve(ref_ba, ref_ba.encode(), cfg)

    ws = b2.Workspace()
    gp = b2.fix_gauge(b2.make_rays(obs, loss=b2.RobustLoss("huber", 0.1), seed=0))
    th_g, rep_g = b2.lm_solve(gp, gp.initial_theta(), cfg, ws)
    info_gp = ws.device_arena().info()
    assert info_gp["live_handles"] == 1 and info_gp["high_water"] >= gp.device_bytes()
    with pytest.raises(ValueError, match="live handles"):
        ws.device_arena().close()
    gp.release()
    assert ws.device_arena().info()["live_handles"] == 0
    ba = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
    th_b, rep_b = b2.lm_solve(ba, ba.encode(), cfg, ws)
    info_ba = ws.device_arena().info()
    assert info_ba["live_handles"] == 1
    # BA fits the GP stage's HBM (or one chunk was added)
    assert info_ba["chunk_mallocs"] <= info_gp["chunk_mallocs"] + 1
    assert np.array_equal(th_g, th_g0) and np.array_equal(th_b, th_b0)
    assert [i.cost_after for i in rep_g.iterations] == [i.cost_after for i in rep_g0.iterations]
    assert [i.cost_after for i in rep_b.iterations] == [i.cost_after for i in rep_b0.iterations]
    ba.release()
    # a third stage of the first shape reuses the coalesced arena without cudaMalloc
    before = ws.device_arena().info()["chunk_mallocs"]
    gp2 = b2.fix_gauge(b2.make_rays(obs, loss=b2.RobustLoss("huber", 0.1), seed=0))
    th_g2, _ = b2.lm_solve(gp2, gp2.initial_theta(), cfg, ws)
    after = ws.device_arena().info()
    assert after["chunk_mallocs"] - before <= 1          # at most the one coalescing allocation
    assert after["capacity"] >= after["high_water"]
    assert np.array_equal(th_g2, th_g0)
    gp2.release()
    ws.release_device()


def test_run_global_sfm_matches_stagewise_host_path(gpu):
    obs = observed(C=30, P=2500, k=6, seed=7)
    out, rep = b2.run_global_sfm(obs)
    gp_scene, rep_gp = b2.run_gp(obs, loss=b2.RobustLoss("huber", 0.1), config=b2.LMConfig(max_iterations=20))
    ba = b2.BAProblem(gp_scene, b2.RobustLoss("huber", 1.0))
    th, rep_ba = b2.lm_solve(ba, ba.encode(), b2.LMConfig(max_iterations=10))
    assert [i.cost_after for i in rep.gp.iterations] == [i.cost_after for i in rep_gp.iterations]
    assert [i.cost_after for i in rep.ba.iterations] == [i.cost_after for i in rep_ba.iterations]
    res = ba.decode(th)
    assert np.array_equal(out.points, res.points) and np.array_equal(out.centers, res.centers)
    assert np.array_equal(out.quats, res.quats) and np.array_equal(out.focals, res.focals)
    # BA minimises its robust cost (not the RMSE the report prints)
    assert rep.ba.iterations[-1].cost_after <= rep.ba.iterations[0].cost_before
    assert np.isfinite(rep.rmse_after_ba) and np.isfinite(rep.rmse_after_gp)


def test_make_rays_device_keeps_rays_on_device(gpu):
    obs = observed(C=10, P=300, k=4, seed=2)
    p = b2.make_rays_device(obs, loss=b2.RobustLoss("huber", 0.1))
    assert p._rays is None and p._rays_dev.is_cuda
    assert np.array_equal(p.rays, b2.make_rays(obs).rays)         # bit-identical (host copy on demand)
    bad = obs.copy()
    bad.cam_idx = bad.cam_idx.copy()
    bad.cam_idx[3] = bad.num_cameras
    with pytest.raises(IndexError):
        b2.make_rays_device(bad)


def test_block_cache_trim(gpu):
    st = synth.perturb_arrays(observed(C=20, P=1000, k=4), rot_deg=1.0, seed=1)
    p = b2.BAProblem(st)
    p.cost(p.encode())
    nbytes = p.device_bytes()
    _native.trim_cache()
    p.release()                                  # blocks go to the reuse cache
    assert _native.load().ssfm_cache_bytes() >= nbytes
    assert _native.trim_cache() >= nbytes
    assert _native.load().ssfm_cache_bytes() == 0
