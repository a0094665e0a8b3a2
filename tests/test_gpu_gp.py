"""GPU parity: global positioning on the B200 path vs the reference's golden
vectors, the CPU oracle and the reference's KATs (test_gp.py).

GP is gauge-fixed (camera 0 centre + mean scale), so parameters are compared
directly: 1e-8 absolute (reference self-spread 5e-14 / 1e-10).
"""
import ctypes as ct
import os

import numpy as np
import pytest

import paper_2510_13310_b200 as b2
import sparsesfm_port as orc
from paper_2510_13310_b200 import _native, synth
from paper_2510_13310_b200.scene import Camera, Observation, Point3D, Scene
from .conftest import golden, gp_prob_from_golden, summary

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def gp_from_golden(z):
    dm = bool(int(z["depth_mode"]))
    p = b2.GPProblem(z["rays"], z["quats"], z["cam"], z["pt"], len(z["points"]),
                     b2.RobustLoss(str(z["loss_kind"]), float(z["loss_delta"])), dm,
                     z["ray_depths"] if dm else None, seed=0)
    return b2.fix_gauge(p)


@pytest.mark.parametrize("name", ["gp_small.npz", "gp_depth.npz"])
def test_cost_residual_jacobian_gradient_vs_reference(gpu, name):
    z = golden(name)
    p = gp_from_golden(z)
    th = z["theta0"]
    assert np.array_equal(th, p.initial_theta())
    assert p.cost(th) == pytest.approx(float(z["cost0"]), rel=1e-14)
    r, jac = p.linearize(th)
    assert rel(r, z["r0"]) < 1e-14
    assert rel(jac.data, z["J0"]) < 1e-14
    assert rel(p.gradient(th), z["grad0"]) < 1e-11


def test_rays_match_reference():
    z = golden("gp_small.npz")
    arr = b2.SceneArrays(z["quats"], z["centers"], z["focals"], z["pps"], z["dists"], "pinhole",
                         z["points"], z["cam"], z["pt"], z["pixels"], None)
    assert np.array_equal(b2.make_rays(arr).rays, z["rays"])


def test_damped_solve_and_post_step_vs_reference(gpu):
    z = golden("gp_small.npz")
    p = gp_from_golden(z)
    p.gradient(z["theta0"])
    d = gpu.empty(p.layout.total_params, dtype=gpu.float64, device="cuda")
    it = ct.c_int32(0)
    _native.check(_native.load().ssfm_solve_normal(ct.c_void_p(p._native_handle().ptr), 1e-2,
                                                   ct.byref(_native.lm_config_c(b2.LMConfig())),
                                                   ct.c_void_p(d.data_ptr()), ct.byref(it),
                                                   ct.c_void_p(gpu.cuda.current_stream().cuda_stream)))
    assert rel(d.cpu().numpy(), z["delta_lam1e2"]) < 1e-7
    assert abs(it.value - int(z["cg_lam1e2"])) <= 2
    th = z["theta0"]
    probe = p.post_step(th + 0.1 * np.sin(np.arange(len(th))))
    assert rel(probe, z["post_step_probe"]) < 1e-13


@pytest.mark.parametrize("name,iters", [("gp_small.npz", 40), ("gp_depth.npz", 30)])
def test_lm_solve_trajectory_vs_reference(gpu, name, iters):
    z = golden(name)
    p = gp_from_golden(z)
    th, rep = b2.lm_solve(p, z["theta0"], b2.LMConfig(max_iterations=iters))
    ref = z["records"]
    assert rep.termination == str(z["termination"])
    assert [i.step_accepted for i in rep.iterations] == [bool(x) for x in ref[:, 4]]
    assert rep.iterations[-1].cost_after == pytest.approx(ref[-1, 2], rel=1e-8)
    assert np.abs(th - z["theta_final"]).max() < 1e-8


def test_c2_forty_iterations_vs_reference(gpu):
    s = summary()["c2"]
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=200, num_points=50000,
                                                     visibility_fraction=6 / 200, pixel_noise_sigma=0.5, seed=0))
    p = b2.fix_gauge(b2.make_rays(obs, depth_mode=False, loss=b2.RobustLoss("huber", 0.1), seed=0))
    th, rep = b2.lm_solve(p, p.initial_theta(), b2.LMConfig(max_iterations=40))
    assert rep.termination == s["termination"]
    assert [i.step_accepted for i in rep.iterations] == s["accepted"]
    assert rep.iterations[-1].cost_after == pytest.approx(s["final_cost"], rel=1e-8)
    ref = np.load(os.path.join(os.path.dirname(__file__), "golden", "c2_theta_final.npy"))
    assert np.abs(th[:len(ref)] - ref).max() < 1e-8


def ray_scene(pixels, f=1.0, q=None):
    q = np.array([1.0, 0, 0, 0]) if q is None else q
    return Scene([Camera(q.copy(), np.zeros(3), f)],
                 [Point3D(np.array([0.0, 0.0, float(j + 1)])) for j in range(len(pixels))],
                 [Observation(0, j, np.asarray(px, float)) for j, px in enumerate(pixels)])


def manual(p, c, x, d=None):
    parts = [np.asarray(c, float).ravel(), np.asarray(x, float).ravel()]
    if not p.depth_mode:
        parts.append(np.asarray(d, float).ravel())
    return np.concatenate(parts)


def test_residual_kats(gpu):                              # test_gp.py:57-74
    p = b2.make_rays(ray_scene([(0.0, 0.0)]))
    assert np.allclose(b2.gp_residuals(p, manual(p, [[0, 0, 0]], [[0, 0, 2]], [0.5])), 0.0)
    assert np.allclose(b2.gp_residuals(p, manual(p, [[0, 0, 0]], [[1, 0, 1]], [1.0])), [-1.0, 0.0, 0.0])
    sc = ray_scene([(0.0, 0.0)])
    sc.observations[0].depth = 2.0
    pd = b2.make_rays(sc, depth_mode=True)
    assert np.allclose(b2.gp_residuals(pd, manual(pd, [[0, 0, 0]], [[0, 0, 2]])), 0.0)


def test_analytic_blocks_and_zero_scale(gpu):             # test_gp.py:93-108
    p = b2.make_rays(ray_scene([(0.0, 0.0)]))
    j = b2.gp_jacobian(p, manual(p, [[0.5, 0, 0]], [[0, 0, 2]], [0.7]))
    span = np.array([-0.5, 0, 2.0])
    assert np.allclose(j.entry_block(0), 0.7 * np.eye(3))
    assert np.allclose(j.entry_block(1), -0.7 * np.eye(3))
    assert np.allclose(j.entry_block(2), -span.reshape(3, 1))
    j0 = b2.gp_jacobian(p, manual(p, [[0.5, 0, 0]], [[0, 0, 2]], [0.0]))
    assert np.all(j0.entry_block(0) == 0.0) and np.all(j0.entry_block(1) == 0.0)


def test_jacobian_finite_differences(gpu):                # test_gp.py:78-91
    rng = np.random.default_rng(4)
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=4, num_points=12, radius=6.0, focal=150.0, seed=8))
    for dm in (False, True):
        p = b2.make_rays(obs, depth_mode=dm)
        th = p.initial_theta() + 0.1 * rng.normal(size=p.layout.total_params)
        if not dm:
            th[3 * (p.num_cameras + p.num_points):] = rng.uniform(0.5, 2.0, p.num_obs)
        J = orc.gp_dense_jacobian(gp_prob(p), orc.gp_linearize(gp_prob(p), th)[1])
        jn = b2.gp_jacobian(p, th)
        assert rel(jn.data, orc.ref_layout(orc.gp_linearize(gp_prob(p), th)[1],
                                           [3, 3] if dm else [3, 3, 1])) < 1e-13
        for k in range(0, p.layout.total_params, 7):
            e = np.zeros_like(th)
            e[k] = 1e-6 * max(1.0, abs(th[k]))
            fd = (b2.gp_residuals(p, th + e) - b2.gp_residuals(p, th - e)) / (2 * e[k])
            assert np.abs(J[:, k] - fd).max() / (1 + np.abs(fd).max()) < 1e-6


def gp_prob(p):
    return dict(C=p.num_cameras, P=p.num_points, cam=p.cam_idx, pt=p.pt_idx, rays=p.rays,
                depth_mode=p.depth_mode, depths=p.depths, gauge_fixed=p.gauge_fixed,
                loss=(p.loss.kind, p.loss.delta))


def test_gauge_invariances(gpu):                          # test_gp.py:124-168
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=4, num_points=10, radius=5.0, focal=100.0, seed=1))
    p = b2.make_rays(obs)
    rng = np.random.default_rng(0)
    c = np.round(rng.uniform(0, 1, (4, 3)) * 1024) / 1024
    x = np.round(rng.uniform(0, 1, (10, 3)) * 1024) / 1024
    d = rng.uniform(0.5, 2.0, p.num_obs)
    assert np.array_equal(b2.gp_residuals(p, manual(p, c, x, d)), b2.gp_residuals(p, manual(p, c + 5.0, x + 5.0, d)))
    c2 = rng.uniform(0, 1, (4, 3))
    x2 = rng.uniform(0, 1, (10, 3))
    assert p.cost(manual(p, c2, x2, d)) == p.cost(manual(p, 2.0 * c2, 2.0 * x2, 0.5 * d))
    pf = b2.fix_gauge(b2.make_rays(obs))
    th = pf.initial_theta()
    th[3 * 14:] = np.random.default_rng(5).uniform(0.5, 3.0, pf.num_obs)
    out = pf.post_step(th)
    assert abs(out[3 * 14:].mean() - 1.0) < 1e-12
    assert abs(pf.cost(out) - pf.cost(th)) < 1e-9 * max(pf.cost(th), 1.0)
    assert np.allclose(out[:3], th[:3], atol=1e-12)


def test_single_camera_converges_immediately(gpu):        # test_gp.py:172-182
    p = b2.fix_gauge(b2.make_rays(ray_scene([(0.0, 0.0), (1.0, 0.0), (0.0, 1.0)])))
    th0 = manual(p, [[0, 0, 0]], p.rays.copy(), np.ones(3))
    th, rep = b2.lm_solve(p, th0, b2.LMConfig())
    assert rep.termination == "converged_grad" and rep.num_accepted == 0
    assert p.cost(th) == 0.0


def test_exact_rays_recover_geometry(gpu):                # test_gp.py:184-196
    truth, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=6, num_points=80, radius=8.0, focal=400.0, seed=11))
    res, rep = b2.run_gp(obs, loss=b2.RobustLoss("trivial"), config=b2.LMConfig(max_iterations=200), seed=0)
    assert rep.termination in ("converged_cost", "converged_grad")
    _, al = synth.align(res, truth, "sim3")
    assert synth.center_rmse(al, truth) < 1e-3 * synth.scene_diameter(truth)
    assert np.array_equal(res.quats, obs.quats) and np.array_equal(res.focals, obs.focals)


def test_depth_mode_metric_scale(gpu):                    # test_gp.py:198-219
    truth, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=6, num_points=80, radius=8.0, focal=400.0, seed=13))
    res, _ = b2.run_gp(obs, depth_mode=True, loss=b2.RobustLoss("trivial"), config=b2.LMConfig(max_iterations=200))
    _, al = synth.align(res, truth, "se3")
    assert synth.center_rmse(al, truth) < 1e-3 * synth.scene_diameter(truth)
    dbl = obs.copy()
    dbl.depths = 2.0 * obs.depths
    res2, _ = b2.run_gp(dbl, depth_mode=True, loss=b2.RobustLoss("trivial"), config=b2.LMConfig(max_iterations=200))
    d1 = np.linalg.norm(res.centers - res.centers.mean(0), axis=1).mean()
    d2 = np.linalg.norm(res2.centers - res2.centers.mean(0), axis=1).mean()
    assert abs(d2 / d1 - 2.0) < 0.02


def test_gp_pattern_export(gpu):
    z = golden("gp_small.npz")
    p = gp_from_golden(z)
    pat = p.export_pattern()
    assert np.array_equal(pat["off_keys"], z["off_keys"])
    assert np.array_equal(pat["schur_slots"], z["schur_slots"])


@pytest.mark.parametrize("depth", [False, True])
def test_make_rays_device_bit_identical(gpu, depth):
    """k_make_rays (numpy operation order, no contraction) vs the host
    restatement and the reference's rays (gp_small golden)."""
    z = golden("gp_small.npz")
    arr = b2.SceneArrays(z["quats"], z["centers"], z["focals"], z["pps"], z["dists"], "pinhole",
                         z["points"], z["cam"], z["pt"], z["pixels"], None)
    if not depth:
        assert np.array_equal(b2.make_rays_device(arr).rays, z["rays"])
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=40, num_points=3000, visibility_fraction=0.2,
                                                     pixel_noise_sigma=1.0, seed=4))
    if depth:
        obs.depths = np.random.default_rng(1).uniform(1.0, 9.0, size=obs.num_observations)
    h = b2.make_rays(obs, depth_mode=depth)
    d = b2.make_rays_device(obs, depth_mode=depth)
    assert np.array_equal(h.rays, d.rays)
    if depth:
        assert np.array_equal(h.depths, d.depths)
