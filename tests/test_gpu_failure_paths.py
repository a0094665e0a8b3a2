"""GPU: failure paths of the native (matrix-free) BA solve, as the reference
defines them:

* a point whose every observation is behind its cameras is masked: its
  residuals, Jacobian rows and gradient are zero, its damped block is pinned
  to identity, and its step is exactly zero (lm.py:495-505, scene.py:368-375);
* a point block whose determinant underflows to 0 is SingularBlock
  (lm.py:508-512): the damped solve fails, lm_solve rejects every step and
  raises SolverFailure once lambda reaches lambda_max (lm.py:775-781);
* post_step rejects quaternions with norm < 1e-12 as ZeroQuaternion
  (lm.py:104-117).
The masked case is also compared with the CPU oracle's dense solve.
"""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
import sparsesfm_port as orc
from paper_2510_13310_b200 import synth
from paper_2510_13310_b200.scene import SceneArrays
from .test_gpu_ba import solve_normal_native

pytestmark = pytest.mark.gpu


def ring_scene(C=12, P=30, seed=3, sigma=0.5):
    """every point observed by every camera (all in front), noisy pixels"""
    cfg = synth.SynthConfig(num_cameras=C, num_points=P, radius=10.0, focal=400.0, seed=seed)
    centers = synth.rig_centers(cfg)
    quats = np.stack([synth.look_at_origin(t) for t in centers])
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(P, 3))
    pts = d / np.linalg.norm(d, axis=1, keepdims=True) * (2.5 * rng.uniform(size=(P, 1)) ** (1 / 3))
    cam = np.repeat(np.arange(C), P)
    pt = np.tile(np.arange(P), C)
    arr = SceneArrays(quats, centers, np.full(C, 400.0), np.zeros((C, 2)), np.zeros((C, 2)), "pinhole", pts,
                      cam, pt, np.zeros((C * P, 2)), None)
    px, _ = b2.scene.project_many(arr)
    arr.pixels = px + rng.normal(0, sigma, px.shape)
    return arr


def with_point(arr, j, position, cams):
    """move point j to `position` and keep only its observations by `cams`"""
    out = arr.copy()
    out.points[j] = position
    keep = (arr.pt_idx != j) | np.isin(arr.cam_idx, cams)
    out.cam_idx, out.pt_idx, out.pixels = arr.cam_idx[keep], arr.pt_idx[keep], arr.pixels[keep]
    return out


def oracle_prob(arr, loss=("huber", 1.0)):
    return dict(C=arr.num_cameras, P=arr.num_points, cam=arr.cam_idx, pt=arr.pt_idx, pixels=arr.pixels,
                pps=arr.pps, dists=arr.dists, focals=arr.focals, model="pinhole", focal_mode=1, loss=loss)


def test_point_behind_all_its_cameras_gets_exactly_zero_step(gpu):
    arr = with_point(ring_scene(), 0, np.array([30.0, 4.0, 0.0]), [0, 1])   # behind cameras 0 and 1
    p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
    th = p.encode()
    r, jac = p.linearize(th)
    m = np.nonzero(arr.pt_idx == 0)[0]
    assert len(m) == 2
    assert np.all(r.reshape(-1, 2)[m] == 0.0) and np.all(jac.data.reshape(-1, 22)[m] == 0.0)
    C = arr.num_cameras
    seg = slice(7 * C, 7 * C + 3)
    g = p.gradient(th)
    assert np.all(g[seg] == 0.0)
    d, _ = solve_normal_native(gpu, p, 1e-3, b2.LMConfig())
    assert np.all(d[seg] == 0.0)                      # pinned: exactly zero (lm.py:500-505)
    assert np.isfinite(d).all()
    # the rest of the step is the damped system's solution (oracle: dense solve)
    prob = oracle_prob(arr)
    r_o, J_o = orc.ba_linearize(prob, th)
    Jd = orc.ba_dense_jacobian(prob, J_o)
    A = Jd.T @ Jd
    A[np.diag_indices_from(A)] *= 1.001
    keep = np.ones(len(th), bool)
    keep[seg] = False
    exact = np.zeros(len(th))
    exact[keep] = np.linalg.solve(A[np.ix_(keep, keep)], -(Jd.T @ r_o)[keep])
    assert np.abs(d - exact).max() / np.abs(exact).max() < 1e-6
    # a full solve never moves the masked point
    th1, rep = b2.lm_solve(p, th, b2.LMConfig(max_iterations=10))
    assert np.array_equal(th1[seg], th[seg])
    assert rep.num_accepted > 0


def test_underflowing_point_block_is_singular(gpu):
    # a point 1e155 in front of its cameras: J_p ~ f/z ~ 1e-152, so the damped
    # 3x3 block's determinant (~1e-915) underflows to 0 -> SingularBlock
    arr = ring_scene()
    far = -arr.centers[0] / np.linalg.norm(arr.centers[0]) * 1e155
    arr2 = with_point(arr, 0, far, [0])
    p = b2.BAProblem(arr2, b2.RobustLoss("trivial"))
    th = p.encode()
    p.gradient(th)
    with pytest.raises(b2.errors.SingularBlock):
        solve_normal_native(gpu, p, 1e-3, b2.LMConfig())
    cfg = b2.LMConfig(max_iterations=40)
    with pytest.raises(b2.errors.SolverFailure) as ei:
        b2.lm_solve(p, th, cfg)
    rep = ei.value.report
    assert rep.termination == "solver_failure"
    assert not any(i.step_accepted for i in rep.iterations)
    lams = [i.lam for i in rep.iterations]
    # the failing solve at lambda_max raises before its record is appended (lm.py:775-779)
    assert lams[0] == cfg.lambda0 and lams[-1] * cfg.lambda_up == pytest.approx(cfg.lambda_max)
    assert all(b == pytest.approx(min(a * cfg.lambda_up, cfg.lambda_max)) for a, b in zip(lams, lams[1:]))


def test_post_step_rejects_zero_quaternion(gpu):
    arr = ring_scene(C=4, P=6)
    p = b2.BAProblem(arr)
    th = p.encode()
    bad = th.copy()
    bad[7:11] = 0.0                                  # camera 1's quaternion
    with pytest.raises(b2.errors.ZeroQuaternion):
        p.post_step(bad)
    tiny = th.copy()
    tiny[7:11] = [5e-13, 0.0, 0.0, 0.0]              # norm below 1e-12
    with pytest.raises(b2.errors.ZeroQuaternion):
        p.post_step(tiny)
    ok = th.copy()
    ok[7:11] = [2e-12, 0.0, 0.0, 0.0]
    out = p.post_step(ok)
    assert np.array_equal(out[7:11], [1.0, 0.0, 0.0, 0.0])
    q = out[:7 * 4].reshape(4, 7)[:, :4]
    assert np.allclose(np.linalg.norm(q, axis=1), 1.0, atol=1e-15)


def test_repeated_persistent_solves_bitwise_equal(gpu):
    """Stress for the persistent PCG kernel's cross-CTA partials protocol
    (p.q and r.r/r.z partials now live in separate buffers): many
    repeated damped solves on the same linearization are bitwise equal."""
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ba_small.npz"))
    from .test_gpu_ba import problem_from_golden
    p = problem_from_golden(z)
    p.gradient(z["theta0"])
    d0, it0 = solve_normal_native(gpu, p, 1e-3, b2.LMConfig(cg_tol=1e-12))
    for _ in range(200):
        d, it = solve_normal_native(gpu, p, 1e-3, b2.LMConfig(cg_tol=1e-12))
        assert it == it0 and np.array_equal(d, d0)
    zz = np.load(os.path.join(os.path.dirname(__file__), "golden", "gp_small.npz"))
    from .test_gpu_gp import gp_from_golden
    q = gp_from_golden(zz)
    q.gradient(zz["theta0"])
    e0, j0 = solve_normal_native(gpu, q, 1e-2, b2.LMConfig(cg_tol=1e-12))
    for _ in range(200):
        e, j = solve_normal_native(gpu, q, 1e-2, b2.LMConfig(cg_tol=1e-12))
        assert j == j0 and np.array_equal(e, e0)
