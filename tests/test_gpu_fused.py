"""GPU: the fused single-pass Schur operator (csrc/fused.cuh) against the
two-pass operator and the reference's damped solve.

Both operators apply the same matrix-free S; only the
summation order of the camera terms differs, so the damped steps agree to the
CG tolerance (cg_tol 1e-12 here: 1e-9 relative) and the CG counts agree
within one iteration. The fused operator must also be bitwise deterministic
(fixed rank order, no floating-point atomics) for every slot-group count.
"""
import ctypes as ct
import os

import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import _native, synth
from .conftest import golden
from .test_gpu_ba import problem_from_golden, rel, solve_normal_native

pytestmark = pytest.mark.gpu


def with_operator(mode, make):
    old = os.environ.get("SSFM_FUSED")
    os.environ["SSFM_FUSED"] = mode
    try:
        p = make()
        p._native_handle()
    finally:
        if old is None:
            os.environ.pop("SSFM_FUSED")
        else:
            os.environ["SSFM_FUSED"] = old
    return p


def op_info(p):
    g, grid, nt, sm = ct.c_int32(), ct.c_int32(), ct.c_int32(), ct.c_int64()
    _native.check(_native.load().ssfm_operator_info(ct.c_void_p(p._native_handle().ptr), ct.byref(g),
                                                    ct.byref(grid), ct.byref(nt), ct.byref(sm)))
    return g.value, grid.value, nt.value, sm.value


def wide_scene():
    """points seen by up to 60 cameras (batches with > 32 observations per point)
    mixed with 2-view points: exercises multi-round batches and high ranks"""
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=80, num_points=3000,
                                                     visibility_fraction=0.05, pixel_noise_sigma=1.0, seed=5))
    st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=2)
    rng = np.random.default_rng(0)
    # add 40 points seen by 40..60 cameras each
    extra_cam, extra_pt, extra_px = [], [], []
    P0 = len(st.points)
    pts = rng.uniform(-2, 2, size=(40, 3))
    for j in range(40):
        cams = rng.choice(80, size=int(rng.integers(40, 61)), replace=False)
        for c in sorted(cams):
            extra_cam.append(c)
            extra_pt.append(P0 + j)
            extra_px.append(rng.normal(size=2) * 50)
    st.points = np.concatenate([st.points, pts])
    st.cam_idx = np.concatenate([st.cam_idx, np.array(extra_cam, dtype=st.cam_idx.dtype)])
    st.pt_idx = np.concatenate([st.pt_idx, np.array(extra_pt, dtype=st.pt_idx.dtype)])
    st.pixels = np.concatenate([st.pixels, np.array(extra_px)])
    st.depths = None
    return st


@pytest.mark.parametrize("groups", ["1", "2", "4", "8"])
def test_fused_matches_two_pass_damped_solve(gpu, groups):
    st = wide_scene()
    loss = b2.RobustLoss("huber", 1.0)
    cfg = b2.LMConfig(cg_tol=1e-12, cg_max_iters=5000)
    ref = with_operator("0", lambda: b2.BAProblem(st, loss))
    assert op_info(ref)[0] == 0
    fz = with_operator(groups, lambda: b2.BAProblem(st, loss))
    assert op_info(fz)[0] == int(groups)
    th = ref.encode()
    ref.gradient(th)
    fz.gradient(th)
    for lam in (1e-4, 1e-1):
        d0, it0 = solve_normal_native(gpu, ref, lam, cfg)
        d1, it1 = solve_normal_native(gpu, fz, lam, cfg)
        assert rel(d1, d0) < 1e-9, (lam, rel(d1, d0))
        # the stop at cg_tol 1e-12 is rounding-sensitive; the two-pass camera
        # pass rebuilds Jc^T Jp from factored records (to rounding) while the
        # fused pass reads the stored Jacobian: 152 vs 157 iterations here
        assert abs(it1 - it0) <= max(2, 0.05 * it0)
        d2, it2 = solve_normal_native(gpu, fz, lam, cfg)
        assert np.array_equal(d1, d2) and it1 == it2       # bitwise deterministic


def test_fused_default_on_reference_golden(gpu):
    z = golden("ba_small.npz")
    p = problem_from_golden(z)
    assert op_info(p)[0] >= 1                     # the default operator is the fused one
    p.gradient(z["theta0"])
    d, it = solve_normal_native(gpu, p, 1e-3, b2.LMConfig())
    assert rel(d, z["delta_lam1e3"]) < 1e-7
    assert abs(it - int(z["cg_lam1e3"])) <= 2


def test_fused_lm_trajectory_matches_two_pass(gpu):
    st = wide_scene()
    loss = b2.RobustLoss("huber", 1.0)
    ref = with_operator("0", lambda: b2.BAProblem(st, loss))
    fz = with_operator("2", lambda: b2.BAProblem(st, loss))
    th0 = ref.encode()
    a, ra = b2.lm_solve(ref, th0, b2.LMConfig(max_iterations=12))
    b, rb = b2.lm_solve(fz, th0, b2.LMConfig(max_iterations=12))
    assert [i.step_accepted for i in ra.iterations] == [i.step_accepted for i in rb.iterations]
    assert abs(ra.iterations[-1].cost_after - rb.iterations[-1].cost_after) <= 1e-10 * ra.iterations[-1].cost_after


def with_env(env, make):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        p = make()
        p._native_handle()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k)
            else:
                os.environ[k] = v
    return p


@pytest.mark.parametrize("fused", ["0", "1"])
def test_graph_pcg_matches_persistent_kernel(gpu, fused):
    """The CUDA-graph PCG (conditional WHILE node, one kernel per phase) and
    the persistent cooperative kernel run the same recurrences; only the
    vector-phase partial sums are grouped differently (148 vs grid blocks)."""
    st = wide_scene()
    loss = b2.RobustLoss("huber", 1.0)
    cfg = b2.LMConfig(cg_tol=1e-12, cg_max_iters=5000)
    per = with_env({"SSFM_FUSED": fused, "SSFM_PCG_GRAPH": "0"}, lambda: b2.BAProblem(st, loss))
    gra = with_env({"SSFM_FUSED": fused, "SSFM_PCG_GRAPH": "1"}, lambda: b2.BAProblem(st, loss))
    th = per.encode()
    per.gradient(th)
    gra.gradient(th)
    for lam in (1e-4, 1e-1):
        d0, it0 = solve_normal_native(gpu, per, lam, cfg)
        d1, it1 = solve_normal_native(gpu, gra, lam, cfg)
        assert rel(d1, d0) < 1e-9 and abs(it1 - it0) <= max(2, 0.03 * it0)
        d2, it2 = solve_normal_native(gpu, gra, lam, cfg)
        assert np.array_equal(d1, d2) and it1 == it2
    # iteration cap and the CGStall path through the graph
    with pytest.raises(b2.errors.CGStall):
        solve_normal_native(gpu, gra, 1e-4, b2.LMConfig(cg_max_iters=3))


def gp_wide():
    """GP rays of the wide scene: multi-round batches (points seen by 40-60
    cameras) next to 2-view points, gauge fixed (camera 0 pinned)"""
    st = wide_scene()
    return lambda: b2.fix_gauge(b2.make_rays(st, depth_mode=False, loss=b2.RobustLoss("huber", 0.1), seed=0))


def test_gp_fused_matches_two_pass_damped_solve(gpu):
    make = gp_wide()
    ref = with_operator("0", make)
    fz = with_operator("1", make)
    assert op_info(ref)[0] == 0 and op_info(fz)[0] == 1
    cfg = b2.LMConfig(cg_tol=1e-12, cg_max_iters=5000)
    th = ref.initial_theta()
    ref.gradient(th)
    fz.gradient(th)
    for lam in (1e-4, 1e-1):
        d0, it0 = solve_normal_native(gpu, ref, lam, cfg)
        d1, it1 = solve_normal_native(gpu, fz, lam, cfg)
        assert rel(d1, d0) < 1e-9, (lam, rel(d1, d0))
        assert abs(it1 - it0) <= max(2, 0.03 * it0)
        d2, it2 = solve_normal_native(gpu, fz, lam, cfg)
        assert np.array_equal(d1, d2) and it1 == it2


def test_gp_fused_default_on_reference_golden(gpu):
    from .test_gpu_gp import gp_from_golden
    z = golden("gp_small.npz")
    assert op_info(gp_from_golden(z))[0] == 0      # small problem: two-pass by default
    p = with_operator("1", lambda: gp_from_golden(z))
    assert op_info(p)[0] == 1
    p.gradient(z["theta0"])
    d, it = solve_normal_native(gpu, p, 1e-2, b2.LMConfig())
    assert rel(d, z["delta_lam1e2"]) < 1e-7
    assert abs(it - int(z["cg_lam1e2"])) <= 2


def test_gp_fused_lm_trajectory_matches_two_pass(gpu):
    make = gp_wide()
    ref = with_operator("0", make)
    fz = with_operator("1", make)
    th0 = ref.initial_theta()
    a, ra = b2.lm_solve(ref, th0, b2.LMConfig(max_iterations=15))
    b, rb = b2.lm_solve(fz, th0, b2.LMConfig(max_iterations=15))
    assert [i.step_accepted for i in ra.iterations] == [i.step_accepted for i in rb.iterations]
    assert abs(ra.iterations[-1].cost_after - rb.iterations[-1].cost_after) <= 1e-10 * ra.iterations[-1].cost_after
    assert np.abs(a - b).max() < 1e-8


def factored_problem(make, fac, graph="0"):
    return with_env({"SSFM_FUSED": "0", "SSFM_FACTORED": fac, "SSFM_PCG_GRAPH": graph}, make)


@pytest.mark.parametrize("graph", ["0", "1"])
@pytest.mark.parametrize("name", ["ba_small.npz", "ba_bal.npz", "ba_nofocal.npz", "ba_shared.npz"])
def test_factored_two_pass_matches_jacobian_two_pass(gpu, name, graph):
    """The factored camera pass (ba_factor: sw du_dp = S E, Jc^T Jp rebuilt from
    the camera cache) applies the stored Jacobian's operator to rounding: same damped
    step (1e-9 at cg_tol 1e-12), CG counts within rounding, deterministic;
    every camera model and focal mode."""
    z = golden(name)
    make = lambda: problem_from_golden(z)  # noqa: E731
    ref = factored_problem(make, "0", graph)
    fac = factored_problem(make, "1", graph)
    th = z["theta0"]
    ref.gradient(th)
    fac.gradient(th)
    cfg = b2.LMConfig(cg_tol=1e-12, cg_max_iters=5000)
    for lam in (1e-4, 1e-1):
        d0, it0 = solve_normal_native(gpu, ref, lam, cfg)
        d1, it1 = solve_normal_native(gpu, fac, lam, cfg)
        assert rel(d1, d0) < 1e-9, (lam, rel(d1, d0))
        # both the camera pass and the Schur preconditioner blocks are rebuilt
        # from the factored record (to rounding): the stop at cg_tol 1e-12 on
        # the shared-focal system (one focal coupled to every camera) moves by
        # up to 4 of 46 iterations; the steps agree to 1e-9
        assert abs(it1 - it0) <= max(4, 0.1 * it0)
        d2, it2 = solve_normal_native(gpu, fac, lam, cfg)
        assert np.array_equal(d1, d2) and it1 == it2


@pytest.mark.parametrize("graph", ["0", "1"])
def test_factored_wide_scene_and_trajectory(gpu, graph):
    st = wide_scene()
    loss = b2.RobustLoss("huber", 1.0)
    ref = with_env({"SSFM_FUSED": "0", "SSFM_FACTORED": "0", "SSFM_PCG_GRAPH": graph},
                   lambda: b2.BAProblem(st, loss))
    fac = with_env({"SSFM_FUSED": "0", "SSFM_FACTORED": "1", "SSFM_PCG_GRAPH": graph},
                   lambda: b2.BAProblem(st, loss))
    th0 = ref.encode()
    a, ra = b2.lm_solve(ref, th0, b2.LMConfig(max_iterations=10))
    b, rb = b2.lm_solve(fac, th0, b2.LMConfig(max_iterations=10))
    assert [i.step_accepted for i in ra.iterations] == [i.step_accepted for i in rb.iterations]
    assert abs(ra.iterations[-1].cost_after - rb.iterations[-1].cost_after) <= 1e-10 * ra.iterations[-1].cost_after


def test_gp_graph_pcg_matches_persistent_kernel(gpu):
    """GP PCG as a CUDA graph (gp_pcg_graph.cuh) vs the persistent two-pass
    kernel: same damped step, deterministic, CGStall at the cap."""
    make = gp_wide()
    per = with_env({"SSFM_FUSED": "0", "SSFM_GP_GRAPH": "0"}, make)
    gra = with_env({"SSFM_FUSED": "0", "SSFM_GP_GRAPH": "1"}, make)
    cfg = b2.LMConfig(cg_tol=1e-12, cg_max_iters=5000)
    th = per.initial_theta()
    per.gradient(th)
    gra.gradient(th)
    for lam in (1e-4, 1e-1):
        d0, it0 = solve_normal_native(gpu, per, lam, cfg)
        d1, it1 = solve_normal_native(gpu, gra, lam, cfg)
        assert rel(d1, d0) < 1e-9 and abs(it1 - it0) <= max(2, 0.03 * it0)
        d2, it2 = solve_normal_native(gpu, gra, lam, cfg)
        assert np.array_equal(d1, d2) and it1 == it2
    with pytest.raises(b2.errors.CGStall):
        solve_normal_native(gpu, gra, 1e-4, b2.LMConfig(cg_max_iters=2))
    a, ra = b2.lm_solve(per, th, b2.LMConfig(max_iterations=10))
    b, rb = b2.lm_solve(gra, th, b2.LMConfig(max_iterations=10))
    assert [i.step_accepted for i in ra.iterations] == [i.step_accepted for i in rb.iterations]
    assert np.abs(a - b).max() < 1e-8


@pytest.mark.parametrize("div", ["4", "37"])
def test_point_pass_partition_independent(gpu, div):
    """The graph PCG's point pass gives each warp a contiguous range of point
    batches and prefetches the next round's indices across batch boundaries
    (ba_point_pass_w). Every point is still summed by one owner lane in
    observation order, so a smaller grid (another batch partition,
    SSFM_PTP_GRID_DIV) must give bit-identical damped steps on the wide scene
    (multi-round batches, points seen by up to 60 cameras)."""
    st = wide_scene()
    loss = b2.RobustLoss("huber", 1.0)
    cfg = b2.LMConfig(cg_tol=1e-12, cg_max_iters=5000)
    ref = with_env({"SSFM_FUSED": "0", "SSFM_PCG_GRAPH": "1"}, lambda: b2.BAProblem(st, loss))
    alt = with_env({"SSFM_FUSED": "0", "SSFM_PCG_GRAPH": "1", "SSFM_PTP_GRID_DIV": div},
                   lambda: b2.BAProblem(st, loss))
    th = ref.encode()
    ref.gradient(th)
    alt.gradient(th)
    for lam in (1e-4, 1e-1):
        d0, it0 = solve_normal_native(gpu, ref, lam, cfg)
        d1, it1 = solve_normal_native(gpu, alt, lam, cfg)
        assert np.array_equal(d0, d1) and it0 == it1
