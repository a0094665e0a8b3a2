"""GPU: solve_normal with the default Schur PCG on an EXPLICIT BlockNormalSystem
(lm.py:537-720 -> csrc/schur_explicit.cuh) and lm_solve over foreign problem
providers that use it.

Ports of the reference's own tests (pkg/tests/test_lm.py:44-159), plus the
reference's damped steps on the ba_small / gp_small goldens (the same system
the reference solved with its default solver: same CG count, step within
1e-7) and the failure paths of _invert_elim_blocks / pinning / CGStall.
"""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200.errors import CGStall, SingularBlock, SolverFailure
from paper_2510_13310_b200.lm import LMConfig, Workspace, lm_solve, solve_normal
from paper_2510_13310_b200.sparse_block import BlockLayout, BlockSparseJacobian, apply_damping, jtj, jtr
from .conftest import golden

pytestmark = pytest.mark.gpu


def dense_jacobian(layout, blocks):
    j = np.zeros((layout.total_residuals, layout.total_params))
    for r, p, arr in blocks:
        arr = np.asarray(arr)
        r0, p0 = layout.residual_offsets[r], layout.param_offsets[p]
        j[r0:r0 + arr.shape[0], p0:p0 + arr.shape[1]] = arr
    return j


def random_ba_blocks(rng, num_cams, num_pts, visibility=1.0):
    """pose 2x7, point 2x3, focal 2x1 per observation (test_sparse_block.py:38-54)"""
    kinds = ["camera_pose"] * num_cams + ["point"] * num_pts + ["focal"] * num_cams
    obs = []
    for j in range(num_pts):
        cams = [i for i in range(num_cams) if rng.uniform() < visibility]
        if len(cams) < 2:
            cams = list(rng.choice(num_cams, size=2, replace=False))
        obs.extend((int(i), j) for i in cams)
    layout = BlockLayout(kinds, [2] * len(obs))
    blocks = []
    for r, (i, j) in enumerate(obs):
        blocks.append((r, i, rng.normal(size=(2, 7))))
        blocks.append((r, num_cams + j, rng.normal(size=(2, 3))))
        blocks.append((r, num_cams + num_pts + i, rng.normal(size=(2, 1))))
    return layout, blocks


def random_gp_blocks(rng, num_cams, num_pts, obs_per_pt=3):
    """centre 3x3, point 3x3 and scale 3x1 per observation (test_lm.py:12-29)"""
    kinds = ["gp_center"] * num_cams + ["gp_point"] * num_pts
    obs = []
    for j in range(num_pts):
        cams = rng.choice(num_cams, size=min(obs_per_pt, num_cams), replace=False)
        obs.extend((int(i), j) for i in sorted(cams))
    kinds += ["gp_scale"] * len(obs)
    layout = BlockLayout(kinds, [3] * len(obs))
    blocks = []
    for r, (i, j) in enumerate(obs):
        blocks.append((r, i, rng.normal(size=(3, 3))))
        blocks.append((r, num_cams + j, rng.normal(size=(3, 3))))
        blocks.append((r, num_cams + num_pts + r, rng.normal(size=(3, 1))))
    return layout, blocks


def build_system(layout, blocks, rng, lam):
    j = BlockSparseJacobian.from_blocks(layout, blocks)
    r = rng.normal(size=layout.total_residuals)
    sys_ = jtj(j)
    g = jtr(j, r)
    sys_.gradient[:] = -g
    damped = apply_damping(sys_, lam)
    jd = dense_jacobian(layout, blocks)
    a = jd.T @ jd
    return damped, a + lam * np.diag(np.diag(a)), -g


def test_diagonal_only_system(gpu):
    layout = BlockLayout(["gp_center", "gp_point"], [3])
    blocks = [(0, 0, np.diag([1.0, 2.0, 4.0])), (0, 1, np.zeros((3, 3)))]
    sys_ = jtj(BlockSparseJacobian.from_blocks(layout, blocks))
    sys_.data[sys_.off_off[0]:] = 0.0
    sys_.gradient[:] = np.array([2.0, 8.0, 32.0, 0, 0, 0])
    for solver in ("schur_pcg", "dense"):
        delta = solve_normal(sys_, layout, LMConfig(solver=solver))
        assert np.allclose(delta, [2.0, 2.0, 2.0, 0, 0, 0], atol=1e-9)


@pytest.mark.parametrize("seed", range(5))
def test_ba_schur_matches_dense_oracle(gpu, seed):
    rng = np.random.default_rng(seed)
    layout, blocks = random_ba_blocks(rng, 3, 7, visibility=0.8)
    damped, a_damped, rhs = build_system(layout, blocks, rng, lam=0.3)
    expect = np.linalg.solve(a_damped, rhs)
    got = solve_normal(damped, layout, LMConfig(cg_tol=1e-12, cg_max_iters=2000))
    assert np.linalg.norm(got - expect) / np.linalg.norm(expect) < 1e-6
    got_dense = solve_normal(damped, layout, LMConfig(solver="dense"))
    assert np.linalg.norm(got_dense - expect) / np.linalg.norm(expect) < 1e-8


@pytest.mark.parametrize("seed", range(5))
def test_gp_two_stage_elimination_matches_dense_oracle(gpu, seed):
    rng = np.random.default_rng(100 + seed)
    layout, blocks = random_gp_blocks(rng, 4, 6)
    damped, a_damped, rhs = build_system(layout, blocks, rng, lam=0.2)
    expect = np.linalg.solve(a_damped, rhs)
    got = solve_normal(damped, layout, LMConfig(cg_tol=1e-12, cg_max_iters=2000))
    assert np.linalg.norm(got - expect) / np.linalg.norm(expect) < 1e-6


@pytest.mark.parametrize("solver", ["schur_pcg", "dense"])
def test_equation_residual_bound(gpu, solver):
    rng = np.random.default_rng(17)
    layout, blocks = random_ba_blocks(rng, 4, 10, visibility=0.6)
    damped, a_damped, rhs = build_system(layout, blocks, rng, lam=1e-4)
    cfg = LMConfig(solver=solver)
    delta = solve_normal(damped, layout, cfg)
    bound = (cfg.cg_tol if solver == "schur_pcg" else 1e-10) * np.linalg.norm(rhs)
    assert np.linalg.norm(a_damped @ delta - rhs) <= bound


def test_masked_point_block_stays_fixed(gpu):
    rng = np.random.default_rng(23)
    layout, blocks = random_ba_blocks(rng, 2, 4, visibility=1.0)
    blocks = [(r, p, np.zeros_like(np.asarray(b)) if p == 3 else b) for r, p, b in blocks]
    j = BlockSparseJacobian.from_blocks(layout, blocks)
    r = rng.normal(size=layout.total_residuals)
    sys_ = jtj(j)
    sys_.gradient[:] = -jtr(j, r)
    damped = apply_damping(sys_, 0.5)
    for solver in ("schur_pcg", "dense"):
        delta = solve_normal(damped, layout, LMConfig(solver=solver))
        seg = slice(layout.param_offsets[3], layout.param_offsets[4])
        assert np.all(delta[seg] == 0.0)          # exactly zero (lm.py:500-505)
        assert np.isfinite(delta).all()


def test_masked_point_with_gradient_raises(gpu):
    rng = np.random.default_rng(23)
    layout, blocks = random_ba_blocks(rng, 2, 4, visibility=1.0)
    blocks = [(r, p, np.zeros_like(np.asarray(b)) if p == 3 else b) for r, p, b in blocks]
    j = BlockSparseJacobian.from_blocks(layout, blocks)
    sys_ = jtj(j)
    sys_.gradient[:] = -jtr(j, rng.normal(size=layout.total_residuals))
    sys_.gradient[layout.param_offsets[3] + 1] = 0.25      # inconsistent: masked direction, non-zero gradient
    with pytest.raises(SingularBlock, match="masked point direction"):
        solve_normal(apply_damping(sys_, 0.5), layout, LMConfig())


def test_indefinite_point_block_raises(gpu):        # det <= 0 (lm.py:508-512)
    rng = np.random.default_rng(3)
    layout, blocks = random_ba_blocks(rng, 3, 5)
    damped, _, _ = build_system(layout, blocks, rng, lam=0.1)
    d0 = damped.diag_off[4]                       # point 1's diagonal block
    damped.data[d0:d0 + 9] = np.array([1.0, 2.0, 0.0, 2.0, 1.0, 0.0, 0.0, 0.0, 1.0])   # det = -3
    with pytest.raises(SingularBlock, match="singular"):
        solve_normal(damped, layout, LMConfig())


def test_masked_retained_direction_with_gradient_raises(gpu):     # lm.py:628-633
    layout = BlockLayout(["focal", "focal"], [2])
    blocks = [(0, 0, np.array([[1.0], [2.0]])), (0, 1, np.zeros((2, 1)))]
    sys_ = jtj(BlockSparseJacobian.from_blocks(layout, blocks))
    sys_.gradient[:] = np.array([1.0, 0.0])
    d = solve_normal(apply_damping(sys_, 0.1), layout, LMConfig())
    assert d[1] == 0.0 and d[0] == pytest.approx(1.0 / 5.5, rel=1e-12)
    sys_.gradient[:] = np.array([1.0, 0.5])
    with pytest.raises(SingularBlock, match="masked retained"):
        solve_normal(apply_damping(sys_, 0.1), layout, LMConfig())


def test_cg_stall_at_iteration_cap(gpu):
    rng = np.random.default_rng(5)
    layout, blocks = random_ba_blocks(rng, 4, 10, visibility=0.7)
    damped, _, _ = build_system(layout, blocks, rng, lam=1e-4)
    with pytest.raises(CGStall, match="did not reach tolerance in 3 iterations"):
        solve_normal(damped, layout, LMConfig(cg_max_iters=3, cg_tol=1e-14))
    info = {}
    solve_normal(damped, layout, LMConfig(), Workspace(), info)
    assert info["cg_iters"] > 3


def test_unsupported_coupling_raises(gpu):
    layout = BlockLayout(["point", "point"], [2])
    blocks = [(0, 0, np.ones((2, 3))), (0, 1, np.ones((2, 3)))]
    sys_ = jtj(BlockSparseJacobian.from_blocks(layout, blocks))
    with pytest.raises(SingularBlock, match="unsupported coupling"):
        solve_normal(apply_damping(sys_, 0.1), layout, LMConfig())


@pytest.mark.parametrize("name,lam,key", [("ba_small.npz", 1e-3, "lam1e3"), ("ba_shared.npz", 1e-3, "lam1e3"),
                                          ("ba_nofocal.npz", 1e-3, "lam1e3"), ("gp_small.npz", 1e-2, "lam1e2")])
def test_explicit_solve_matches_reference_step(gpu, name, lam, key):
    """The reference's solve_normal on its own linearization (make_golden.py):
    same CG iteration count, step within 1e-8 relative."""
    z = golden(name)
    if name.startswith("gp"):
        from .test_gpu_gp import gp_from_golden
        p = gp_from_golden(z)
    else:
        from .test_gpu_ba import problem_from_golden
        p = problem_from_golden(z)
    r, jac = p.linearize(z["theta0"])
    sys_ = jtj(jac)
    sys_.gradient[:] = -jtr(jac, r)
    info = {}
    ws = Workspace()
    d = solve_normal(apply_damping(sys_, lam), p.layout, LMConfig(), ws, info)
    ref = z[f"delta_{key}"]
    # both are PCG solutions at cg_tol 1e-8 of the same reduced system, summed
    # in different orders (dense S assembled per slot, own matvec): the same
    # iteration count, steps within 1e-7 relative (largest on the focal scalars)
    assert info["cg_iters"] == int(z[f"cg_{key}"])
    assert np.abs(d - ref).max() / np.abs(ref).max() < 1e-7
    # the plan is cached per pattern in the workspace and the result is deterministic
    d2 = solve_normal(apply_damping(sys_, lam), p.layout, LMConfig(), ws, info)
    assert np.array_equal(d, d2)
    assert sum(1 for k in ws.caches if k[0] == "schur_xplan") == 1


class _Toy1D:
    """r(theta) = theta - 3 in a height-2 residual block (test_lm.py:113-124)"""

    def __init__(self):
        self.layout = BlockLayout(["focal"], [2])
        self.jac = BlockSparseJacobian.allocate(self.layout, [0], [0])
        self.jac.data[:] = [1.0, 0.0]

    def cost(self, theta):
        return float((theta[0] - 3.0) ** 2)

    def linearize(self, theta):
        return np.array([theta[0] - 3.0, 0.0]), self.jac


def test_lm_one_damped_step_value(gpu):
    theta, report = lm_solve(_Toy1D(), np.array([0.0]), LMConfig(max_iterations=1, lambda0=0.1))
    assert np.isclose(theta[0], 3.0 / 1.1)
    assert report.num_accepted == 1


def test_lm_already_optimal_terminates_immediately(gpu):
    theta, report = lm_solve(_Toy1D(), np.array([3.0]), LMConfig())
    assert report.termination == "converged_grad"
    assert len(report.iterations) == 0 and theta[0] == 3.0


def test_lm_converges_to_solution(gpu):
    theta, report = lm_solve(_Toy1D(), np.array([-20.0]), LMConfig())
    assert abs(theta[0] - 3.0) < 1e-6
    costs = report.accepted_costs
    assert all(b < a for a, b in zip(costs, costs[1:]))


def test_lm_lambda_stays_in_bounds(gpu):
    cfg = LMConfig(max_iterations=50)
    _, report = lm_solve(_Toy1D(), np.array([100.0]), cfg)
    assert all(cfg.lambda_min <= it.lam <= cfg.lambda_max for it in report.iterations)


def test_lm_solver_failure_at_lambda_max(gpu):
    cfg = LMConfig(max_iterations=5, lambda0=9e9, lambda_max=1e10, cg_max_iters=0, solver="schur_pcg")
    with pytest.raises(SolverFailure) as exc_info:
        lm_solve(_Toy1D(), np.array([0.0]), cfg)
    assert exc_info.value.report.termination == "solver_failure"
    assert not any(it.step_accepted for it in exc_info.value.report.iterations)


def test_foreign_provider_schur_matches_native_problem(gpu):
    """A duck-typed provider that hands lm_solve the BAProblem's own reference-
    layout Jacobian runs the explicit Schur path; it follows the native
    matrix-free solve (same accept sequence, final cost within 1e-9)."""
    from .test_gpu_ba import problem_from_golden
    z = golden("ba_small.npz")
    p = problem_from_golden(z)

    class Foreign:
        layout = p.layout

        def cost(self, th):
            return p.cost(th)

        def linearize(self, th):
            r, j = p.linearize(th)
            return r.copy(), j

        def post_step(self, th):
            return b2.lm.renormalize(th, p.layout)

    th_f, rep_f = lm_solve(Foreign(), z["theta0"], LMConfig(max_iterations=30))
    th_n, rep_n = lm_solve(p, z["theta0"], LMConfig(max_iterations=30))
    assert rep_f.termination == rep_n.termination == str(z["termination"])
    assert [i.step_accepted for i in rep_f.iterations] == [i.step_accepted for i in rep_n.iterations]
    assert rep_f.iterations[-1].cost_after == pytest.approx(rep_n.iterations[-1].cost_after, rel=1e-9)
    assert rep_f.iterations[-1].cost_after == pytest.approx(float(z["records"][-1, 2]), rel=1e-9)
