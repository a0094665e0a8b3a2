"""GPU: the generic block-sparse API (sparse_block.jtj / jtr / apply_damping)
against the reference's own Cython output (tests/golden/block_algebra.npz,
made by tests/golden/make_golden.py block) -- bit-identical -- and against the
oracle's dense algebra on mixed layouts."""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200.sparse_block import (BlockLayout, BlockSparseJacobian, apply_damping, jtj, jtr)
from .conftest import golden

pytestmark = pytest.mark.gpu


def jac_from(z, tag):
    lay = BlockLayout(z[f"{tag}_kinds"], z[f"{tag}_heights"])
    return BlockSparseJacobian(lay, z[f"{tag}_res_ids"], z[f"{tag}_param_ids"], z[f"{tag}_data"],
                               z[f"{tag}_data_off"])


@pytest.mark.parametrize("tag", ["ba", "gp"])
def test_block_algebra_bitwise_vs_reference(gpu, tag):
    z = golden("block_algebra.npz")
    j = jac_from(z, tag)
    sys_ = jtj(j)
    assert np.array_equal(sys_.off_keys, z[f"{tag}_off_keys"])
    assert np.array_equal(sys_.data, z[f"{tag}_jtj"])            # bit-identical
    assert np.array_equal(jtr(j, z[f"{tag}_r"]), z[f"{tag}_jtr"])
    assert np.array_equal(apply_damping(sys_, 0.37).data, z[f"{tag}_damped"])


def dense(j):
    lay = j.layout
    A = np.zeros((lay.total_residuals, lay.total_params))
    for e in range(j.num_entries):
        r0, p0 = lay.residual_offsets[j.res_ids[e]], lay.param_offsets[j.param_ids[e]]
        blk = j.entry_block(e)
        A[r0:r0 + blk.shape[0], p0:p0 + blk.shape[1]] = blk
    return A


def test_block_algebra_mixed_layout_vs_dense(gpu):
    rng = np.random.default_rng(4)
    kinds = rng.integers(0, 6, size=40)
    heights = rng.choice([2, 3], size=60)
    lay = BlockLayout(kinds, heights)
    blocks = []
    for r in range(60):
        for p in sorted(rng.choice(40, size=int(rng.integers(1, 5)), replace=False)):
            blocks.append((r, int(p), rng.normal(size=(int(heights[r]), int(lay.widths[p])))))
    j = BlockSparseJacobian.from_blocks(lay, blocks)
    A = dense(j)
    sys_ = jtj(j)
    full = A.T @ A
    for k in range(lay.num_param_blocks):
        o, w = lay.param_offsets[k], lay.widths[k]
        assert np.allclose(sys_.diag_block(k), full[o:o + w, o:o + w], rtol=1e-13, atol=1e-12)
    for i, (a, b) in enumerate(sys_.off_keys):
        oa, wa, ob, wb = lay.param_offsets[a], lay.widths[a], lay.param_offsets[b], lay.widths[b]
        assert np.allclose(sys_.off_block(i), full[oa:oa + wa, ob:ob + wb], rtol=1e-13, atol=1e-12)
    r = rng.normal(size=lay.total_residuals)
    assert np.allclose(jtr(j, r), A.T @ r, rtol=1e-13, atol=1e-12)
    d = apply_damping(sys_, 0.5)
    assert d.lam == 0.5 and sys_.lam == 0.0
    for k in range(lay.num_param_blocks):
        assert np.array_equal(np.diag(d.diag_block(k)), np.diag(sys_.diag_block(k)) * 1.5)


def test_dense_solver_step_matches_exact_solve(gpu):     # lm.py:170-220 on the device
    import sparsesfm_port as orc
    from .conftest import ba_prob_from_golden
    from .test_gpu_ba import problem_from_golden
    z = golden("ba_small.npz")
    p = problem_from_golden(z)
    r, jac = p.linearize(z["theta0"])
    sys_ = jtj(jac)
    sys_.gradient[:] = -jtr(jac, r)
    damped = apply_damping(sys_, 1e-3)
    info = {}
    d = b2.lm.solve_normal(damped, p.layout, b2.LMConfig(solver="dense"), b2.Workspace(), info)
    prob = ba_prob_from_golden(z)
    r_o, J_o = orc.ba_linearize(prob, z["theta0"])
    Jd = orc.ba_dense_jacobian(prob, J_o)
    A = Jd.T @ Jd
    A[np.diag_indices_from(A)] *= 1.001
    exact = np.linalg.solve(A, -(Jd.T @ r_o))
    assert np.abs(d - exact).max() / np.abs(exact).max() < 1e-9
    assert info["cg_iters"] == 0


def test_lm_solve_dense_solver_and_foreign_provider(gpu):
    from .test_gpu_ba import problem_from_golden
    z = golden("ba_small.npz")
    p = problem_from_golden(z)
    th, rep = b2.lm_solve(p, z["theta0"], b2.LMConfig(solver="dense", max_iterations=30))
    assert rep.termination == "converged_cost"
    assert rep.iterations[-1].cost_after == pytest.approx(float(z["records"][-1, 2]), rel=1e-8)
    assert all(i.cg_iters == 0 for i in rep.iterations)
    # tensor in, tensor out (as on the native path)
    tht, rept = b2.lm_solve(p, gpu.as_tensor(z["theta0"]).cuda(), b2.LMConfig(solver="dense", max_iterations=30))
    assert isinstance(tht, gpu.Tensor) and tht.is_cuda
    assert np.array_equal(tht.cpu().numpy(), th) and rept.termination == rep.termination

    class Line:                     # a duck-typed provider (lm.py:730-739): fit y = a x + b
        def __init__(self):
            self.layout = BlockLayout(np.array([2], np.int8), np.full(20, 2, np.int32))  # one 'focal'... width-1
            self.x = np.linspace(0, 1, 40)
            self.y = 3.0 * self.x + 0.5

        def residual(self, th):
            return th[0] * self.x + (self.y[0] - 0.5) * 0 + 0.5 - self.y

        def cost(self, th):
            return float(np.sum(self.residual(th) ** 2))

        def linearize(self, th):
            blocks = [(k, 0, self.x[2 * k:2 * k + 2].reshape(2, 1)) for k in range(20)]
            return self.residual(th), BlockSparseJacobian.from_blocks(self.layout, blocks)

    prov = Line()
    th, rep = b2.lm_solve(prov, np.array([0.0]), b2.LMConfig(solver="dense"))
    assert th[0] == pytest.approx(3.0, rel=1e-9)
    th, rep = b2.lm_solve(prov, np.array([0.0]), b2.LMConfig())    # default: explicit-system Schur PCG
    assert th[0] == pytest.approx(3.0, rel=1e-9)
    assert rep.iterations[0].cg_iters >= 1
