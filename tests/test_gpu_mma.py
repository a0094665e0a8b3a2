"""Tile-group sums on the fp64 tensor cores against the scalar kernels.

ba_k_lin_tile_mma (the camera blocks Jc^T Jc and Jc^T r of linearize,
ba.py:140-194 + sparse_block.jtj / jtr) and ba_k_precond_mma (the Schur
diagonal blocks and b_red, lm.py:599-626) sum a camera tile group with DMMA
m8n8k4 when SSFM_MMA=1 (opt-in: slower at C5); the default
keeps the scalar per-thread sums. Both are fixed-order reductions of the same
per-observation terms, so they agree to rounding: the gradient to 1e-12; a
damped step to the CG tolerance (the preconditioner's rounding moves the CG
iterates), so the costs after each step to 1e-8 relative and the final cost
and parameters to the parity bars of tests/test_gpu_ba.py; the DMMA path is
deterministic run to run.
"""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from .conftest import golden
from .test_gpu_ba import problem_from_golden
from .test_gpu_lm_graph import env

pytestmark = pytest.mark.gpu

TWO_PASS = {"SSFM_FUSED": "0", "SSFM_PCG_GRAPH": "0", "SSFM_LM_GRAPH": "0"}


def solve(z, mma, iters=40):
    with env(dict(TWO_PASS, SSFM_MMA=mma)):
        p = problem_from_golden(z)
        p._native_handle()
    th, rep = b2.lm_solve(p, z["theta0"].copy(), b2.LMConfig(max_iterations=iters))
    g = p.gradient(z["theta0"])
    return np.asarray(th), rep, np.asarray(g)


@pytest.mark.parametrize("name", ["ba_small.npz", "ba_shared.npz", "ba_nofocal.npz", "ba_bal.npz"])
def test_mma_group_sums_match_scalar(gpu, name):
    z = golden(name)
    th1, rep1, g1 = solve(z, "1")
    th0, rep0, g0 = solve(z, "0")
    scale = np.max(np.abs(g0))
    assert np.max(np.abs(g1 - g0)) <= 1e-12 * scale
    assert [i.step_accepted for i in rep1.iterations] == [i.step_accepted for i in rep0.iterations]
    assert rep1.termination == rep0.termination
    c1 = np.array([i.cost_after for i in rep1.iterations if i.step_accepted])
    c0 = np.array([i.cost_after for i in rep0.iterations if i.step_accepted])
    np.testing.assert_allclose(c1, c0, rtol=1e-8, atol=0)
    np.testing.assert_allclose(c1[-1], c0[-1], rtol=1e-10, atol=0)
    diam = max(1.0, float(np.max(np.abs(th0))))
    assert np.max(np.abs(th1 - th0)) <= 1e-8 * diam
    d_cg = [abs(a.cg_iters - b.cg_iters) for a, b in zip(rep1.iterations, rep0.iterations)]
    assert max(d_cg) <= 2


def test_mma_deterministic(gpu):
    z = golden("ba_small.npz")
    th_a, rep_a, g_a = solve(z, "1")
    th_b, rep_b, g_b = solve(z, "1")
    assert np.array_equal(g_a, g_b)
    assert np.array_equal(th_a, th_b)
    assert [i.cg_iters for i in rep_a.iterations] == [i.cg_iters for i in rep_b.iterations]
