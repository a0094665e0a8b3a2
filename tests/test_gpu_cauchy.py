"""Cauchy robust loss -- an extension: north_star names it, the reference has
only trivial / Huber (scene.py:233-242), so there are no reference goldens.
PARITY UNPINNED: the device path is checked against the CPU oracle's
restatement (oracle/sparsesfm_port.huber, kind "cauchy": cost =
delta^2 log1p(s / delta^2), IRLS weight = 1 / (1 + s / delta^2), the
reference's cost / weight convention) on the reference's BA and GP golden
scenes. The API keeps the reference's RobustLoss validation (kind "cauchy"
raises ValueError, test_api_cpu.py); the extension is the CauchyLoss class."""
import numpy as np
import pytest

import paper_2510_13310_b200 as b2
import sparsesfm_port as orc
from paper_2510_13310_b200.scene import cauchy_cost_weight
from .conftest import ba_prob_from_golden, golden, gp_prob_from_golden
from .conftest import arrays_from_golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def test_cauchy_weight_is_the_cost_derivative():
    s = np.logspace(-6, 6, 50)
    for delta in (0.1, 1.0, 7.0):
        c, w = cauchy_cost_weight(delta, s)
        h = 1e-6 * s
        c1, _ = cauchy_cost_weight(delta, s + h)
        c0, _ = cauchy_cost_weight(delta, s - h)
        assert np.allclose((c1 - c0) / (2 * h), w, rtol=1e-6)
        assert np.all(c <= s) and np.all(w <= 1.0)


@pytest.mark.parametrize("delta", [0.5, 2.0])
def test_ba_cauchy_cost_linearize_and_trajectory(gpu, delta):
    z = golden("ba_small.npz")
    arr = arrays_from_golden(z)
    p = b2.BAProblem(arr, b2.CauchyLoss(delta))
    prob = ba_prob_from_golden(z)
    prob["loss"] = ("cauchy", delta)
    th0 = p.encode()
    assert rel(p.cost(th0), orc.ba_cost(prob, th0)) < 1e-13
    r, _ = p.linearize(th0)
    r_o, J_o = orc.ba_linearize(prob, th0)
    assert rel(r, r_o) < 1e-12
    g_o = orc.ba_dense_jacobian(prob, J_o).T @ r_o       # J^T r
    assert rel(p.gradient(th0), g_o) < 1e-10
    th, rep = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=25))
    th_o, recs, term = orc.lm_solve("ba", prob, th0, max_iterations=25)
    assert rep.termination == term
    assert [bool(i.step_accepted) for i in rep.iterations] == [bool(rc[4]) for rc in recs]
    assert rep.iterations[-1].cost_after == pytest.approx(recs[-1][2], rel=1e-9)


def test_gp_cauchy_trajectory(gpu):
    z = golden("gp_small.npz")
    p = b2.fix_gauge(b2.GPProblem(z["rays"], z["quats"], z["cam"], z["pt"], len(z["points"]),
                                  b2.CauchyLoss(0.2), False, None, seed=0))
    prob = gp_prob_from_golden(z)
    prob["loss"] = ("cauchy", 0.2)
    th0 = p.initial_theta()
    assert rel(p.cost(th0), orc.gp_cost(prob, th0)) < 1e-13
    th, rep = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=25))
    th_o, recs, term = orc.lm_solve("gp", prob, th0, max_iterations=25)
    assert rep.termination == term
    assert rep.iterations[-1].cost_after == pytest.approx(recs[-1][2], rel=1e-9)
