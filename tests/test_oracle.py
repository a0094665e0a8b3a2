"""Pin the CPU oracle (oracle/sparsesfm_port.py) to the reference's golden
vectors (tests/golden, produced by tests/golden/make_golden.py from the
unmodified reference). CPU only."""
import numpy as np
import pytest

import sparsesfm_port as orc
from .conftest import ba_prob_from_golden, golden, gp_prob_from_golden, summary


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("name", ["ba_small.npz", "ba_nofocal.npz", "ba_bal.npz", "ba_shared.npz"])
def test_ba_cost_residual_jacobian_gradient(name):
    z = golden(name)
    prob = ba_prob_from_golden(z)
    th = z["theta0"]
    assert orc.ba_cost(prob, th) == pytest.approx(float(z["cost0"]), rel=1e-13)
    r, J = orc.ba_linearize(prob, th)
    assert rel(r, z["r0"]) < 1e-13
    assert rel(orc.ref_layout(J, [7, 3, 1] if prob["focal_mode"] else [7, 3]), z["J0"]) < 1e-12
    Jd = orc.ba_dense_jacobian(prob, J)
    assert rel(Jd.T @ r, z["grad0"]) < 1e-11


@pytest.mark.parametrize("name", ["ba_small.npz", "ba_shared.npz"])
def test_ba_solve_normal_matches_reference(name):
    z = golden(name)
    prob = ba_prob_from_golden(z)
    r, J = orc.ba_linearize(prob, z["theta0"])
    Jd = orc.ba_dense_jacobian(prob, J)
    d, it = orc.schur_pcg_solve(Jd.T @ Jd, -(Jd.T @ r), orc.ba_param_blocks(prob), 1e-3)
    assert rel(d, z["delta_lam1e3"]) < 1e-7
    assert abs(it - int(z["cg_lam1e3"])) <= 2


@pytest.mark.parametrize("name", ["ba_small.npz", "ba_nofocal.npz", "ba_bal.npz", "ba_shared.npz"])
def test_ba_lm_solve_matches_reference(name):
    z = golden(name)
    prob = ba_prob_from_golden(z)
    th, recs, term = orc.lm_solve("ba", prob, z["theta0"], max_iterations=30)
    ref = z["records"]
    assert term == str(z["termination"])
    assert len(recs) == len(ref)
    assert [bool(x[4]) for x in recs] == [bool(x) for x in ref[:, 4]]
    assert recs[-1][2] == pytest.approx(ref[-1, 2], rel=1e-10)


@pytest.mark.parametrize("name", ["gp_small.npz", "gp_depth.npz"])
def test_gp_cost_residual_jacobian_gradient(name):
    z = golden(name)
    prob = gp_prob_from_golden(z)
    th = z["theta0"]
    assert orc.gp_cost(prob, th) == pytest.approx(float(z["cost0"]), rel=1e-13)
    r, J = orc.gp_linearize(prob, th)
    assert rel(r, z["r0"]) < 1e-13
    assert rel(orc.ref_layout(J, [3, 3] if prob["depth_mode"] else [3, 3, 1]), z["J0"]) < 1e-13
    Jd = orc.gp_dense_jacobian(prob, J)
    assert rel(Jd.T @ r, z["grad0"]) < 1e-11


def test_gp_solve_and_post_step():
    z = golden("gp_small.npz")
    prob = gp_prob_from_golden(z)
    r, J = orc.gp_linearize(prob, z["theta0"])
    Jd = orc.gp_dense_jacobian(prob, J)
    d, it = orc.schur_pcg_solve(Jd.T @ Jd, -(Jd.T @ r), orc.gp_param_blocks(prob), 1e-2)
    assert rel(d, z["delta_lam1e2"]) < 1e-7
    th = z["theta0"]
    probe = orc.gp_post_step(prob, th + 0.1 * np.sin(np.arange(len(th))))
    assert rel(probe, z["post_step_probe"]) < 1e-14


@pytest.mark.parametrize("name", ["gp_small.npz", "gp_depth.npz"])
def test_gp_lm_solve_matches_reference(name):
    z = golden(name)
    prob = gp_prob_from_golden(z)
    th, recs, term = orc.lm_solve("gp", prob, z["theta0"], max_iterations=40 if "small" in name else 30)
    ref = z["records"]
    assert term == str(z["termination"])
    assert [bool(x[4]) for x in recs] == [bool(x) for x in ref[:, 4]]
    assert recs[-1][2] == pytest.approx(ref[-1, 2], rel=1e-8)
    assert np.abs(th - z["theta_final"]).max() < 1e-8


def test_pattern_keys_match_reference():
    z = golden("ba_small.npz")
    C, P = len(z["quats"]), len(z["points"])
    per_obs = [(int(c), C + int(p), C + P + int(c)) for c, p in zip(z["cam"], z["pt"])]
    assert np.array_equal(orc.jtj_off_keys(per_obs), z["off_keys"])
    ret_lists = {}
    for c, p in zip(z["cam"], z["pt"]):
        ret_lists.setdefault(int(p), []).extend([int(c), C + int(c)])
    widths = [7] * C + [1] * C
    assert np.array_equal(orc.schur_slots(ret_lists.values(), widths), z["schur_slots"])


def test_survey_goldens_recorded():
    s = summary()
    assert s["c1"]["termination"] == "converged_cost"
    assert s["c1"]["iterations"] == 22
    assert s["c1"]["final_cost"] == pytest.approx(20994.9852668881, rel=1e-12)
    assert s["c2"]["final_cost"] == pytest.approx(0.990124903324729, rel=1e-12)


@pytest.mark.parametrize("tag", ["ba", "gp"])
def test_block_algebra_golden_vs_dense(tag):
    """The reference's jtj / jtr fixture (tests/golden/block_algebra.npz) agrees
    with dense J^T J / J^T r built from the same blocks (CPU, no device)."""
    from paper_2510_13310_b200.sparse_block import BlockLayout, BlockSparseJacobian, BlockNormalSystem
    z = golden("block_algebra.npz")
    lay = BlockLayout(z[f"{tag}_kinds"], z[f"{tag}_heights"])
    j = BlockSparseJacobian(lay, z[f"{tag}_res_ids"], z[f"{tag}_param_ids"], z[f"{tag}_data"],
                            z[f"{tag}_data_off"])
    A = np.zeros((lay.total_residuals, lay.total_params))
    for e in range(j.num_entries):
        r0, p0 = lay.residual_offsets[j.res_ids[e]], lay.param_offsets[j.param_ids[e]]
        blk = j.entry_block(e)
        A[r0:r0 + blk.shape[0], p0:p0 + blk.shape[1]] = blk
    full = A.T @ A
    sys_ = BlockNormalSystem.empty(lay, z[f"{tag}_off_keys"])
    sys_.data[:] = z[f"{tag}_jtj"]
    for k in range(lay.num_param_blocks):
        o, w = lay.param_offsets[k], lay.widths[k]
        assert np.allclose(sys_.diag_block(k), full[o:o + w, o:o + w], rtol=1e-12, atol=1e-10)
    assert rel(z[f"{tag}_jtr"], A.T @ z[f"{tag}_r"]) < 1e-12
