"""GPU parity at scale against the UNMODIFIED reference.

Fixtures (tests/golden/scale_*.npz, made by tests/golden/make_golden_scale.py
from oracle/_ref in the build container) hold the reference's own runs:

  C3   BA 1700 cams / 150k pts / 680k obs (the survey's trimmed recipe), 10 its
  C5s  BA 5000 cams / 200k pts / 2M obs (a 5000-camera C5 sample), 10 its
  C4   GP 20 its (Huber 0.1) -> BA 10 its (Huber 1.0), 1000 / 500k / 4M

Here the inputs are regenerated bit-identically by the array-native replay
(paper_2510_13310_b200/synth.py; the sha256 of the arrays must equal the
reference's) and solved on the device through the public API. Bars (SURVEY.md
8(d)): the same accept/reject and lambda sequence; BA final cost and RMSE
within 1e-10 / 1e-6 relative and camera centres / points within 1e-8 x scene
diameter after a Sim(3) registration onto the reference's cameras; GP centres
and points within 1e-8 absolute. Integer structures (JtJPattern.off_keys, the
_SchurPlan slot list) are bit-exact at C3. CG iteration counts are reported
per LM iteration; the bar on them is `cg_count_ok`.
"""
import hashlib
import os

import numpy as np
import pytest

import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import synth
from .conftest import GOLDEN

pytestmark = pytest.mark.gpu
PERTURB = dict(rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)


def load(name):
    path = os.path.join(GOLDEN, f"scale_{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing reference fixture {path} (tests/golden/make_golden_scale.py {name})")
    return np.load(path)


def digest(a) -> str:
    h = hashlib.sha256()
    for x in (a.quats, a.centers, a.focals, a.points, a.cam_idx.astype(np.int64), a.pt_idx.astype(np.int64),
              a.pixels):
        h.update(np.ascontiguousarray(x).tobytes())
    return h.hexdigest()


def scene(C, P, k, trim=None, perturb=True):
    _, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=C, num_points=P, visibility_fraction=k / C,
                                                     pixel_noise_sigma=1.0, seed=0))
    arr = synth.perturb_arrays(obs, **PERTURB) if perturb else obs
    return synth.trim_points_arrays(arr, trim) if trim is not None else arr


def umeyama(x, y):
    """s, R, t with y ~ s R x + t (least squares over rows)"""
    mx, my = x.mean(0), y.mean(0)
    xc, yc = x - mx, y - my
    cov = yc.T @ xc / len(x)
    U, D, Vt = np.linalg.svd(cov)
    S = np.eye(3)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        S[2, 2] = -1
    R = U @ S @ Vt
    s = np.trace(np.diag(D) @ S) / (xc ** 2).sum(1).mean()
    return s, R, my - s * R @ mx


def cg_count_ok(ours, ref):
    """The CG iteration count of a damped solve is a rounding-sensitive
    quantity: the PCG residual of these ill-conditioned reduced systems
    plateaus near the stop tolerance, so summing in a different order can move
    the stop by several iterations while the step agrees to ~1e-11 (the final
    parameters below). The bar is on the CG work: total within 5 % of the
    reference's and every count within 25 %. The measured counts are recorded
    (and listed in DESIGN.md) next to the reference's own spread under a 1e-13
    perturbation of theta0."""
    ours, ref = np.asarray(ours, float), np.asarray(ref, float)
    return bool(abs(ours.sum() - ref.sum()) <= 0.05 * ref.sum() and (np.abs(ours - ref) <= 0.25 * ref).all())


def check_ba_run(z, prob, th, rep, prefix="", report=None):
    """compare one device BA solve with the reference's; every figure is
    collected into `report` (printed and recorded) before the asserts"""
    from paper_2510_13310_b200.pipeline import reproj_rmse_device
    recs = z[prefix + "records"]
    C = z[prefix + "cam_theta"].shape[0]
    got = np.array([(i.cost_before, i.cost_after, i.lam, float(i.step_accepted)) for i in rep.iterations])
    cg = [i.cg_iters for i in rep.iterations]
    final_rel = abs(rep.iterations[-1].cost_after - float(z[prefix + "final_cost"])) / float(z[prefix + "final_cost"])
    rmse = reproj_rmse_device(prob, th)
    rmse_rel = abs(rmse - float(z[prefix + "rmse"])) / float(z[prefix + "rmse"])
    # parameters after Sim(3) registration of our camera centres onto the reference's
    th = np.asarray(th)
    P = (len(th) - 7 * C - len(z[prefix + "focals"])) // 3
    ours_c = th[:7 * C].reshape(C, 7)[:, 4:]
    ref_c = z[prefix + "cam_theta"][:, 4:]
    s, R, t = umeyama(ours_c, ref_c)
    diam = float(z[prefix + "diameter"])
    c_err = np.abs((s * ours_c @ R.T + t) - ref_c).max() / diam
    pts = th[7 * C:7 * C + 3 * P].reshape(P, 3)[z[prefix + "point_idx"]]
    p_err = np.abs((s * pts @ R.T + t) - z[prefix + "points"]).max() / diam
    f_err = np.abs(th[7 * C + 3 * P:] - z[prefix + "focals"]).max() / np.abs(z[prefix + "focals"]).max()
    out = dict(termination=rep.termination, iterations=len(cg), cg_ours=cg, cg_ref=recs[:, 5].astype(int).tolist(),
               accepted=got[:, 3].astype(int).tolist(), final_cost_rel=final_rel, rmse=rmse, rmse_rel=rmse_rel,
               center_err_over_diam=c_err, point_err_over_diam=p_err, focal_rel=f_err)
    if report is not None:
        report.update(out)
    print(prefix or "ba", out)
    assert rep.termination == str(z[prefix + "termination"])
    assert len(rep.iterations) == len(recs)
    assert np.array_equal(got[:, 3], recs[:, 4]), "accept sequence"
    assert np.array_equal(got[:, 2], recs[:, 3]), "lambda sequence"
    assert final_rel < 1e-10, final_rel
    assert rmse_rel < 1e-6, rmse_rel
    assert c_err < 1e-8 and p_err < 1e-8, (c_err, p_err)
    assert f_err < 1e-8, f_err
    assert cg_count_ok(cg, recs[:, 5]), (cg, recs[:, 5].tolist())
    return out


def test_c3_integer_structures_and_solve(gpu, record_property):
    z = load("c3")
    arr = scene(1700, 150000, 5, trim=80000)
    assert arr.num_observations == 680000
    assert digest(arr) == str(z["input_digest"])
    prob = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
    th0 = prob.encode()
    assert prob.cost(th0) == pytest.approx(float(z["cost0"]), rel=1e-12)
    pat = prob.export_pattern()
    keys = np.ascontiguousarray(pat["off_keys"].astype(np.int32))
    slots = np.ascontiguousarray(pat["schur_slots"].astype(np.int32))
    assert len(keys) == int(z["n_off"]) and len(slots) == int(z["n_slots"])
    assert hashlib.sha256(keys.tobytes()).hexdigest() == str(z["off_keys_digest"])
    assert hashlib.sha256(slots.tobytes()).hexdigest() == str(z["slots_digest"])
    rep_d = {}
    record_property("c3", rep_d)
    th, rep = b2.lm_solve(prob, th0, b2.LMConfig(max_iterations=10))
    check_ba_run(z, prob, th, rep, report=rep_d)


def test_c5_sample_solve(gpu, record_property):
    z = load("c5s")
    arr = scene(5000, 200000, 10)
    assert digest(arr) == str(z["input_digest"])
    prob = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
    th0 = prob.encode()
    assert prob.cost(th0) == pytest.approx(float(z["cost0"]), rel=1e-12)
    rep_d = {}
    record_property("c5s", rep_d)
    th, rep = b2.lm_solve(prob, th0, b2.LMConfig(max_iterations=10))
    check_ba_run(z, prob, th, rep, report=rep_d)


def test_c4_gp_then_ba(gpu, record_property):
    z = load("c4")
    obs = scene(1000, 500000, 8, perturb=False)
    assert digest(obs) == str(z["input_digest"])
    gp_scene, rep_gp = b2.run_gp(obs, depth_mode=False, loss=b2.RobustLoss("huber", 0.1),
                                 config=b2.LMConfig(max_iterations=20), seed=0)
    recs = z["gp_records"]
    c_err = np.abs(gp_scene.centers - z["gp_centers"]).max()
    p_err = np.abs(gp_scene.points[z["gp_point_idx"]] - z["gp_points"]).max()
    rep_d = dict(gp_cg_ours=[i.cg_iters for i in rep_gp.iterations], gp_cg_ref=recs[:, 5].astype(int).tolist(),
                 gp_final_cost_rel=abs(rep_gp.iterations[-1].cost_after - float(z["gp_final_cost"]))
                 / float(z["gp_final_cost"]), gp_center_err=c_err, gp_point_err=p_err,
                 gp_termination=rep_gp.termination)
    record_property("c4", rep_d)
    print("gp", rep_d)
    assert rep_gp.termination == str(z["gp_termination"])
    assert [float(i.step_accepted) for i in rep_gp.iterations] == recs[:, 4].tolist()
    assert [i.lam for i in rep_gp.iterations] == recs[:, 3].tolist()
    assert rep_d["gp_final_cost_rel"] < 1e-10
    assert c_err < 1e-8 and p_err < 1e-8, (c_err, p_err)
    assert cg_count_ok(rep_d["gp_cg_ours"], recs[:, 5])
    prob = b2.BAProblem(gp_scene, b2.RobustLoss("huber", 1.0))
    th0 = prob.encode()
    assert prob.cost(th0) == pytest.approx(float(z["ba_cost0"]), rel=1e-9)
    th, rep = b2.lm_solve(prob, th0, b2.LMConfig(max_iterations=10))
    check_ba_run(z, prob, th, rep, prefix="ba_", report=rep_d)
    # the device pipeline (run_global_sfm) takes the same trajectory
    _, prep = b2.run_global_sfm(obs)
    assert [i.cost_after for i in prep.gp.iterations] == [i.cost_after for i in rep_gp.iterations]
    assert [i.step_accepted for i in prep.ba.iterations] == [i.step_accepted for i in rep.iterations]
    assert prep.ba.iterations[-1].cost_after == pytest.approx(rep.iterations[-1].cost_after, rel=1e-12)
