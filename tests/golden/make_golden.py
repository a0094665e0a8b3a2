"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref, built by oracle/build_ref.sh
from /root/reference):

    python tests/golden/make_golden.py

Every fixture records reference inputs and outputs for the hot path; the
tests compare the oracle port (oracle/sparsesfm_port.py) and the B200 path
against them. Nothing here runs at test time.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
os.environ["SPARSESFM_BACKEND"] = "cython"

import sparsesfm as ref  # noqa: E402
from sparsesfm import synth_metrics as rsm  # noqa: E402
from sparsesfm.lm import _get_schur_plan  # noqa: E402
from sparsesfm.scene import (project, quat_from_axis_angle, quat_multiply,  # noqa: E402
                             scene_to_arrays)
from sparsesfm.sparse_block import apply_damping, jtj, jtr  # noqa: E402


def arrays_of(scene):
    a = scene_to_arrays(scene)
    return dict(quats=a.quats, centers=a.centers, focals=a.focals, pps=a.pps, dists=a.dists,
                points=a.points, cam=a.cam_idx, pt=a.pt_idx, pixels=a.pixels,
                depths=a.depths if a.depths is not None else np.zeros(0))


def records(rep):
    return np.array([(i.iteration, i.cost_before, i.cost_after, i.lam, float(i.step_accepted),
                      i.cg_iters) for i in rep.iterations], dtype=np.float64).reshape(-1, 6)


def schur_slot_pairs(sys, ws):
    plan = _get_schur_plan(sys, ws)
    ret_off = plan.ret_s_off
    ra = np.searchsorted(ret_off, plan.slot_row, side="right") - 1
    rb = np.searchsorted(ret_off, plan.slot_col, side="right") - 1
    return np.stack([ra, rb], axis=1).astype(np.int64)


def ba_fixture(name, scene, loss, optimize_focal=True, shared_focal=False, iters=30, model_tag=None):
    prob = ref.BAProblem(scene, loss, optimize_focal, shared_focal)
    th0 = prob.encode()
    cost0 = prob.cost(th0)
    r0, J0 = prob.linearize(th0)
    r0 = r0.copy()
    Jd = J0.data.copy()
    g0 = jtr(J0, r0)
    sys_ = jtj(J0)
    sys_.gradient[:] = -g0
    ws = ref.Workspace()
    delta = ref.solve_normal(apply_damping(sys_, 1e-3), prob.layout, ref.LMConfig(), ws,
                             info := {})
    slots = schur_slot_pairs(apply_damping(sys_, 1e-3), ws)
    th, rep = ref.lm_solve(prob, th0, ref.LMConfig(max_iterations=iters))
    out = arrays_of(scene)
    out.update(theta0=th0, cost0=cost0, r0=r0, J0=Jd, grad0=g0, off_keys=sys_.off_keys.astype(np.int64),
               schur_slots=slots, delta_lam1e3=delta, cg_lam1e3=info.get("cg_iters", 0),
               theta_final=th, records=records(rep), termination=rep.termination,
               optimize_focal=int(optimize_focal), shared_focal=int(shared_focal),
               loss_kind=loss.kind, loss_delta=loss.delta,
               model=scene.cameras[0].model_tag)
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, rep.termination, len(rep.iterations), "its, final", rep.iterations[-1].cost_after)


def gp_fixture(name, scene, loss, depth_mode, iters=40):
    prob = ref.fix_gauge(ref.make_rays(scene, depth_mode, loss, seed=0))
    th0 = prob.initial_theta()
    cost0 = prob.cost(th0)
    r0, J0 = prob.linearize(th0)
    r0 = r0.copy()
    Jd = J0.data.copy()
    g0 = jtr(J0, r0)
    sys_ = jtj(J0)
    sys_.gradient[:] = -g0
    ws = ref.Workspace()
    delta = ref.solve_normal(apply_damping(sys_, 1e-2), prob.layout, ref.LMConfig(), ws, info := {})
    slots = schur_slot_pairs(apply_damping(sys_, 1e-2), ws)
    post = prob.post_step(th0 + 0.1 * np.sin(np.arange(len(th0))))
    th, rep = ref.lm_solve(prob, th0, ref.LMConfig(max_iterations=iters))
    out = arrays_of(scene)
    out.update(rays=prob.rays, ray_depths=prob.depths if prob.depths is not None else np.zeros(0),
               theta0=th0, cost0=cost0, r0=r0, J0=Jd, grad0=g0, off_keys=sys_.off_keys.astype(np.int64),
               schur_slots=slots, delta_lam1e2=delta, cg_lam1e2=info.get("cg_iters", 0),
               post_step_probe=post, theta_final=th, records=records(rep), termination=rep.termination,
               depth_mode=int(depth_mode), loss_kind=loss.kind, loss_delta=loss.delta)
    np.savez_compressed(os.path.join(HERE, name), **out)
    print(name, rep.termination, len(rep.iterations), "its, final", rep.iterations[-1].cost_after)


def bal_scene(seed=5):
    """BAL-radial scene: cameras look down -z (rotation composed with 180 deg
    about x), pixels from the reference's own bal_radial projection + noise."""
    truth, _ = rsm.generate(rsm.SynthConfig(num_cameras=6, num_points=80, visibility_fraction=4 / 6,
                                            radius=8.0, focal=300.0, seed=seed))
    rng = np.random.default_rng(seed)
    flip = quat_from_axis_angle([1.0, 0.0, 0.0], np.pi)
    cams = []
    for c in truth.cameras:
        cams.append(ref.Camera(quat_multiply(flip, np.asarray(c.rotation)), c.center, c.focal,
                               np.array([1.5, -2.0]), "bal_radial",
                               np.array([rng.uniform(-0.05, 0.05), rng.uniform(-0.01, 0.01)])))
    obs = []
    for o in truth.observations:
        px = project(cams[o.camera_id], truth.points[o.point_id]) + rng.normal(0, 0.5, 2)
        obs.append(ref.Observation(o.camera_id, o.point_id, px))
    scene = ref.Scene(cams, truth.points, obs)
    return rsm.perturb(scene, rot_deg=0.5, center_frac=0.005, focal_frac=0.01, point_frac=0.003, seed=2)


def digest(arrs):
    h = hashlib.sha256()
    for k in ("quats", "centers", "focals", "points", "cam", "pt", "pixels", "depths"):
        h.update(np.ascontiguousarray(arrs[k]).tobytes())
    return h.hexdigest()


def shared_focal_fixture():
    """BA with ONE focal shared by every camera (ba.py:49, 61, 77, 89)."""
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=8, num_points=120, visibility_fraction=0.5,
                                              pixel_noise_sigma=1.0, seed=3))
    start = rsm.perturb(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    ba_fixture("ba_shared.npz", start, ref.RobustLoss("huber", 1.0), shared_focal=True)


def block_algebra_fixture():
    """Reference jtj / jtr / apply_damping outputs (Cython backend) on the
    ba_small and gp_small linearizations: pins the generic block API."""
    out = {}
    for tag, z in (("ba", np.load(os.path.join(HERE, "ba_small.npz"))),
                   ("gp", np.load(os.path.join(HERE, "gp_small.npz")))):
        if tag == "ba":
            sc = rsm.generate(rsm.SynthConfig(num_cameras=8, num_points=120, visibility_fraction=0.5,
                                              pixel_noise_sigma=1.0, seed=3))[1]
            sc = rsm.perturb(sc, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
            prob = ref.BAProblem(sc, ref.RobustLoss("huber", 1.0))
            th = prob.encode()
        else:
            sc = rsm.generate(rsm.SynthConfig(num_cameras=10, num_points=200, visibility_fraction=0.4,
                                              pixel_noise_sigma=0.5, seed=2))[1]
            prob = ref.fix_gauge(ref.make_rays(sc, False, ref.RobustLoss("huber", 0.1), seed=0))
            th = prob.initial_theta()
        r, J = prob.linearize(th)
        sys_ = jtj(J)
        g = jtr(J, r)
        damped = apply_damping(sys_, 0.37)
        out[f"{tag}_res_ids"] = J.res_ids
        out[f"{tag}_param_ids"] = J.param_ids
        out[f"{tag}_data"] = J.data.copy()
        out[f"{tag}_data_off"] = J.data_off
        out[f"{tag}_r"] = r.copy()
        out[f"{tag}_kinds"] = prob.layout.kind_codes
        out[f"{tag}_heights"] = prob.layout.residual_heights
        out[f"{tag}_jtj"] = sys_.data.copy()
        out[f"{tag}_off_keys"] = sys_.off_keys
        out[f"{tag}_jtr"] = g.copy()
        out[f"{tag}_damped"] = damped.data.copy()
    np.savez_compressed(os.path.join(HERE, "block_algebra.npz"), **out)
    print("block_algebra.npz", {k: v.shape for k, v in out.items() if k.endswith("jtj")})


def metrics_fixture():
    """Reference synth_metrics.align (sim3, se3), center_rmse and rotation_auc
    on a perturbed scene moved by a known similarity: pins the device metrics
    (paper_2510_13310_b200/metrics.py)."""
    from sparsesfm.scene import Camera, Point3D, Scene, quat_to_matrix
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=60, num_points=400, visibility_fraction=0.2,
                                              pixel_noise_sigma=1.0, seed=11))
    est = rsm.perturb(obs, rot_deg=2.0, center_frac=0.02, focal_frac=0.0, point_frac=0.01, seed=4)
    qs = quat_from_axis_angle(np.array([0.3, -0.5, 0.8]), 0.7)
    Rs, s, t = quat_to_matrix(qs), 1.7, np.array([0.5, -2.0, 3.0])
    qs_c = np.array([qs[0], -qs[1], -qs[2], -qs[3]])
    moved = Scene([Camera(quat_multiply(c.rotation, qs_c), s * Rs @ c.center + t, c.focal,
                          c.principal_point.copy(), c.model_tag, c.bal_distortion.copy()) for c in est.cameras],
                  [Point3D(s * Rs @ p.position + t) for p in est.points], list(est.observations))
    taus = np.array([1.0, 2.0, 5.0, 10.0, 30.0])
    out = {"taus": taus}
    a = scene_to_arrays(moved)
    tr = scene_to_arrays(truth)
    out.update(est_quats=a.quats, est_centers=a.centers, est_points=a.points, true_quats=tr.quats,
               true_centers=tr.centers)
    for kind in ("sim3", "se3"):
        al, aligned = rsm.align(moved, truth, kind)
        b = scene_to_arrays(aligned)
        out[f"{kind}_rotation"] = al.rotation
        out[f"{kind}_translation"] = al.translation
        out[f"{kind}_scale"] = al.scale
        out[f"{kind}_quats"] = b.quats
        out[f"{kind}_centers"] = b.centers
        out[f"{kind}_points"] = b.points
        out[f"{kind}_center_rmse"] = rsm.center_rmse(aligned, truth)
        auc = rsm.rotation_auc(aligned, truth, taus)
        out[f"{kind}_auc"] = np.array([auc[float(x)] for x in taus])
    auc = rsm.rotation_auc(moved, truth, taus)
    out["moved_auc"] = np.array([auc[float(x)] for x in taus])
    out["moved_center_rmse"] = rsm.center_rmse(moved, truth)
    np.savez_compressed(os.path.join(HERE, "metrics.npz"), **out)
    print("metrics.npz", out["sim3_scale"], out["sim3_auc"], out["moved_auc"])


def bal_cases():
    """BAL texts for the reader (valid files and every error path of io.read_bal)"""
    truth, _ = rsm.generate(rsm.SynthConfig(num_cameras=20, num_points=300, visibility_fraction=0.3,
                                            pixel_noise_sigma=1.0, seed=9))
    rng = np.random.default_rng(3)
    a = scene_to_arrays(truth)
    lines = [f"{len(a.quats)} {len(a.points)} {len(a.cam_idx)}"]
    lines += [f"{c} {p} {float(u)!r} {float(v)!r}" for c, p, (u, v) in zip(a.cam_idx, a.pt_idx, a.pixels)]
    for i in range(len(a.quats)):
        lines += [repr(float(x)) for x in np.concatenate([rng.normal(size=3) * 0.3, rng.normal(size=3),
                                                          [500 + 50 * rng.random()], rng.normal(size=2) * 1e-3])]
    lines += [" ".join(repr(float(x)) for x in pt) for pt in a.points]
    synth_text = "\n".join(lines) + "\n"
    mini = ("# a BAL file with comments\r\n3 4 7  # header\r\n"
            "0 0 1.5 -0.5\r\n0 1\t-2.0 +0.25\r\n1 0 0.75 0.125\n001 3 -0.25 2.0\r2 2 1_000.5 3\f"
            "2 3 -1e3 .5\v0 2 5. -0E0\n"
            "0.01 -0.02 0.03 0.1 -0.2 1.5 420.0 -1e-7 2e-13\n"
            "0 0 0 0.3 -0.4 2 415.5 0 0\n"
            "1e-13 0 -0 0 0 -1 300 0.5 -0.5 # tiny angle\n"
            "-0.1 0.2 -3.0\n0.5 -0.25 -2.5\n1 2 -4\ninf -inf 6\n")
    head = "2 2 3\n0 0 1 2\n1 1 3 4\n0 1 5 6\n"
    cams = " ".join(["0.1"] * 18) + "\n"
    pts = "1 2 3\n4 5 6\n"
    ok = head + cams + pts
    return {
        "synth": synth_text,
        "mini": mini,
        "header_only": "0 0 0\n",
        "empty": "",
        "comment_only": "# nothing here\n\n",
        "truncated_obs": head[:-6] + "\n",
        "truncated_cams": head + " ".join(["0.1"] * 11) + "\n",
        "truncated_pts": head + cams + "1 2 3\n4\n",
        "bad_camera": ok.replace("1 1 3 4", "2 1 3 4"),
        "bad_point": ok.replace("0 1 5 6", "0 -1 5 6"),
        "negative_count": "2 -2 3\n",
        "float_index": ok.replace("1 1 3 4", "1.0 1 3 4"),
        "bad_number": ok.replace("1 2 3\n4 5 6", "1 2 3\n4 5.5.5 6"),
        "hex_number": ok.replace("0 0 1 2", "0 0 0x1p3 2"),
        "bad_underscore": ok.replace("1 2 3\n4", "1 2_ 3\n4"),
        "nan_payload": ok.replace("1 2 3\n4", "1 nan(1) 3\n4"),
        "trailing": ok + "42.0\n7\n",
        "duplicate": "2 2 3\n0 0 1 2\n1 1 3 4\n1 1 5 6\n" + cams + pts,
        "bad_header": "two 2 3\n",
    }


def bal_fixture():
    """Reference io.read_bal on every case of bal_cases(): arrays or the error"""
    import tempfile
    from sparsesfm.io import read_bal
    cases = bal_cases()
    arrays, expect = {}, {}
    with tempfile.TemporaryDirectory() as d:
        for name, text in cases.items():
            path = os.path.join(d, name + ".bal")
            with open(path, "w", newline="") as fh:
                fh.write(text)
            try:
                sc = read_bal(path)
            except Exception as e:   # noqa: BLE001 - the error is the golden output
                expect[name] = {"error": type(e).__name__, "message": str(e), "line": getattr(e, "line", None)}
                continue
            a = scene_to_arrays(sc)
            expect[name] = {"error": None, "counts": [len(a.quats), len(a.points), len(a.cam_idx)]}
            for k in ("quats", "centers", "focals", "dists", "points", "cam_idx", "pt_idx", "pixels"):
                arrays[f"{name}__{k}"] = getattr(a, k)
    with open(os.path.join(HERE, "bal_cases.json"), "w") as fh:
        json.dump({"texts": cases, "expect": expect}, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "bal.npz"), **arrays)
    print("bal cases", {k: v["error"] for k, v in expect.items()})


def main():
    if "bal" in sys.argv[1:]:
        bal_fixture()
        return
    if "metrics" in sys.argv[1:]:
        metrics_fixture()
        return
    if "shared" in sys.argv[1:]:
        shared_focal_fixture()
        return
    if "block" in sys.argv[1:]:
        block_algebra_fixture()
        return
    shared_focal_fixture()
    metrics_fixture()
    bal_fixture()
    # --- BA fixtures
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=8, num_points=120, visibility_fraction=0.5,
                                              pixel_noise_sigma=1.0, seed=3))
    start = rsm.perturb(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    ba_fixture("ba_small.npz", start, ref.RobustLoss("huber", 1.0))
    ba_fixture("ba_nofocal.npz", start, ref.RobustLoss("trivial"), optimize_focal=False)
    ba_fixture("ba_bal.npz", bal_scene(), ref.RobustLoss("huber", 2.0))
    # --- GP fixtures
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=10, num_points=200, visibility_fraction=0.4,
                                              pixel_noise_sigma=0.5, seed=2))
    gp_fixture("gp_small.npz", obs, ref.RobustLoss("huber", 0.1), depth_mode=False)
    gp_fixture("gp_depth.npz", obs, ref.RobustLoss("trivial"), depth_mode=True, iters=30)
    # --- C1 and generator digests
    summary = {}
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=50, num_points=5000, visibility_fraction=4 / 50,
                                              pixel_noise_sigma=1.0, seed=0))
    start = rsm.perturb(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    prob = ref.BAProblem(start, ref.RobustLoss("huber", 1.0))
    th, rep = ref.lm_solve(prob, prob.encode(), ref.LMConfig())
    res = prob.decode(th)
    summary["c1"] = dict(termination=rep.termination, iterations=len(rep.iterations),
                         final_cost=rep.iterations[-1].cost_after,
                         cg_iters=[i.cg_iters for i in rep.iterations],
                         accepted=[bool(i.step_accepted) for i in rep.iterations],
                         rmse=rsm.reproj_rmse(res), cost0=prob.cost(prob.encode()),
                         start_digest=digest(arrays_of(start)))
    np.save(os.path.join(HERE, "c1_theta_final.npy"), th)
    digests = {}
    for name, cfg, pert in [
        ("c1_observed", dict(num_cameras=50, num_points=5000, visibility_fraction=4 / 50,
                             pixel_noise_sigma=1.0, seed=0), None),
        ("sphere_outliers", dict(num_cameras=30, num_points=3000, rig="sphere", visibility_fraction=0.2,
                                 pixel_noise_sigma=0.7, outlier_fraction=0.05, seed=4), None),
        ("big_pop", dict(num_cameras=12000, num_points=200, visibility_fraction=10 / 12000,
                         pixel_noise_sigma=1.0, seed=9), None),
        ("c5_shape_small", dict(num_cameras=5000, num_points=20000, visibility_fraction=10 / 5000,
                                pixel_noise_sigma=1.0, seed=0),
         dict(rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)),
    ]:
        t, o = rsm.generate(rsm.SynthConfig(**cfg))
        digests[name + ":truth"] = digest(arrays_of(t))
        digests[name + ":observed"] = digest(arrays_of(o))
        if pert:
            digests[name + ":perturbed"] = digest(arrays_of(rsm.perturb(o, **pert)))
        digests[name + ":config"] = cfg
        digests[name + ":perturb"] = pert
    summary["digests"] = digests
    # --- GP C2 at 40 iterations (SURVEY.md 8(c) survey-recorded golden)
    truth, obs = rsm.generate(rsm.SynthConfig(num_cameras=200, num_points=50000, visibility_fraction=6 / 200,
                                              pixel_noise_sigma=0.5, seed=0))
    gp = ref.fix_gauge(ref.make_rays(obs, depth_mode=False, loss=ref.RobustLoss("huber", 0.1), seed=0))
    th, rep = ref.lm_solve(gp, gp.initial_theta(), ref.LMConfig(max_iterations=40))
    summary["c2"] = dict(termination=rep.termination, iterations=len(rep.iterations),
                         final_cost=rep.iterations[-1].cost_after,
                         cg_iters=[i.cg_iters for i in rep.iterations],
                         accepted=[bool(i.step_accepted) for i in rep.iterations])
    np.save(os.path.join(HERE, "c2_theta_final.npy"), th[:3 * 200 + 3 * 50000])
    with open(os.path.join(HERE, "summary.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps({k: (v if k != "digests" else "...") for k, v in summary.items()}, indent=1)[:2000])


if __name__ == "__main__":
    main()
