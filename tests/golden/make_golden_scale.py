"""Reference runs at scale (SURVEY.md 8(d) C3, C4 and a 5000-camera C5 sample).

Run in the build container, where the UNMODIFIED reference is importable from
oracle/_ref (built by oracle/build_ref.sh from /root/reference):

    python tests/golden/make_golden_scale.py c3|c4|c5s

Each run writes tests/golden/scale_<name>.npz: the reference's iteration
records, termination, final cost and RMSE, every camera's parameters, a
strided sample of the points, and sha256 digests of the inputs (so the GPU
test can prove it regenerated the same arrays with the array-native replay,
paper_2510_13310_b200/synth.py) and, for C3, of the reference's integer
structures (JtJPattern.off_keys and the _SchurPlan slot list). The GPU tests
(tests/test_gpu_scale.py) rebuild the inputs bit-identically on the box and
compare the device solve against these records. Nothing here runs at test
time, and nothing under /root/reference is read on the GPU box.
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
os.environ["SPARSESFM_BACKEND"] = "cython"
os.environ.setdefault("SPARSESFM_WORKERS", str(os.cpu_count()))

import sparsesfm as ref  # noqa: E402
from sparsesfm import synth_metrics as rsm  # noqa: E402
from sparsesfm.lm import _get_schur_plan  # noqa: E402
from sparsesfm.scene import Observation, Scene, scene_to_arrays  # noqa: E402
from sparsesfm.sparse_block import apply_damping, jtj  # noqa: E402

PERTURB = dict(rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
POINT_SAMPLES = 2000


def sha(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def input_digest(a) -> str:
    """sha256 over the SoA a problem is built from (same fields and dtypes as
    tests/test_gpu_scale.py: quats, centers, focals, points f64; cam/pt int64;
    pixels f64)."""
    return sha(a.quats, a.centers, a.focals, a.points, a.cam_idx.astype(np.int64),
               a.pt_idx.astype(np.int64), a.pixels)


def records(rep):
    return np.array([(i.iteration, i.cost_before, i.cost_after, i.lam, float(i.step_accepted),
                      i.cg_iters) for i in rep.iterations], dtype=np.float64).reshape(-1, 6)


def point_sample(P: int) -> np.ndarray:
    return np.unique(np.linspace(0, P - 1, POINT_SAMPLES).astype(np.int64))


def trim_c3(scene: Scene, keep_full: int = 80000) -> Scene:
    """for points j >= keep_full drop the observation with
    the highest camera id (exactly 680,000 observations at 150k points, k=5).
    Camera-major order is kept."""
    best = {}
    for m, o in enumerate(scene.observations):
        if o.point_id >= keep_full:
            if o.point_id not in best or o.camera_id > scene.observations[best[o.point_id]].camera_id:
                best[o.point_id] = m
    drop = set(best.values())
    obs = [o for m, o in enumerate(scene.observations) if m not in drop]
    return Scene(scene.cameras, scene.points, obs)


def ba_run(name, start, iters, loss_delta=1.0, with_pattern=False):
    a = scene_to_arrays(start)
    t0 = time.time()
    prob = ref.BAProblem(start, ref.RobustLoss("huber", loss_delta))
    th0 = prob.encode()
    out = dict(input_digest=input_digest(a), cost0=prob.cost(th0))
    if with_pattern:
        r, J = prob.linearize(th0)
        sys_ = jtj(J)
        out["off_keys_digest"] = sha(sys_.off_keys.astype(np.int32))
        out["n_off"] = len(sys_.off_keys)
        ws = ref.Workspace()
        damped = apply_damping(sys_, 1e-3)
        plan = _get_schur_plan(damped, ws)
        ra = np.searchsorted(plan.ret_s_off, plan.slot_row, side="right") - 1
        rb = np.searchsorted(plan.ret_s_off, plan.slot_col, side="right") - 1
        slots = np.stack([ra, rb], axis=1).astype(np.int32)
        out["slots_digest"] = sha(slots)
        out["n_slots"] = len(slots)
        del sys_, damped, plan, ws, J
        print(name, "pattern", time.time() - t0, "s", flush=True)
    th, rep = ref.lm_solve(prob, th0, ref.LMConfig(max_iterations=iters))
    res = prob.decode(th)
    C = a.quats.shape[0]
    P = a.points.shape[0]
    sel = point_sample(P)
    out.update(records=records(rep), termination=rep.termination, final_cost=rep.iterations[-1].cost_after,
               rmse=rsm.reproj_rmse(res), rmse0=rsm.reproj_rmse(start),
               cam_theta=th[:7 * C].reshape(C, 7), focals=th[7 * C + 3 * P:], point_idx=sel,
               points=th[7 * C:7 * C + 3 * P].reshape(P, 3)[sel], diameter=rsm.scene_diameter(start),
               wall_s=time.time() - t0, num_obs=len(a.cam_idx),
               wall_ns=np.array([i.wall_time_ns for i in rep.iterations], dtype=np.int64))
    return out, res


def c3():
    _, obs = rsm.generate(rsm.SynthConfig(num_cameras=1700, num_points=150000, visibility_fraction=5 / 1700,
                                          pixel_noise_sigma=1.0, seed=0))
    start = trim_c3(rsm.perturb(obs, **PERTURB))
    assert len(start.observations) == 680000, len(start.observations)
    out, _ = ba_run("c3", start, 10, with_pattern=True)
    return out


def c5s():
    _, obs = rsm.generate(rsm.SynthConfig(num_cameras=5000, num_points=200000, visibility_fraction=10 / 5000,
                                          pixel_noise_sigma=1.0, seed=0))
    start = rsm.perturb(obs, **PERTURB)
    out, _ = ba_run("c5s", start, 10)
    return out


def c4():
    t0 = time.time()
    _, obs = rsm.generate(rsm.SynthConfig(num_cameras=1000, num_points=500000, visibility_fraction=8 / 1000,
                                          pixel_noise_sigma=1.0, seed=0))
    a = scene_to_arrays(obs)
    out = {"input_digest": input_digest(a)}
    gp_scene, rep_gp = ref.run_gp(obs, depth_mode=False, loss=ref.RobustLoss("huber", 0.1),
                                  config=ref.LMConfig(max_iterations=20), seed=0)
    g = scene_to_arrays(gp_scene)
    P = g.points.shape[0]
    sel = point_sample(P)
    out.update(gp_records=records(rep_gp), gp_termination=rep_gp.termination,
               gp_final_cost=rep_gp.iterations[-1].cost_after, gp_centers=g.centers, gp_point_idx=sel,
               gp_points=g.points[sel], gp_wall_s=time.time() - t0)
    print("c4 gp", rep_gp.termination, len(rep_gp.iterations), time.time() - t0, "s", flush=True)
    ba, _ = ba_run("c4ba", gp_scene, 10)
    out.update({"ba_" + k: v for k, v in ba.items()})
    return out


def main():
    which = sys.argv[1]
    t0 = time.time()
    out = {"c3": c3, "c4": c4, "c5s": c5s}[which]()
    out["numpy_version"] = np.__version__
    np.savez_compressed(os.path.join(HERE, f"scale_{which}.npz"), **out)
    summ = {k: (v if np.ndim(v) == 0 else np.shape(v)) for k, v in out.items()}
    print(which, f"{time.time() - t0:.1f} s", summ, flush=True)


if __name__ == "__main__":
    main()
