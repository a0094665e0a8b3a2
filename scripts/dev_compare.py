"""B200 vs reference (oracle/_ref) on a configurable synthetic BA problem."""
import argparse, os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
os.environ.setdefault("SPARSESFM_BACKEND", "cython")
ap = argparse.ArgumentParser()
ap.add_argument("--cams", type=int, default=1000); ap.add_argument("--pts", type=int, default=40000)
ap.add_argument("--k", type=int, default=10); ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--noref", action="store_true")
a = ap.parse_args()
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import synth
cfg = synth.SynthConfig(num_cameras=a.cams, num_points=a.pts, visibility_fraction=a.k / a.cams, pixel_noise_sigma=1.0, seed=0)
_, obs = synth.generate_arrays(cfg)
st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
pb = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
th = pb.encode()
t0 = time.time(); thb, rb = b2.lm_solve(pb, th, b2.LMConfig(max_iterations=a.iters)); tb = time.time() - t0
print("b2  ", rb.termination, [(i.cg_iters, int(i.step_accepted), i.status, f"{i.lam:.0e}") for i in rb.iterations], f"{tb:.2f}s")
print("b2 costs", [f"{i.cost_after:.10e}" for i in rb.iterations])
if not a.noref:
    import sparsesfm as ref
    pr = ref.BAProblem(b2.arrays_to_scene(st), ref.RobustLoss("huber", 1.0))
    t0 = time.time(); thr, rr = ref.lm_solve(pr, th, ref.LMConfig(max_iterations=a.iters)); tr = time.time() - t0
    print("ref ", rr.termination, [(i.cg_iters, int(i.step_accepted), f"{i.lam:.0e}") for i in rr.iterations], f"{tr:.2f}s")
    print("ref costs", [f"{i.cost_after:.10e}" for i in rr.iterations])
    print("theta rel", float(np.abs(thb - thr).max() / np.abs(thr).max()))
