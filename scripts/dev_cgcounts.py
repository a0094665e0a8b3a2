"""Diagnostic: per-LM-iteration CG counts of the fused and two-pass operators
against the reference records (ba_small golden) and the C1 summary."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2510_13310_b200 as b2  # noqa: E402
from paper_2510_13310_b200 import synth  # noqa: E402
from tests.conftest import golden, summary  # noqa: E402
from tests.test_gpu_ba import problem_from_golden  # noqa: E402


def run(mode, make, th0, cfg):
    os.environ["SSFM_FUSED"] = mode
    p = make()
    p._native_handle()
    th, rep = b2.lm_solve(p, th0, cfg)
    return [i.cg_iters for i in rep.iterations], rep.iterations[-1].cost_after


z = golden("ba_small.npz")
print("ref     ", [int(x) for x in z["records"][:, 5]], z["records"][-1, 2])
for mode in ("0", "1", "2", "4", "8"):
    print("mode", mode, *run(mode, lambda: problem_from_golden(z), z["theta0"], b2.LMConfig(max_iterations=30)))
s = summary()["c1"]
_, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=50, num_points=5000, visibility_fraction=4 / 50,
                                                 pixel_noise_sigma=1.0, seed=0))
st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
print("c1 ref  ", s["cg_iters"], s["final_cost"])
for mode in ("0", "1", "2"):
    mk = lambda: b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
    print("c1 mode", mode, *run(mode, mk, mk().encode(), b2.LMConfig()))
