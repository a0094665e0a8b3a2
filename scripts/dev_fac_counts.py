"""CG counts per LM iteration on the reference goldens: two-pass operator with
and without the factored camera pass (SSFM_FUSED=0), against the reference."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import paper_2510_13310_b200 as b2
from tests.test_gpu_ba import problem_from_golden
from tests.conftest import golden
for name in ("ba_small.npz", "ba_bal.npz", "ba_nofocal.npz", "ba_shared.npz"):
    z = golden(name)
    if "records" not in z.files:
        continue
    ref = [int(x) for x in z["records"][:, 5]]
    out = {}
    for fused, fac in (("1", "1"), ("0", "0"), ("0", "1")):
        os.environ["SSFM_FUSED"], os.environ["SSFM_FACTORED"] = fused, fac
        p = problem_from_golden(z)
        p._native_handle()
        th, rep = b2.lm_solve(p, z["theta0"], b2.LMConfig(max_iterations=len(ref)))
        out[f"fused{fused}/fac{fac}"] = [i.cg_iters for i in rep.iterations]
    print(name, "ref", ref)
    for k, v in out.items():
        print("   ", k, v, "max|d|", max(abs(a - b) for a, b in zip(v, ref)))
