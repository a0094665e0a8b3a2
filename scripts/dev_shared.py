"""Diagnostic: shared-focal damped solves, device vs oracle, several lambdas."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle")]
import numpy as np
import paper_2510_13310_b200 as b2
import sparsesfm_port as orc
from tests.conftest import golden, ba_prob_from_golden
from tests.test_gpu_ba import problem_from_golden, solve_normal_native, rel
import torch
for name in ["ba_shared.npz", "ba_small.npz"]:
    z = golden(name)
    prob = ba_prob_from_golden(z)
    th = z["theta0"]
    r, J = orc.ba_linearize(prob, th)
    Jd = orc.ba_dense_jacobian(prob, J)
    for mode in ["1", "0"]:
        os.environ["SSFM_FUSED"] = mode
        p = problem_from_golden(z)
        p.gradient(th)
        for lam in [1e-3, 1e-4, 1e-5, 1e-6]:
            d, it = solve_normal_native(torch, p, lam, b2.LMConfig())
            do, ito = orc.schur_pcg_solve(Jd.T @ Jd, -(Jd.T @ r), orc.ba_param_blocks(prob), lam)
            print(name, mode, lam, "dev", it, "orc", ito, "rel", rel(d, do))
