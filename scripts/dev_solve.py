"""Compare one damped solve (solve_normal) B200 vs reference at several shapes."""
import os, sys, ctypes as ct
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
os.environ.setdefault("SPARSESFM_BACKEND", "cython")
import torch
import sparsesfm as ref
from sparsesfm.sparse_block import jtj as rjtj, jtr as rjtr, apply_damping as rdamp
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import synth, _native
for cams, pts, k in [(50, 5000, 4), (200, 2000, 4), (200, 2000, 10), (40, 400, 10), (12, 60, 10), (8, 40, 3)]:
    cfg = synth.SynthConfig(num_cameras=cams, num_points=pts, visibility_fraction=k / cams, pixel_noise_sigma=1.0, seed=0)
    _, obs = synth.generate_arrays(cfg)
    st = synth.perturb_arrays(obs, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
    pb = b2.BAProblem(st, b2.RobustLoss("huber", 1.0))
    pr = ref.BAProblem(b2.arrays_to_scene(st), ref.RobustLoss("huber", 1.0))
    th = pb.encode()
    r1, j1 = pr.linearize(th); r1 = r1.copy()
    g1 = rjtr(j1, r1)
    g2 = pb.gradient(th)
    lam = 1e-3
    s = rjtj(j1); s.gradient[:] = -g1
    d_r = ref.solve_normal(rdamp(s, lam), pr.layout, ref.LMConfig(cg_tol=1e-12, cg_max_iters=3000))
    cfgc = _native.lm_config_c(b2.LMConfig(cg_tol=1e-12, cg_max_iters=3000))
    delta = torch.empty(len(th), dtype=torch.float64, device="cuda")
    it = ct.c_int32(0)
    h = pb._native_handle()
    rc = _native.load().ssfm_solve_normal(ct.c_void_p(h.ptr), lam, ct.byref(cfgc), ct.c_void_p(delta.data_ptr()), ct.byref(it), ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    d = delta.cpu().numpy()
    print(cams, pts, k, "rc", rc, "cg", it.value, "grad rel", float(np.abs(g2 - g1).max() / np.abs(g1).max()),
          "delta rel", float(np.abs(d - d_r).max() / np.abs(d_r).max()), flush=True)
