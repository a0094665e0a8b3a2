"""Developer check on a GPU box: B200 solver vs the reference (oracle/_ref)."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))
os.environ.setdefault("SPARSESFM_BACKEND", "cython")
import sparsesfm as ref
from sparsesfm import synth_metrics as rsm
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import synth

def rel(a, b):
    a = np.asarray(a); b = np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

# ---- C1 BA
cfg = dict(num_cameras=50, num_points=5000, visibility_fraction=4/50, pixel_noise_sigma=1.0, seed=0)
t0 = time.time()
truth_r, obs_r = rsm.generate(rsm.SynthConfig(**cfg))
start_r = rsm.perturb(obs_r, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
print("ref gen", time.time() - t0)
t0 = time.time()
truth_a, obs_a = synth.generate_arrays(synth.SynthConfig(**cfg))
start_a = synth.perturb_arrays(obs_a, rot_deg=1.0, center_frac=0.01, focal_frac=0.02, point_frac=0.005, seed=1)
print("b200 gen", time.time() - t0)
ra = ref.scene.scene_to_arrays(start_r)
for f in ("quats", "centers", "focals", "points", "cam_idx", "pt_idx", "pixels"):
    print("gen", f, np.array_equal(getattr(ra, f), getattr(start_a, f)))
loss_r = ref.RobustLoss("huber", 1.0)
pr = ref.BAProblem(start_r, loss_r)
pb = b2.BAProblem(start_a, b2.RobustLoss("huber", 1.0))
th = pr.encode()
print("encode equal", np.array_equal(th, pb.encode()))
cr, cb = pr.cost(th), pb.cost(th)
print("cost", cr, cb, abs(cr - cb) / cr)
r1, j1 = pr.linearize(th); r1 = r1.copy(); j1d = j1.data.copy()
r2, j2 = pb.linearize(th)
print("resid rel", rel(r2, r1), "J rel", rel(j2.data, j1d))
from sparsesfm.sparse_block import jtr as rjtr
g1 = rjtr(j1, r1); g2 = pb.gradient(th)
print("grad rel", rel(g2, g1))
# one damped solve
from sparsesfm.sparse_block import jtj as rjtj, apply_damping as rdamp
sys_r = rjtj(j1); sys_r.gradient[:] = -g1
d_r = ref.solve_normal(rdamp(sys_r, 1e-3), pr.layout, ref.LMConfig())
import ctypes as ct, torch
from paper_2510_13310_b200 import _native
cfgc = _native.lm_config_c(b2.LMConfig())
delta = torch.empty(len(th), dtype=torch.float64, device="cuda")
it = ct.c_int32(0)
h = pb._native_handle()
_native.check(_native.load().ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-3, ct.byref(cfgc), ct.c_void_p(delta.data_ptr()), ct.byref(it), ct.c_void_p(torch.cuda.current_stream().cuda_stream)))
print("solve_normal rel", rel(delta.cpu().numpy(), d_r), "cg", it.value)
# full solve
t0 = time.time(); thr, rep_r = ref.lm_solve(pr, th, ref.LMConfig()); tr = time.time() - t0
t0 = time.time(); thb, rep_b = b2.lm_solve(pb, th, b2.LMConfig()); tb = time.time() - t0
print("ref", rep_r.termination, len(rep_r.iterations), rep_r.iterations[-1].cost_after, tr)
print("b2 ", rep_b.termination, len(rep_b.iterations), rep_b.iterations[-1].cost_after, tb)
print("cg ref", [i.cg_iters for i in rep_r.iterations])
print("cg b2 ", [i.cg_iters for i in rep_b.iterations])
print("theta rel", rel(thb, thr))
print("dev ms", [round(i.device_ms, 2) for i in rep_b.iterations])

# ---- GP small
cfg2 = dict(num_cameras=20, num_points=2000, visibility_fraction=6/20, pixel_noise_sigma=0.5, seed=0)
truth_r, obs_r = rsm.generate(rsm.SynthConfig(**cfg2))
gr = ref.fix_gauge(ref.make_rays(obs_r, depth_mode=False, loss=ref.RobustLoss("huber", 0.1), seed=0))
truth_a, obs_a = synth.generate_arrays(synth.SynthConfig(**cfg2))
gb = b2.fix_gauge(b2.make_rays(obs_a, depth_mode=False, loss=b2.RobustLoss("huber", 0.1), seed=0))
print("rays equal", np.array_equal(gr.rays, gb.rays))
th0 = gr.initial_theta()
print("gp cost", gr.cost(th0), gb.cost(th0))
r1, j1 = gr.linearize(th0); r1 = r1.copy(); j1d = j1.data.copy()
r2, j2 = gb.linearize(th0)
print("gp resid rel", rel(r2, r1), "J rel", rel(j2.data, j1d))
print("gp grad rel", rel(gb.gradient(th0), rjtr(j1, r1)))
t0 = time.time(); thr, rep_r = ref.lm_solve(gr, th0, ref.LMConfig(max_iterations=40)); tr = time.time() - t0
t0 = time.time(); thb, rep_b = b2.lm_solve(gb, th0, b2.LMConfig(max_iterations=40)); tb = time.time() - t0
print("gp ref", rep_r.termination, len(rep_r.iterations), rep_r.iterations[-1].cost_after, tr)
print("gp b2 ", rep_b.termination, len(rep_b.iterations), rep_b.iterations[-1].cost_after, tb)
print("gp cg ref", [i.cg_iters for i in rep_r.iterations])
print("gp cg b2 ", [i.cg_iters for i in rep_b.iterations])
print("gp acc ref", [int(i.step_accepted) for i in rep_r.iterations])
print("gp acc b2 ", [int(i.step_accepted) for i in rep_b.iterations])
print("gp theta rel", rel(thb, thr))
