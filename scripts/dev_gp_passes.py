"""GP (C4 shape by default): standalone point / camera pass times of the
two-pass Schur operator (ssfm_bench_operator) after one damped solve."""
import ctypes as ct
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2510_13310_b200 as b2  # noqa: E402
from paper_2510_13310_b200 import _native  # noqa: E402
from bench import CONFIGS, make_arrays  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4gp"
cams, pts, k, sigma, delta, _ = CONFIGS[cfgname]
arr = make_arrays(cams, pts, k, sigma)
p = b2.fix_gauge(b2.make_rays_device(arr, depth_mode=False, loss=b2.RobustLoss("huber", delta), seed=0))
th = p.initial_theta()
p.gradient(th)
lib = _native.load()
h = p._native_handle()
st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
d = torch.empty(p.layout.total_params, dtype=torch.float64, device="cuda")
it = ct.c_int32()
_native.check(lib.ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-4, ct.byref(_native.lm_config_c(b2.LMConfig())),
                                    ct.c_void_p(d.data_ptr()), ct.byref(it), st))
N, P, C = arr.num_observations, arr.num_points, arr.num_cameras
for which, name, byts in [(0, "point pass", 36 * N + 48 * P + 32 * P), (1, "camera pass", 36 * N + 32 * N)]:
    ms = ct.c_double()
    _native.check(lib.ssfm_bench_operator(ct.c_void_p(h.ptr), which, 20, ct.byref(ms), st))
    print(f"{name}: {ms.value:.4f} ms, {byts / ms.value / 1e6:.0f} GB/s (bytes {byts / 1e9:.3f} GB); cg {it.value}")
