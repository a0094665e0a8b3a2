"""Diagnostic: per-pass time and algorithmic bandwidth of the two-pass operator at C5."""
import ctypes as ct, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("SSFM_FUSED", "0")
import torch
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import _native
from bench import make_arrays
cams, pts, k = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (5000, 2000000, 10))]
arr = make_arrays(cams, pts, k, 1.0)
p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
th = p.encode()
p.gradient(th)
lib = _native.load()
h = p._native_handle()
st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
d = torch.empty(p.layout.total_params, dtype=torch.float64, device="cuda")
it = ct.c_int32()
lib.ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-4, ct.byref(_native.lm_config_c(b2.LMConfig())), ct.c_void_p(d.data_ptr()), ct.byref(it), st)
N, P, C = arr.num_observations, arr.num_points, arr.num_cameras
fac = os.environ.get("SSFM_FACTORED", "1") != "0"
wf = fac and os.environ.get("SSFM_WFORM", "1") != "0"
for which, name, byts in [(0, "point pass", ((64 + 8) if wf else (128 + 4)) * N + 48 * P + 32 * P + (32 * P if wf else 0)),
                          (1, "camera pass", (56 if fac else 128) * N + 4 * N + 32 * N)]:
    ms = ct.c_double()
    _native.check(lib.ssfm_bench_operator(ct.c_void_p(h.ptr), which, 20, ct.byref(ms), st))
    print(f"{name}: {ms.value:.4f} ms, {byts / ms.value / 1e6:.0f} GB/s (bytes {byts/1e9:.2f} GB)")
