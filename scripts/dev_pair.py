"""The two-pass operator's passes back to back (ssfm_bench_operator which=2) at
C5, for ncu with --cache-control none (in-situ L2 state of the camera pass)."""
import ctypes as ct, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
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
ms = ct.c_double()
_native.check(lib.ssfm_bench_operator(ct.c_void_p(h.ptr), 2, 3, ct.byref(ms), st))
print("pair ms", ms.value)
