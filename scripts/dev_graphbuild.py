"""Diagnostic: cost of the first damped solve (graph build) vs later ones at C5."""
import ctypes as ct, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import _native
from bench import make_arrays
arr = make_arrays(5000, 2000000, 10, 1.0)
for g in ("1", "0"):
    os.environ["SSFM_PCG_GRAPH"] = g
    p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
    p.gradient(p.encode())
    lib = _native.load(); h = p._native_handle()
    st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
    d = torch.empty(p.layout.total_params, dtype=torch.float64, device="cuda")
    it = ct.c_int32()
    for k in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        lib.ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-4, ct.byref(_native.lm_config_c(b2.LMConfig())), ct.c_void_p(d.data_ptr()), ct.byref(it), st)
        torch.cuda.synchronize()
        print(f"graph={g} solve {k}: {1e3*(time.perf_counter()-t):.1f} ms, cg {it.value}")
    del p
