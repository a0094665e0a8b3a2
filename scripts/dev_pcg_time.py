"""Time of a fixed number of graph-PCG iterations at a bench config (cg_max_iters
caps the solve; a CGStall at the cap is expected and ignored): ms per CG iteration.
Usage: python scripts/dev_pcg_time.py [c5] [iters]"""
import ctypes as ct
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import paper_2510_13310_b200 as b2  # noqa: E402
from paper_2510_13310_b200 import _native  # noqa: E402
from bench import CONFIGS, make_arrays  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cams, pts, k, sigma, delta, _ = CONFIGS[cfgname]
p = b2.BAProblem(make_arrays(cams, pts, k, sigma), b2.RobustLoss("huber", delta))
th = p.encode()
p.gradient(th)
lib = _native.load()
h = p._native_handle()
st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
d = torch.empty(p.layout.total_params, dtype=torch.float64, device="cuda")
it = ct.c_int32()
cfg = _native.lm_config_c(b2.LMConfig(cg_tol=1e-30, cg_max_iters=iters))
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rc = lib.ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-4, ct.byref(cfg), ct.c_void_p(d.data_ptr()), ct.byref(it), st)
    e1.record()
    torch.cuda.synchronize()
    print(f"{os.path.basename(_native.LIB_PATH)} rc={rc} iters={it.value} {e0.elapsed_time(e1) / max(1, it.value):.4f} ms per CG iteration", flush=True)
