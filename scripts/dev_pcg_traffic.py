"""One damped solve (ssfm_solve_normal) of a bench config: prints the CG
iteration count, so that an ncu capture of the PCG graph (--graph-profiling
graph) gives DRAM bytes per CG iteration (profiles/traffic_<config>.json).
Usage: python scripts/dev_pcg_traffic.py [c5|c4ba|c3]"""
import ctypes as ct
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2510_13310_b200 as b2  # noqa: E402
from paper_2510_13310_b200 import _native  # noqa: E402
from bench import CONFIGS, C3_TRIM, make_arrays  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c5"
cams, pts, k, sigma, delta, _ = CONFIGS[cfgname]
arr = make_arrays(cams, pts, k, sigma, trim=C3_TRIM if cfgname == "c3" else None)
p = b2.BAProblem(arr, b2.RobustLoss("huber", delta))
th = p.encode()
p.gradient(th)
lib = _native.load()
h = p._native_handle()
st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
d = torch.empty(p.layout.total_params, dtype=torch.float64, device="cuda")
it = ct.c_int32()
for _ in range(2):
    _native.check(lib.ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-4, ct.byref(_native.lm_config_c(b2.LMConfig())),
                                        ct.c_void_p(d.data_ptr()), ct.byref(it), st))
torch.cuda.synchronize()
print(json.dumps({"config": cfgname, "cg_iters_per_solve": it.value, "solves": 2,
                  "N": arr.num_observations, "P": arr.num_points, "C": arr.num_cameras}))
