"""A/B of kernel-variant libraries (scripts/build_variants.sh) at one config:
per variant, the standalone operator passes (ssfm_bench_operator) and a short
LM solve (device ms per iteration). Usage: python scripts/dev_ab.py C P k lib1.so lib2.so ..."""
import ctypes as ct, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import _native
from bench import make_arrays
cams, pts, k = (int(x) for x in sys.argv[1:4])
libs = sys.argv[4:]
# a lib path may carry env settings: "path.so:SSFM_L2_PERSIST=0,SSFM_X=1"
arr = make_arrays(cams, pts, k, 1.0)
N, P, C = arr.num_observations, arr.num_points, arr.num_cameras
st = ct.c_void_p(torch.cuda.current_stream().cuda_stream)
for rep in range(2):
    for spec in libs:
        lib_path, _, envs = spec.partition(":")
        for kv in filter(None, envs.split(",")):
            kk, vv = kv.split("=")
            os.environ[kk] = vv
        _native._lib = None
        _native.LIB_PATH = lib_path
        lib = _native.load()
        p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
        th = p.encode()
        p.gradient(th)
        h = p._native_handle()
        d = torch.empty(p.layout.total_params, dtype=torch.float64, device="cuda")
        it = ct.c_int32()
        _native.check(lib.ssfm_solve_normal(ct.c_void_p(h.ptr), 1e-4, ct.byref(_native.lm_config_c(b2.LMConfig())),
                                            ct.c_void_p(d.data_ptr()), ct.byref(it), st))
        out = []
        for which in (0, 1, 2):
            ms = ct.c_double()
            _native.check(lib.ssfm_bench_operator(ct.c_void_p(h.ptr), which, 20, ct.byref(ms), st))
            out.append(ms.value)
        lib.ssfm_profile_enable(ct.c_void_p(h.ptr), 1)
        _, r = b2.lm_solve(p, th, b2.LMConfig(max_iterations=4))
        pms, pl, cgit = ct.c_double(0), ct.c_int64(0), ct.c_double(0)
        lib.ssfm_profile_get(ct.c_void_p(h.ptr), 0, ct.byref(pms), ct.byref(pl), ct.byref(cgit))
        lib.ssfm_profile_enable(ct.c_void_p(h.ptr), 0)
        dm = [round(i.device_ms, 2) for i in r.iterations]
        cg = [i.cg_iters for i in r.iterations]
        per_cg = sum(i.device_ms for i in r.iterations[1:]) / max(1, sum(cg[1:]))
        non_pcg = (sum(i.device_ms for i in r.iterations) - pms.value) / max(1, len(r.iterations))
        print(f"{os.path.basename(lib_path) + ' ' + envs:40s} point {out[0]:.4f} camera {out[1]:.4f} pair {out[2]:.4f} ms | "
              f"lm ms {dm} cg {cg} ({per_cg:.4f} ms/cg incl. step overhead; non-PCG {non_pcg:.2f} ms/it, "
              f"PCG {pms.value / max(1, cgit.value):.4f} ms/cg)", flush=True)
        p.release(trim=True)
        for kv in filter(None, envs.split(",")):
            os.environ.pop(kv.split("=")[0], None)
