"""Diagnostic: phase times of handle creation + first solve at C5 (SSFM_TIMING=1)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SSFM_TIMING"] = "1"
import numpy as np
import torch
import paper_2510_13310_b200 as b2
from bench import make_arrays
arr = make_arrays(5000, 2000000, 10, 1.0)
torch.zeros(1, device="cuda")
def pinned(x):
    t = torch.empty(x.shape, dtype=getattr(torch, str(x.dtype)), pin_memory=True)
    t.numpy()[...] = x
    return t.numpy()
arr.cam_idx, arr.pt_idx, arr.pixels = pinned(np.asarray(arr.cam_idx)), pinned(np.asarray(arr.pt_idx)), pinned(np.asarray(arr.pixels))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
    th0 = p.encode()
    t1 = time.perf_counter()
    p._native_handle(); torch.cuda.synchronize()
    t2 = time.perf_counter()
    th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=3))
    t3 = time.perf_counter()
    dev = sum(i.device_ms for i in r.iterations)
    print(f"rep {rep}: ctor+encode {1e3*(t1-t0):.0f} ms, create {1e3*(t2-t1):.0f} ms, lm_solve(3) {1e3*(t3-t2):.0f} ms (device {dev:.0f} ms)", flush=True)
    del p
