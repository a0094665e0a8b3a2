"""Diagnostic: where the end-to-end (host arrays -> solve -> host) time goes at C5."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2510_13310_b200 as b2
from bench import make_arrays
arr = make_arrays(5000, 2000000, 10, 1.0)
torch.cuda.init(); torch.zeros(1, device="cuda")
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
    t1 = time.perf_counter()
    th0 = p.encode()
    t2 = time.perf_counter()
    p._native_handle(); torch.cuda.synchronize()
    t3 = time.perf_counter()
    th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=13))
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    dev = sum(i.device_ms for i in r.iterations)
    print(f"ctor {1e3*(t1-t0):.0f} ms, encode {1e3*(t2-t1):.0f} ms, create {1e3*(t3-t2):.0f} ms, "
          f"lm_solve {1e3*(t4-t3):.0f} ms ({len(r.iterations)} its, device {dev:.0f} ms)")
    del p
