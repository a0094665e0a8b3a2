"""Diagnostic: where does GP LM time go outside the per-iteration device time?"""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2510_13310_b200 as b2
from bench import make_arrays
arr = make_arrays(1000, 500000, 8, 1.0)
p = b2.fix_gauge(b2.make_rays(arr, depth_mode=False, loss=b2.RobustLoss("huber", 0.1), seed=0))
th0 = torch.as_tensor(p.initial_theta()).cuda()
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=6))
    torch.cuda.synchronize(); w = time.perf_counter() - t
    print(f"wall {w*1e3:.1f} ms; iterations {len(r.iterations)}; device {[round(i.device_ms,2) for i in r.iterations]}; "
          f"host wall per it {[round(i.wall_time_ns/1e6,2) for i in r.iterations]}")
