"""Diagnostic: replicate bench.py's GP timed loop and time each piece."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2510_13310_b200 as b2
from bench import make_arrays, ClockSampler
arr = make_arrays(1000, 500000, 8, 1.0)
loss = b2.RobustLoss("huber", 0.1)
p = b2.fix_gauge(b2.make_rays(arr, depth_mode=False, loss=loss, seed=0))
th0 = torch.as_tensor(p.initial_theta()).cuda()
p._native_handle()
thw, rw = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=3))
print("warmup term", rw.termination, [i.step_accepted for i in rw.iterations])
for sampler_on in (False, True):
    s = ClockSampler(0)
    if sampler_on:
        s.start(); time.sleep(0.3)
    torch.cuda.synchronize(); t = time.perf_counter()
    th, r = b2.lm_solve(p, thw, b2.LMConfig(max_iterations=6, lambda0=1.25e-5))
    torch.cuda.synchronize(); w = time.perf_counter() - t
    if sampler_on: s.stop()
    print(f"sampler={sampler_on} wall {1e3*w:.1f} ms, device {sum(i.device_ms for i in r.iterations):.1f} ms, "
          f"host per it {[round(i.wall_time_ns/1e6,2) for i in r.iterations]}, term {r.termination}")
