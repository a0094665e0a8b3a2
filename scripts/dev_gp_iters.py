"""Diagnostic: per-LM-iteration wall vs device time of the C4 GP solve."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2510_13310_b200 as b2
from bench import make_arrays
arr = make_arrays(1000, 500000, 8, 1.0)
p = b2.fix_gauge(b2.make_rays(arr, depth_mode=False, loss=b2.RobustLoss("huber", 0.1), seed=0))
th0 = torch.as_tensor(p.initial_theta(), device="cuda")
b2.lm_solve(p, th0, b2.LMConfig(max_iterations=3))
for rep in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=8))
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"total wall {1e3*(t1-t0):.1f} ms, events {e0.elapsed_time(e1):.1f} ms, sum device {sum(i.device_ms for i in r.iterations):.1f} ms")
    print("  wall ms", [round(i.wall_time_ns / 1e6, 2) for i in r.iterations])
    print("  dev  ms", [round(i.device_ms, 2) for i in r.iterations], [i.cg_iters for i in r.iterations])
import subprocess
proc = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                         "-lms", "100"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
time.sleep(0.5)
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=8))
    e1.record(); torch.cuda.synchronize()
    print(f"with nvidia-smi -lms 100: events {e0.elapsed_time(e1):.1f} ms, sum device {sum(i.device_ms for i in r.iterations):.1f} ms")
proc.terminate()
import ctypes as ct
from paper_2510_13310_b200 import _native
lib = _native.load()
h = p._native_handle()
lib.ssfm_profile_enable(ct.c_void_p(h.ptr), 1)
for rep in range(3):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=8))
    e1.record(); torch.cuda.synchronize()
    print(f"with profile on: events {e0.elapsed_time(e1):.1f} ms, sum device {sum(i.device_ms for i in r.iterations):.1f} ms")
