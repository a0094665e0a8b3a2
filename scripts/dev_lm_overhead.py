"""Where the time of one lm_solve call goes (host clock, CUDA events, the
records' device time) for a bench config, LM loop on the device or on the host.
Usage: python scripts/dev_lm_overhead.py c4gp|c5|c1 [iters]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2510_13310_b200 as b2  # noqa: E402
from bench import CONFIGS, GP_CONFIGS, make_arrays  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c4gp"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cams, pts, k, sigma, delta, _ = CONFIGS[cfgname]
arr = make_arrays(cams, pts, k, sigma)
loss = b2.RobustLoss("huber", delta)
if cfgname in GP_CONFIGS:
    p = b2.fix_gauge(b2.make_rays_device(arr, depth_mode=False, loss=loss, seed=0))
    th0 = torch.as_tensor(p.initial_theta()).cuda()
else:
    p = b2.BAProblem(arr, loss)
    th0 = torch.as_tensor(p.encode()).cuda()
for mode in ("1", "0", "1"):
    os.environ["SSFM_LM_GRAPH"] = mode
    b2.lm_solve(p, th0, b2.LMConfig(max_iterations=2))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    th, rep = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=iters))
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev = sum(i.device_ms for i in rep.iterations)
    print(f"{cfgname} SSFM_LM_GRAPH={mode}: {len(rep.iterations)} its, events {e0.elapsed_time(e1):.1f} ms, "
          f"host call {1e3 * (t1 - t0):.1f} ms (+sync {1e3 * (t2 - t1):.1f}), records {dev:.1f} ms, "
          f"per-it {[round(i.device_ms, 2) for i in rep.iterations]}", flush=True)
