"""Diagnostic: mid-size two-pass BA (C too large for the fused operator, N < 1M:
persistent kernel) with and without the factored camera pass."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2510_13310_b200 as b2
from bench import make_arrays
arr = make_arrays(3000, 100000, 8, 1.0)
for fac in ("1", "0", "1", "0"):
    for graph in ("0", "1"):
        os.environ["SSFM_FACTORED"], os.environ["SSFM_PCG_GRAPH"] = fac, graph
        p = b2.BAProblem(arr, b2.RobustLoss("huber", 1.0))
        th0 = p.encode()
        p._native_handle()
        th, r = b2.lm_solve(p, th0, b2.LMConfig(max_iterations=8))
        dev = [i.device_ms for i in r.iterations]
        cg = [i.cg_iters for i in r.iterations]
        print(f"factored={fac} graph={graph}: ms/it {sum(dev[2:])/len(dev[2:]):.2f}  ms/cg {sum(dev[2:])/sum(cg[2:]):.4f}  cg {cg}", flush=True)
        p.release()
