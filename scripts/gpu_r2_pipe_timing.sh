#!/usr/bin/env bash
# where does run_global_sfm spend its non-LM time (C4 pipeline)? python-level profile + handle phases
set -x
SSFM_TIMING=1 timeout 600 python -c "
import time, cProfile, pstats, sys
sys.path.insert(0, '.')
import paper_2510_13310_b200 as b2
from paper_2510_13310_b200 import synth
_, obs = synth.generate_arrays(synth.SynthConfig(num_cameras=1000, num_points=500000, visibility_fraction=8/1000, pixel_noise_sigma=1.0, seed=0))
b2.run_global_sfm(obs)
t=time.perf_counter(); b2.run_global_sfm(obs); print('second call', time.perf_counter()-t, flush=True)
pr=cProfile.Profile(); pr.enable(); t=time.perf_counter(); b2.run_global_sfm(obs); print('third call', time.perf_counter()-t, flush=True); pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
" > gpurun_out/pipe_timing.log 2>&1
grep -E "call|ssfm" gpurun_out/pipe_timing.log | head -30
grep -A40 "cumulative" gpurun_out/pipe_timing.log | head -45
