#!/usr/bin/env bash
# compute-sanitizer evidence: racecheck + synccheck on the fused ticket protocol (shared-memory acquire/release),
# the cluster vector-phase kernel (DSMEM) and the graph PCG; memcheck on a BA solve and the LM graph
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
T="tests/test_gpu_fused.py::test_fused_default_on_reference_golden tests/test_gpu_fused.py::test_gp_fused_default_on_reference_golden tests/test_gpu_fused.py::test_graph_pcg_matches_persistent_kernel"
timeout 1500 $CS --tool racecheck --racecheck-report hazard --print-limit 5000 python -m pytest $T -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitize_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/sanitize_racecheck.log
timeout 1500 $CS --tool synccheck --print-limit 20 python -m pytest $T -m gpu -q -x -p no:cacheprovider > gpurun_out/sanitize_synccheck.log 2>&1; echo "synccheck rc=$?" >> gpurun_out/sanitize_synccheck.log
timeout 1500 $CS --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_lm_graph.py -m gpu -q -x -k "ba_small or gp_small" -p no:cacheprovider > gpurun_out/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/sanitize_memcheck.log
tail -4 gpurun_out/sanitize_*.log
