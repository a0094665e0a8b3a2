#!/usr/bin/env bash
timeout 600 python -m pytest tests/test_gpu_ba.py tests/test_gpu_fused.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 4 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
python -c "
import json; b=json.load(open('gpurun_out/q_bench.json'))
print('c5 ms/step', round(b['ms_per_step'],2), 'pcg share', b['roofline']['kernel_share_of_step'], 'cg', b['cg_iters_per_step'])"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:linearize -c 2 --csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print $5, $(NF-2), $NF}'
