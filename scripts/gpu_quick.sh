#!/usr/bin/env bash
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29533 bench.py --gpus 2 --config c3 --steps 4 --warmup 3 --same-device --no-cpu-baseline > gpurun_out/bench_dist2.json 2> gpurun_out/bench_dist2.err
tail -3 gpurun_out/bench_dist2.err; cat gpurun_out/bench_dist2.json | cut -c1-600
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
