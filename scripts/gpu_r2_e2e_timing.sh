SSFM_TIMING=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/e2e_t.json 2> gpurun_out/e2e_t.err; grep -E "ssfm|e2e" gpurun_out/e2e_t.err | head -60
