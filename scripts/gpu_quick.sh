#!/usr/bin/env bash
SSFM_FUSED=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:ba_k_pcg -c 1 --csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time|lts__" 
