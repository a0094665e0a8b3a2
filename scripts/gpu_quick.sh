#!/usr/bin/env bash
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/q_c5.json 2> gpurun_out/q_c5.err
python -c "
import json; b=json.load(open('gpurun_out/q_c5.json'))
print('value', round(b['value']/1e6,1), 'M obs/s; ms/step', round(b['ms_per_step'],2), 'e2e', round(b['e2e']['value']/1e6,1), 'M obs/s', b['e2e'])"
