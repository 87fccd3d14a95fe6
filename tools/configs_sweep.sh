#!/bin/bash
# bench lines for every config stand-in (device-resident, count step; per-m breakdown)
mkdir -p gpurun_out
for c in c1 c2 c3 c4; do
  timeout 600 python bench.py --config $c --no-e2e --no-report --no-cpu --steps 3 > gpurun_out/cfg_$c.json 2>gpurun_out/cfg_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/cfg_$c.json'))
print('$c', d['config']['text_bytes'], d['value'], d['roofline']['frac'], d['plans'])
print({k: (v['GBps'], v['frac_of_peak']) for k, v in d['per_m'].items()})"
done
