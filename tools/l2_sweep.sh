#!/bin/bash
# L2 reuse knobs: alternating scan direction x TMA L2 eviction policy, c2 bench step (count only)
mkdir -p gpurun_out
for alt in 0 1; do for pol in 0 1 2; do
  SMGPU_ALTERNATE=$alt SMGPU_L2_POLICY=$pol timeout 300 python bench.py --no-e2e --no-report --no-cpu --steps 3 \
    > gpurun_out/l2_${alt}_${pol}.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/l2_${alt}_${pol}.json'))
print('alt=$alt pol=$pol', d['value'], d['roofline']['frac'], {k: v['frac_of_peak'] for k, v in d['per_m'].items()})"
done; done
