#!/bin/bash
# A/B of two environment settings on the full count step (bench.py, 20 steps: long enough to meet
# the power limit), interleaved
for rep in 1 2 3; do
  for v in A B; do
    ev=AB_ENV_$v
    env ${!ev} timeout 300 python bench.py --steps 20 --no-e2e --no-report --no-cpu --no-dense > /tmp/ab_$v.json 2>/dev/null
    python -c "
import json; d=json.load(open('/tmp/ab_$v.json'))
print('$v', d['value'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
done
