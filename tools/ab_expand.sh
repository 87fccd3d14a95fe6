#!/bin/bash
# A/B of the report expand (SMGPU_EXPAND_PARTS / _CTAS): dense report + c2 report
for rep in 1 2 3; do
  for v in "SMGPU_EXPAND_CTAS=2" "SMGPU_EXPAND_CTAS=1" "SMGPU_EXPAND_CTAS=1 SMGPU_EXPAND_PARTS=2"; do
    echo -n "$v "; env $v timeout 300 python tools/dense_parts.py 17 | sed -n 1p
    echo -n "$v "; env $v timeout 300 python tools/report_breakdown.py
  done
done
