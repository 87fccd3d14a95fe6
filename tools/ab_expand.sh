#!/bin/bash
# A/B of the report expand launch (SMGPU_EXPAND_*): dense report + c2 report
for rep in 1 2 3; do
  for v in "SMGPU_EXPAND_CS=0" "SMGPU_EXPAND_CS=1" "SMGPU_EXPAND_CTAS=1" "SMGPU_EXPAND_CS=1 SMGPU_EXPAND_CTAS=1"; do
    echo -n "$v "; env $v timeout 300 python tools/dense_report.py | tail -1
    echo -n "$v "; env $v timeout 300 python tools/report_breakdown.py
  done
done
