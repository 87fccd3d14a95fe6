#!/bin/bash
# A/B of two environment settings on single-pattern PACKED work: dense report, single counts
for rep in 1 2 3; do
  for v in A B; do
    ev=AB_ENV_$v
    echo -n "$v "; env ${!ev} timeout 300 python tools/dense_report.py | tail -1
    for w in "c4 32 1 1073741824" "c1 16 1" "c4 8 1 1073741824"; do
      echo -n "$v "; env ${!ev} timeout 120 python tools/kcount.py $w | sed 's/plans.*//'
    done
  done
done
