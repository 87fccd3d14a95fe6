#!/bin/bash
# A/B of two environment settings of the same build ($AB_ENV_A vs $AB_ENV_B), interleaved.
IFS=';' read -ra W <<< "${AB_WORK:-c2 16 64;c2 2 64;c3 4 64;c2 256 64}"
for rep in 1 2 3; do
  for v in A B; do
    ev=AB_ENV_$v
    for w in "${W[@]}"; do
      echo -n "$v "; env ${!ev} timeout 120 python tools/kcount.py $w | sed 's/plans.*//'
    done
  done
done
