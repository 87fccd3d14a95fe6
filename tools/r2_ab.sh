# round-2 A/B: PACKED sparse verification (threshold / peel target) on c4 and c1, FILTER vs PAIR for
# m = 3, 4 with the one-pass phase B on c3 and c2.  Output: gpurun_out/$TAG/ab_*.json
OUT=gpurun_out/${TAG:-ab}
mkdir -p $OUT
for sp in 0 64 128 256; do
  for ps in 16 32 64; do
    if [ $sp = 0 ] && [ $ps != 32 ]; then continue; fi
    SMGPU_PACKED_SPARSE=$sp SMGPU_PACKED_PEEL_SURV=$ps timeout 300 python tools/kbench.py --config c4 --lengths 8,32,128,1024 \
      --per-m 20 --batch --reps 2 --tag "sparse=$sp surv=$ps" >> $OUT/ab_packed_c4.json 2>&1
    SMGPU_PACKED_SPARSE=$sp SMGPU_PACKED_PEEL_SURV=$ps timeout 300 python tools/kbench.py --config c1 --lengths 4,8,16,32 \
      --per-m 50 --batch --reps 20 --tag "sparse=$sp surv=$ps" >> $OUT/ab_packed_c1.json 2>&1
  done
done
for cfg in c3 c2; do
  for st in 0 1 4; do
    timeout 300 python tools/kbench.py --config $cfg --lengths 4 --per-m 64 --batch --reps 3 --strategy $st \
      --tag "strategy=$st" >> $OUT/ab_short_$cfg.json 2>&1
  done
done
echo done
