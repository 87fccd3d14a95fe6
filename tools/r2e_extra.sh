# extra measurements of GPU call r2e: report path (pool, list/bitmap threshold), binary r sweep to 16
OUT=gpurun_out/${TAG:-r2e}
OUT=$OUT/report bash tools/report_probe.sh
for L in 8 16 32 64; do
  SMGPU_LIST_MAX=$L timeout 300 python tools/report_breakdown.py > $OUT/report/report_list$L.log 2>&1
done
SMGPU_LIST_MAX=16 timeout 300 python tools/dense_report.py > $OUT/report/dense_list16.log 2>&1
timeout 300 python tools/dense_report.py > $OUT/report/dense_default.log 2>&1
timeout 900 python tools/ablation_r2.py --mode rsweep --configs c4 --lengths 16,32,128 --rmax 16 > $OUT/ablation_rsweep_c4.jsonl 2> $OUT/ablation_rsweep_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-report --no-cpu > $OUT/ncu_launch.log 2>&1
