# ncu --set full captures on the last build of round 2: the c2 FILTER launch (kcount: m = 16 x 64 patterns,
# the launch profiles/traffic_c2.json describes) and one search launch taken from the bench command itself
OUT=gpurun_out/${TAG:-r2j}
mkdir -p $OUT
timeout 300 python tools/kcount.py c2 16 64 0 > $OUT/kcount_plain.log 2>&1; echo "exit $?" >> $OUT/kcount_plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/count_c2m16x64 python tools/kcount.py c2 16 64 0 > $OUT/ncu_kcount.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 70 --launch-count 1 -o $OUT/bench_launch70 python bench.py --steps 1 --warmup 3 --no-e2e --no-report --no-cpu > $OUT/ncu_bench.log 2>&1
ls -la $OUT
echo done
