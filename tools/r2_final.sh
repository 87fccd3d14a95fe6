# round-2 full GPU pass on the final build: tests, smoke, default bench, per-config bench lines,
# launch list of the default step, ncu --set full of the dominant c2 launch (traffic)
OUT=gpurun_out/${TAG:-r2final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
if [ -z "$NOTEST" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
fi
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
for c in ${CONFIGS:-c1 c3 c4 c4p c5}; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "exit $?" >> $OUT/bench_$c.err
done
if [ -z "$NONCU" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-report --no-cpu > $OUT/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/count_c2m16x64 python tools/kcount.py c2 16 64 0 > $OUT/ncu_full.log 2>&1
fi
echo done
