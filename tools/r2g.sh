# re-entry check on a rebuilt container: GPU tests, smoke, default bench, c1 (L2 flush between steps), reference arm
OUT=gpurun_out/${TAG:-r2g}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
for c in ${CONFIGS:-c1}; do
  timeout 900 python bench.py --config $c --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "exit $?" >> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo done
