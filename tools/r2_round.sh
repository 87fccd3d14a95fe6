# round-2 full GPU pass: tests, smoke, default bench, reference arm, launch list ($TAG names the output dir)
set -x
OUT=gpurun_out/${TAG:-r2}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench exit $?" >> $OUT/bench.err
if [ -z "$NOREF" ]; then timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err; fi
if [ -z "$NOLAUNCH" ]; then timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-report --no-cpu > $OUT/ncu_launch.log 2>&1; fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
echo done
