# last pass of round 2 on the final build: randomised parity stress (release + bounds-asserting
# debug build) and one bench line per config, all from the same container build
OUT=gpurun_out/${TAG:-r2h}
mkdir -p $OUT
SEED=101 timeout 400 python tools/stress_parity.py 240 > $OUT/stress_release.log 2>&1; echo "exit $?" >> $OUT/stress_release.log
SEED=202 SMGPU_LIB=debug timeout 400 python tools/stress_parity.py 180 > $OUT/stress_debug.log 2>&1; echo "exit $?" >> $OUT/stress_debug.log
for c in c1 c3 c4 c4p c5; do
  timeout 1500 python bench.py --config $c --no-cpu > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "exit $?" >> $OUT/bench_$c.err
done
timeout 300 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err; echo "exit $?" >> $OUT/bench_c2.err
echo done
