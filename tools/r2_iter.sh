# one GPU iteration of round 2: GPU tests, smoke, config bench lines (per-m), optional $EXTRA
set -x
OUT=gpurun_out/${TAG:-iter}
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for c in ${CONFIGS:-c2 c3}; do
  timeout 600 python bench.py --config $c --no-e2e --no-report --no-cpu --steps 3 > $OUT/cfg_$c.json 2>$OUT/cfg_$c.err
done
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
echo done
