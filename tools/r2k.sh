# closing pass: full GPU suite on the final tree (incl. the host-thread test), then long randomised stress parity
OUT=gpurun_out/${TAG:-r2k}
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q --durations=5 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
for s in 11 12 13; do
  SEED=$s timeout 400 python tools/stress_parity.py 300 > $OUT/stress_release_$s.log 2>&1; echo "exit $?" >> $OUT/stress_release_$s.log
done
SEED=21 SMGPU_LIB=debug timeout 400 python tools/stress_parity.py 300 > $OUT/stress_debug_21.log 2>&1; echo "exit $?" >> $OUT/stress_debug_21.log
echo done
