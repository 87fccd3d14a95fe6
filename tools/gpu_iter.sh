# one GPU iteration: tests, bench (JSON line to gpurun_out/bench.json); extra commands via $EXTRA
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
echo done
