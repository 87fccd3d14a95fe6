# after the host-planning change: GPU tests, c1 host phases, c1 / c2 bench lines
OUT=gpurun_out/${TAG:-c1h2}; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
SMGPU_HOST_TIMING=1 timeout 300 python bench.py --config c1 --no-cpu --no-e2e --no-report --no-dense --steps 20 > $OUT/host.json 2> $OUT/host.err
for i in 1 2; do timeout 300 python bench.py --config c1 --no-cpu --steps 20 > $OUT/bench_c1_$i.json 2> $OUT/bench_c1_$i.err; done
echo done
timeout 600 python bench.py --no-cpu > $OUT/bench_c2.json 2> $OUT/bench_c2.err
