# c1 host-bound breakdown: host phase timing per call, kernel launch list of one step
OUT=gpurun_out/c1h; mkdir -p $OUT
SMGPU_HOST_TIMING=1 timeout 300 python bench.py --config c1 --no-cpu --no-e2e --no-report --no-dense --steps 20 > $OUT/bench.json 2> $OUT/host.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/launches.csv python bench.py --config c1 --steps 1 --warmup 3 --no-e2e --no-report --no-cpu --no-dense > $OUT/ncu.log 2>&1
echo done
