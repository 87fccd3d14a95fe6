OUT=gpurun_out/${TAG:-r2f}
SMGPU_HOST_TIMING=1 timeout 300 python tools/host_overhead.py 64 > $OUT/host_timing_64.log 2>&1
SMGPU_HOST_TIMING=1 timeout 300 python tools/host_overhead.py 200 > $OUT/host_timing_200.log 2>&1
timeout 600 python bench.py --config c1 --no-report --no-cpu --steps 20 > $OUT/cfg_c1_full.json 2> $OUT/cfg_c1_full.err
