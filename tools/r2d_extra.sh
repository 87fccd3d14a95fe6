# extra measurements of GPU call r2d
OUT=gpurun_out/${TAG:-r2d}
OUT=$OUT/report bash tools/report_probe.sh
for tile in 8192 16384 32768; do
  SMGPU_TILE=$tile timeout 300 python tools/kbench.py --config c4 --lengths 8,32,1024 --per-m 20 --batch --reps 2 --tag "tile=$tile" >> $OUT/tile_c4.json 2>&1
done
timeout 300 python tools/host_overhead.py 64 > $OUT/host_overhead.log 2>&1
timeout 300 python tools/host_overhead.py 200 >> $OUT/host_overhead.log 2>&1
