# c1 bench A/B (host-bound small config): current library vs $BASE, twice each
OUT=gpurun_out/${TAG:-abc1}
mkdir -p $OUT
for rep in 1 2; do
  timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-e2e --no-report --no-cpu > $OUT/cur_$rep.json 2>/dev/null
  SMGPU_LIB=$BASE timeout 300 python bench.py --config c1 --steps 20 --warmup 5 --no-e2e --no-report --no-cpu > $OUT/base_$rep.json 2>/dev/null
done
