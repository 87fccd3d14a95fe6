# compute-sanitizer memcheck / racecheck / synccheck over the edge-case workload
# (tests/debug_workload.py: every strategy x epilogue, unaligned views, ragged ends,
# dense reports through a small staging pool) -- SURVEY.md §5 race detection.
# usage (GPU box): OUT=gpurun_out/san bash tools/sanitize.sh
OUT=${OUT:-gpurun_out/san}
mkdir -p $OUT
export SMGPU_WORKLOAD_SMALL=1
for tool in memcheck racecheck synccheck; do
  extra=""
  if [ $tool = racecheck ]; then extra="--racecheck-report hazard"; fi
  SMGPU_STAGE_BYTES=24896 timeout ${SAN_TIMEOUT:-1500} compute-sanitizer --tool $tool $extra \
      --target-processes all --print-limit 50 --error-exitcode 9 \
      python tests/debug_workload.py > $OUT/$tool.log 2>&1
  echo "$tool exit $?" >> $OUT/$tool.log
  tail -3 $OUT/$tool.log
done
