# report-path timing: default scratch pool vs a pool that keeps everything cached, plus the
# launch list of one c2 report call.  OUT = output dir
OUT=${OUT:-gpurun_out/report}
mkdir -p $OUT
timeout 300 python tools/report_breakdown.py > $OUT/report_default.log 2>&1
SMGPU_POOL_KEEP_BYTES=18446744073709551615 timeout 300 python tools/report_breakdown.py > $OUT/report_keepall.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $OUT/report_launches.csv \
  python tools/report_breakdown.py > $OUT/report_ncu.log 2>&1
