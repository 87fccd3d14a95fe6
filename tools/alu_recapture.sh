# ALU-pipe work per step of the compare-bound configs (profiles/alu_<cfg>.json) + a source-level capture of PACKED-PRE c4
OUT=gpurun_out/${TAG:-alu}
mkdir -p $OUT
for c in c1 c4 c4p; do
  timeout 900 ncu --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:search_kernel --clock-control none --csv --log-file $OUT/alu_$c.csv python tools/ncu_alu.py run $c > $OUT/alu_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/packedpre_c4m32 python tools/kcount.py c4 32 20 $((1 << 30)) > $OUT/ncu_pp.log 2>&1
