# round-2 final pass on the final build: r2_final.sh + ALU re-capture + FILTER/PAIR/PACKED ncu captures
TAG=${TAG:-r2final2} bash tools/r2_final.sh
OUT=gpurun_out/${TAG:-r2final2}
for c in c1 c4 c4p; do
  timeout 900 ncu --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:search_kernel --clock-control none --csv --log-file $OUT/alu_$c.csv python tools/ncu_alu.py run $c > $OUT/alu_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/filter_c5m16 python tools/kcount.py c5 16 8 $((4 << 30)) > $OUT/ncu_f.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/pair_c3m4 python tools/kcount.py c3 4 64 0 4 > $OUT/ncu_p.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/packedpre_c4m32 python tools/kcount.py c4 32 20 $((1 << 30)) > $OUT/ncu_pp.log 2>&1
echo done2
