# PAIR c3 m = 4 (the sigma >= 20 case furthest below its roofline): ncu --set full with source, for the
# per-line attribution of its shared-memory bank conflicts (tools/ncu_smem_lines.py)
OUT=gpurun_out/${TAG:-r2l}
mkdir -p $OUT
timeout 300 python tools/kcount.py c3 4 64 0 4 > $OUT/kcount_plain.log 2>&1; echo "exit $?" >> $OUT/kcount_plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/pair_c3m4 python tools/kcount.py c3 4 64 0 4 > $OUT/ncu_pair.log 2>&1
echo done
