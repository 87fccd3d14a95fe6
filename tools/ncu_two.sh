# ncu --set full of the FILTER (c5 m = 16, 4 GiB) and PAIR (c3 m = 4, 256 MiB) count launches
OUT=gpurun_out/${TAG:-n2}
mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/filter_c5m16 python tools/kcount.py c5 16 8 $((4 << 30)) > $OUT/ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/pair_c3m4 python tools/kcount.py c3 4 64 0 4 > $OUT/ncu2.log 2>&1
