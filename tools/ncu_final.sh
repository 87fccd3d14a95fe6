# final-build ncu --set full captures: FILTER (c5 m = 16, 4 GiB), PAIR (c3 m = 4, 256 MiB), hist (c2 text)
OUT=gpurun_out/${TAG:-nf}
mkdir -p $OUT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "histogram or fig1 or seams" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 600 python tools/hist_probe.py > $OUT/hp.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/filter_c5m16 python tools/kcount.py c5 16 8 $((4 << 30)) > $OUT/ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/pair_c3m4 python tools/kcount.py c3 4 64 0 4 > $OUT/ncu2.log 2>&1
