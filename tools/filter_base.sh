# FILTER baseline: sustained c5 rate (64 GiB, 8 x m=16 per call) and a clean ncu capture (4 GiB)
OUT=gpurun_out/${TAG:-fb}
mkdir -p $OUT
KCOUNT_ITERS=${ITERS:-40} timeout 600 python tools/kcount.py c5 16 8 $((64 << 30)) >> $OUT/kc.log 2>&1
KCOUNT_ITERS=${ITERS:-40} timeout 600 python tools/kcount.py c3 16 64 $((1 << 30)) >> $OUT/kc.log 2>&1
KCOUNT_ITERS=${ITERS:-40} timeout 600 python tools/kcount.py c3 4 64 $((1 << 30)) >> $OUT/kc.log 2>&1
for m in 2 8 32; do KCOUNT_ITERS=${ITERS:-40} timeout 600 python tools/kcount.py c2 $m 64 0 >> $OUT/kc.log 2>&1; done
if [ -z "$NONCU" ]; then
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/c5m16_4g python tools/kcount.py c5 16 8 $((4 << 30)) > $OUT/ncu.log 2>&1
fi
