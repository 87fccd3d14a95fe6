# ncu --set full of the c5 count launch below and above the rate knee (16 vs 24 GiB text)
OUT=gpurun_out/${TAG:-szn}
mkdir -p $OUT
for g in 16 24; do
timeout 900 ncu --set full --import-source on --clock-control none -k regex:search_kernel --launch-skip 2 --launch-count 1 -o $OUT/c5m16_${g}g python tools/kcount.py c5 16 8 $((g << 30)) > $OUT/ncu_${g}.log 2>&1
done
