# count-kernel rate vs text size (c5 text, m = 16, 8 patterns per call) and two dispatch knobs at 64 GiB
OUT=gpurun_out/${TAG:-sz}
mkdir -p $OUT
for g in 4 8 16 24 32 48 64; do timeout 300 python tools/kcount.py c5 16 8 $((g << 30)) >> $OUT/kc.log 2>&1; done
SMGPU_ALTERNATE=0 timeout 300 python tools/kcount.py c5 16 8 $((64 << 30)) >> $OUT/kc.log 2>&1; echo "  ^ alternate=0" >> $OUT/kc.log
SMGPU_DISPATCH=0 timeout 300 python tools/kcount.py c5 16 8 $((64 << 30)) >> $OUT/kc.log 2>&1; echo "  ^ dispatch=0" >> $OUT/kc.log
