# sustained A/B of env knobs: VARIANTS="A=1 B=2;A=3" (';'-separated env sets), ITERS per kcount call
OUT=gpurun_out/${TAG:-abs}
mkdir -p $OUT
IFS=';' read -ra VS <<< "${VARIANTS:-}"
CASES=${CASES:-c5:16:8:68719476736 c3:16:64:1073741824 c2:8:64:0}
for cm in $CASES; do
  IFS=: read -r c m p n <<< "$cm"
  for v in "" "${VS[@]}"; do
    env $v KCOUNT_ITERS=${ITERS:-30} timeout 600 python tools/kcount.py $c $m $p $n >> $OUT/kc.log 2>&1; echo "  ^ [$v]" >> $OUT/kc.log
  done
done
