# A/B (not adopted unless it wins): PAIR phase A takes the fifth word of pi(2)'s unaligned window from the
# neighbouring lane (__shfl_down) instead of a bank-conflicted LDS.32 -- ab/libsmgpu_shfl.so vs the tree's build
OUT=gpurun_out/${TAG:-r2m}
mkdir -p $OUT
for i in 1 2 3; do
  for lib in base shfl; do
    if [ $lib = shfl ]; then export SMGPU_LIB=$PWD/ab/libsmgpu_shfl.so; else unset SMGPU_LIB; fi
    for m in 3 4 8; do
      KCOUNT_ITERS=12 timeout 200 python tools/kcount.py c3 $m 64 0 4 >> $OUT/ab_$lib.log 2>&1
    done
  done
done
SMGPU_LIB=$PWD/ab/libsmgpu_shfl.so SEED=5 timeout 200 python tools/stress_parity.py 60 > $OUT/stress_shfl.log 2>&1; echo "exit $?" >> $OUT/stress_shfl.log
echo done
