# PACKED b=1 A/B (c4 binary, c4p periodic) + parity/counter tests
OUT=gpurun_out/${TAG:-abp}
mkdir -p $OUT
for cm in "c4 8 20 1073741824" "c4 32 20 1073741824" "c4 512 20 1073741824"; do
  KCOUNT_ITERS=10 timeout 600 python tools/kcount.py $cm >> $OUT/kc.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_counters.py tests/test_gpu_configs.py tests/test_gpu_debug_checks.py -x -q -m gpu > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
