set -x
mkdir -p gpurun_out/r2base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2base/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2base/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2base/pytest_gpu.log
for c in c3 c4 c1; do
  timeout 600 python bench.py --config $c --no-e2e --no-report --no-cpu --steps 3 > gpurun_out/r2base/cfg_$c.json 2>gpurun_out/r2base/cfg_$c.err
done
timeout 300 python tools/kbench.py --config c3 --lengths 4 --per-m 64 --batch --reps 3 > gpurun_out/r2base/kb_c3m4.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 6 -c 1 -o gpurun_out/r2base/ncu_pair_c3m4 python tools/kbench.py --config c3 --lengths 4 --per-m 64 --batch --reps 3 > gpurun_out/r2base/ncu.log 2>&1
echo done
