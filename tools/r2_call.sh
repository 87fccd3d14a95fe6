# round-2 GPU call: tests, ALU probe + ALU work of the compare-bound configs, per-config
# bench lines (c1 c3 c4 c4p c5), a full ncu capture of c3 m = 4 (PAIR), sanitizers.
# Sections are selected by $SECTIONS (default all); output in gpurun_out/$TAG.
set -x
OUT=gpurun_out/${TAG:-call}
mkdir -p $OUT
S=${SECTIONS:-tests probe alu cfg c5 ncu san}
# also: ab (tools/r2_ab.sh), abl (tools/ablation_r2.py orders + r sweep), bench (default bench line)
has() { case " $S " in *" $1 "*) return 0;; esac; return 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $OUT/smi.txt 2>&1
if has tests; then
  timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
fi
if has probe; then
  timeout 300 python tools/alu_probe.py --out $OUT/alu_probe_r2.json > $OUT/alu_probe.log 2>&1
fi
if has alu; then
  for c in c4 c4p c1; do
    timeout 900 ncu --metrics smsp__inst_executed_pipe_alu.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
      --clock-control none -k regex:search_kernel --csv --log-file $OUT/alu_$c.csv python tools/ncu_alu.py run $c > $OUT/alu_$c.log 2>&1
  done
fi
if has cfg; then
  for c in ${CONFIGS:-c1 c3 c4 c4p}; do
    timeout 900 python bench.py --config $c --no-e2e --no-report --no-cpu --steps 3 > $OUT/cfg_$c.json 2>$OUT/cfg_$c.err
  done
fi
if has c5; then
  timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 > $OUT/cfg_c5.json 2>$OUT/cfg_c5.err
fi
if has ncu; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:search_kernel -s 6 -c 1 -o $OUT/ncu_pair_c3m4 python tools/kbench.py --config c3 --lengths 4 --per-m 64 --batch --reps 3 > $OUT/ncu_c3m4.log 2>&1
fi
if has san; then
  OUT=$OUT/san bash tools/sanitize.sh > $OUT/sanitize.log 2>&1
fi
if has ab; then
  TAG=${TAG:-call} bash tools/r2_ab.sh > $OUT/ab.log 2>&1
fi
if has abl; then
  timeout 900 python tools/ablation_r2.py --mode orders --configs c2,c3,c1 > $OUT/ablation_orders.jsonl 2> $OUT/ablation_orders.err
  timeout 900 python tools/ablation_r2.py --mode rsweep --configs c1,c3,c4 --lengths 8,16,32,128 > $OUT/ablation_rsweep.jsonl 2> $OUT/ablation_rsweep.err
fi
if has bench; then
  timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
fi
if [ -n "$EXTRA" ]; then bash -c "$EXTRA"; fi
echo done
