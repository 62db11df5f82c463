OUT=gpurun_out/${1:-ab3}; mkdir -p $OUT
for v in wide narrow; do
  if [ $v = narrow ]; then export BDDC_SOLVE_WIDE_SEP=0; else unset BDDC_SOLVE_WIDE_SEP; fi
  for w in cfg2_L4h cfg3 cfg2_Lh; do
    timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'solve', d['solve_ms'], 'acoarse', d['phases']['apply.coarse']['avg_ms'], d['phases']['apply.coarse']['frac'])"
  done
done
unset BDDC_SOLVE_WIDE_SEP
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
