# 4 CTAs/SM defaults: full GPU suite (incl. full-size pins, checked build), every BASELINE config
OUT=gpurun_out/${1:-r2z}; mkdir -p $OUT
timeout 2400 python -m pytest tests -q -m gpu -x -s -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; grep "^\.\?cfg" $OUT/pytest_gpu.log | cut -c1-200; tail -4 $OUT/pytest_gpu.log
for w in cfg5 cfg3 cfg4 cfg2_L4h cfg2_Lh cfg2_L16h cfg2_LH cfg1; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('$w', d['value'], 'e2e', d['e2e']['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'coarse', p['setup.coarse']['avg_ms'], p['setup.coarse']['frac'])"
done
