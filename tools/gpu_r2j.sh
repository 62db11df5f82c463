OUT=gpurun_out/${1:-r2j}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['setup_ms'], d['solve_ms'], d['apply_ms'], d['first_setup_s']); print({k:(v['avg_ms'], v.get('frac')) for k,v in d['phases'].items()})"
for w in cfg2_L4h cfg3; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1; echo "$w exit $?"
  python -c "import json; d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1]); print('$w', d['value'], d['setup_ms'], d['solve_ms'], d['apply_ms'], d['iterations']); print({k:(v['avg_ms'], v.get('frac')) for k,v in d['phases'].items()})"
done
BDDC_COOP_TIMING=1 timeout 900 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/coop.log 2> $OUT/coop.err; echo "coop exit $?"
grep -v "^bddc_setup" $OUT/coop.err | head -12
