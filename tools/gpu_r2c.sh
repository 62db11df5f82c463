# grouped coarse engine: tests + cfg2/cfg3/cfg5 bench lines
OUT=gpurun_out/${OUTD:-r2c}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 $OUT/pytest_gpu.log
for w in cfg2_L4h cfg3; do
  timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1; echo "$w exit $?"
  python -c "import json,sys; d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1]); print('$w', d['value'], 'Mdof/s setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d['iterations'], 'coarse', d['phases'].get('setup.coarse'))"
done
BDDC_HOST_TIMING=1 timeout 1200 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench_cfg5.log 2>&1; echo "cfg5 exit $?"
grep "bddc_setup host" $OUT/bench_cfg5.log
python -c "import json,sys; d=json.loads(open('$OUT/bench_cfg5.log').read().strip().splitlines()[-1]); print('cfg5', d['value'], 'Mdof/s setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d['iterations'], 'coarse', d['phases'].get('setup.coarse'))"
