# full GPU tests + bench lines of the BASELINE workloads (summary per line)
OUT=gpurun_out/${1:-r2q}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
for w in ${W:-cfg3 cfg2_L4h cfg5}; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1
  python - <<PY
import json
d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1])
print('$w', d['value'], 'e2e', d['e2e']['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d.get('iterations'))
print('   ', {k: (round(v['avg_ms'],3), v.get('frac')) for k,v in d['phases'].items()})
PY
done
