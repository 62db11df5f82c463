# tiled cp.async-ring operator sweep: parity + bench lines
OUT=gpurun_out/${1:-r2t}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -s -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; grep "^cfg" $OUT/pytest_gpu.log; tail -3 $OUT/pytest_gpu.log
for w in cfg2_L4h cfg3 cfg5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1]); print('$w', d['value'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'spmv', d['phases']['pcg.spmv_dot'])"
done
