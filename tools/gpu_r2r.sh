# sweep depth (rows in flight) A/B + the full-size pin test
OUT=gpurun_out/${1:-r2r}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -rxXs > $OUT/pytest_fullsize.log 2>&1; echo "fullsize exit $?"; tail -3 $OUT/pytest_fullsize.log
for w in cfg2_L4h cfg3 cfg5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1]); print('$w', d['value'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'spmv', d['phases']['pcg.spmv_dot'])"
done
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
