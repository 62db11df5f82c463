OUT=gpurun_out/${1:-pcgfuse}; mkdir -p $OUT
for w in cfg2_L4h cfg3 cfg2_Lh cfg5; do
  timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_$w.log 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_$w.log').read().strip().splitlines()[-1]); print('$w', d['value'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'launches', d.get('gpu_launches'))"
done
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
