OUT=gpurun_out/${1:-r2o}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['setup_ms'], d['solve_ms'], d['phases']['setup.coarse']['avg_ms'], d['cold_e2e']['value'])"
