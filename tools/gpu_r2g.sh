OUT=gpurun_out/${1:-r2g}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 $OUT/pytest_gpu.log
BDDC_HOST_TIMING=1 timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
grep "bddc_setup host" $OUT/bench.err | tail -30
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['setup_ms'], d['solve_ms'], d['cold_e2e'], d['prep_s'], d['first_setup_s'])"
