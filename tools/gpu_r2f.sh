OUT=gpurun_out/${1:-r2f}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 $OUT/pytest_gpu.log
BDDC_HOST_TIMING=1 timeout 1200 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
grep "bddc_setup host" $OUT/bench.err | tail -30
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['setup_ms'], d['solve_ms'], d['cold_e2e'], d['prep_s'], d['first_setup_s'])"
BDDC_COOP_TIMING=1 timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $OUT/coop.log 2> $OUT/coop.err; echo "coop exit $?"
grep -i "coarse\|coop\|task" $OUT/coop.err | tail -40
