OUT=gpurun_out/${1:-r2n}; mkdir -p $OUT
BDDC_HOST_TIMING=1 timeout 1200 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
grep "bddc_setup host" $OUT/bench.err | tail -22
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['setup_ms'], d['solve_ms'], d['cold_e2e'])"
