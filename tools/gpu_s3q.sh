# quick check: GPU parity tests + cfg2 (default) bench line [+ cfg3 when Q3=1]
mkdir -p gpurun_out/q
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/q/tests.log
tail -2 gpurun_out/q/tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/q/bench_cfg2.log 2>&1; echo "cfg2 exit $?"
if [ "${Q3:-0}" = 1 ]; then
timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/q/bench_cfg3.log 2>&1; echo "cfg3 exit $?"
fi
