# quick GPU check: parity tests (pattern $K) + one bench workload ($W)
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests -m gpu -x -q ${K:+-k "$K"} > gpurun_out/quick/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/quick/tests.log
tail -3 gpurun_out/quick/tests.log
for w in ${W:-cfg3}; do
timeout 900 python bench.py --workload $w --steps ${STEPS:-3} --warmup 3 ${BARGS:---no-cpu-baseline} > gpurun_out/quick/bench_$w.log 2>&1; echo "bench $w exit $?"
done
