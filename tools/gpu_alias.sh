# aliased coarse fronts: parity tests, then cfg3 with aliasing forced (memory + time vs resident)
mkdir -p gpurun_out/al
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "aliased or apply_matches" > gpurun_out/al/tests.log 2>&1; echo "tests exit $?" >> gpurun_out/al/tests.log
tail -3 gpurun_out/al/tests.log
BDDC_FRONT_ALIAS=1 timeout 900 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/al/bench_cfg3_alias.log 2>&1; echo "cfg3 alias exit $?"
tail -c 400 gpurun_out/al/bench_cfg3_alias.log
