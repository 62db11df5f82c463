set -x
mkdir -p gpurun_out/s3
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/s3/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/s3/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/s3/smoke.log
timeout 600 python bench.py > gpurun_out/s3/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/s3/bench.log
timeout 600 python bench.py --workload cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s3/bench_cfg3.log 2>&1; echo "cfg3 exit $?" >> gpurun_out/s3/bench_cfg3.log
tail -3 gpurun_out/s3/gpu_tests.log gpurun_out/s3/smoke.log
tail -c 1500 gpurun_out/s3/bench.log
tail -c 1500 gpurun_out/s3/bench_cfg3.log
