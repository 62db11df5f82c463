set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_r1s2.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_r1s2.log
tail -3 gpurun_out/gpu_tests.log gpurun_out/smoke.log
tail -c 600 gpurun_out/bench_r1s2.log
