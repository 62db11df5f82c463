# round 2 first check: GPU tests, smoke, cfg5 cold-start breakdown
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a/smi.txt
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/r2a/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/r2a/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1; echo "smoke exit $?"
tail -2 gpurun_out/r2a/smoke.log
BDDC_HOST_TIMING=1 timeout 1200 python bench.py --workload cfg5 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2a/cfg5.log 2>&1; echo "cfg5 exit $?"
grep "bddc_setup host" gpurun_out/r2a/cfg5.log
tail -c 1500 gpurun_out/r2a/cfg5.log
