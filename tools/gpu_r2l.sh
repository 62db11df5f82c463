OUT=gpurun_out/${1:-r2l}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_shard.py -q -x -rxXs > $OUT/pytest_shard.log 2>&1; echo "shard pytest exit $?"; tail -15 $OUT/pytest_shard.log
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
