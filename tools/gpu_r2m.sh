OUT=gpurun_out/${1:-r2m}; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_shard.py -q -rxXs > $OUT/pytest_shard.log 2>&1; echo "shard pytest exit $?"; tail -4 $OUT/pytest_shard.log
timeout 1500 python -m pytest tests -q -m gpu -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
# sharded cfg3 on one GPU through the host transport (2 ranks): distributed vs replicated coarse
for v in 1 0; do
  BDDC_DIST_COARSE=$v timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --workload cfg3 --gpus 2 --steps 2 --warmup 1 --transport host --no-cpu-baseline > $OUT/bench_shard2_dist$v.log 2>&1; echo "shard bench dist=$v exit $?"
  tail -c 600 $OUT/bench_shard2_dist$v.log
done
