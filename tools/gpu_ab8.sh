OUT=gpurun_out/${1:-ab8}; mkdir -p $OUT
BDDC_GROUP_MIN_SEP=4096 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "apply_matches or fused_pcg or l21 or scale or aliased" > $OUT/pytest_g4096.log 2>&1; echo "g4096 pytest exit $?"; tail -1 $OUT/pytest_g4096.log
for v in 0 512 1024 2048 4096; do
  export BDDC_GROUP_MIN_SEP=$v
  for w in cfg5 cfg3 cfg2_L4h cfg2_Lh; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'setup', d['setup_ms'], 'coarse', d['phases']['setup.coarse']['avg_ms'], 'its', d['iterations'])"
  done
done
