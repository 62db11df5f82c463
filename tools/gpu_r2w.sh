# rotating-register operator sweep: 2 vs 3 CTAs/SM (variant library), parity subset
OUT=gpurun_out/${1:-r2w}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard.py -q -x -k "spmv or fused_pcg or apply_matches or shard" > $OUT/pytest_sub.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest_sub.log
for v in default sw3; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg2_L4h cfg3 cfg5; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'spmv', d['phases']['pcg.spmv_dot']['avg_ms'], d['phases']['pcg.spmv_dot']['frac'])"
  done
done
