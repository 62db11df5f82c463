# one barrier per K slice in gemm_tile (default) vs two (variant ob0): parity subset + cfg3 / cfg5 / cfg2 lines
OUT=gpurun_out/${1:-r2aa}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_fullsize.py -q -x > $OUT/pytest_sub.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest_sub.log
for v in default ob0 default ob0; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg3 cfg5 cfg2_L4h; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('$v $w', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'coarse', p['setup.coarse']['avg_ms'], 'schur', p['setup.schur']['avg_ms'], 'SK', p['setup.SK']['avg_ms'], 'Linv', p['setup.Linv']['avg_ms'], 'Phi', p['setup.Phi']['avg_ms'])"
  done
done
