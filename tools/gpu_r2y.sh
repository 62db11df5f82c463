# half-epilogue GEMM tiles: 3 vs 4 CTAs/SM for the batched GEMM (g4) and the coarse engine (c4); cfg4 full-size diagnostics
OUT=gpurun_out/${1:-r2y}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -s -rxXs -k cfg4 > $OUT/pytest_fullsize_cfg4.log 2>&1; echo "fullsize cfg4 exit $?"; grep "^\.\?cfg" $OUT/pytest_fullsize_cfg4.log
timeout 900 python tools/coarse_forward_error.py cfg4 > $OUT/coarse_forward_error_cfg4.log 2>&1; echo "fwd exit $?"; tail -6 $OUT/coarse_forward_error_cfg4.log
timeout 900 python tools/coarse_forward_error.py cfg3 > $OUT/coarse_forward_error_cfg3.log 2>&1; echo "fwd exit $?"; tail -6 $OUT/coarse_forward_error_cfg3.log
for v in default g4 c4 default g4 c4; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg3 cfg5; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('$v $w', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d.get('iterations'), 'coarse', p['setup.coarse']['avg_ms'], 'schur', p['setup.schur']['avg_ms'], 'SK', p['setup.SK']['avg_ms'], 'Linv', p['setup.Linv']['avg_ms'], 'Phi', p['setup.Phi']['avg_ms'], 'T', p['setup.T']['avg_ms'])"
  done
done
unset BDDC_LIB
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x > $OUT/pytest_sub.log 2>&1; echo "pytest exit $?"; tail -2 $OUT/pytest_sub.log
