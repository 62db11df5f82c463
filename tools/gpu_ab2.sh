OUT=gpurun_out/${1:-ab2}; mkdir -p $OUT
run() {  # name, env...
  local v=$1; shift
  env "$@" timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "apply_matches or fused_pcg or l21 or scale" > $OUT/pytest_$v.log 2>&1; echo "$v pytest exit $?"; tail -1 $OUT/pytest_$v.log
  env "$@" timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_$v.log 2>&1
  python -c "import json; d=json.loads(open('$OUT/bench_$v.log').read().strip().splitlines()[-1]); print('$v', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'coarse', d['phases']['setup.coarse']['avg_ms'], 'acoarse', d['phases']['apply.coarse']['avg_ms'], 'first', d['first_setup_s'])"
}
run g8 FOO=1
run g12 BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_g12.so
run g16 BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_g16.so
run wide2048 BDDC_SOLVE_WIDE_SEP=2048
run wide512 BDDC_SOLVE_WIDE_SEP=512
run wide128 BDDC_SOLVE_WIDE_SEP=128
