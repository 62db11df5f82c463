# A/B of the coarse panel group size (libvar_g6 / libvar_g8 vs default 4): parity subset + benches
OUT=gpurun_out/${1:-ab_group}; mkdir -p $OUT
for v in default g6 g8; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "apply_matches or fused_pcg or l21" > $OUT/pytest_$v.log 2>&1; echo "$v pytest exit $?"; tail -1 $OUT/pytest_$v.log
  for w in cfg5 cfg3 cfg2_L4h; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'setup', d['setup_ms'], 'coarse', d['phases']['setup.coarse']['avg_ms'], 'first_setup', d['first_setup_s'])"
  done
done
