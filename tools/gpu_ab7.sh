OUT=gpurun_out/${1:-ab7}; mkdir -p $OUT
export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_x512.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "apply_matches or fused_pcg or l21 or scale or aliased" > $OUT/pytest_x512.log 2>&1; echo "x512 pytest exit $?"; tail -1 $OUT/pytest_x512.log
for v in default x512 default x512; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg5 cfg3; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'setup', d['setup_ms'], 'coarse', d['phases']['setup.coarse']['avg_ms'], 'its', d['iterations'])"
  done
done
