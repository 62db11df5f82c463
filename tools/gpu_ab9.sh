OUT=gpurun_out/${1:-ab9}; mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
for v in default nopfc default nopfc; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg5 cfg3 cfg2_L4h; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'setup', d['setup_ms'], 'coarse', d['phases']['setup.coarse']['avg_ms'], 'its', d['iterations'])"
  done
done
