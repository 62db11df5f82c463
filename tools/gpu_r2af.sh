# batched GEMM with 3 cp.async stages at 4 CTAs/SM (variant gs3); 512-wide coarse-solve tasks threshold
OUT=gpurun_out/${1:-r2af}; mkdir -p $OUT
for v in default gs3 default gs3; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg3 cfg5; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('$v $w', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'schur', p['setup.schur']['avg_ms'], 'SK', p['setup.SK']['avg_ms'], 'Linv', p['setup.Linv']['avg_ms'], 'Phi', p['setup.Phi']['avg_ms'], 'T', p['setup.T']['avg_ms'])"
  done
done
unset BDDC_LIB
for v in 1024 4096; do
  export BDDC_SOLVE_512_SEP=$v
  for w in cfg5 cfg3; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_s512_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_s512_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('s512=$v $w', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'acoarse', p['apply.coarse']['avg_ms'])"
  done
done
