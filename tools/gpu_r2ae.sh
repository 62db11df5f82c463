# panel group size / X1 chunk re-tuned at 4 CTAs/SM (variant libraries), cfg5 + cfg3
OUT=gpurun_out/${1:-r2ae}; mkdir -p $OUT
for v in default kg6 kg12 x512 default; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in cfg5 cfg3; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('$v $w', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'its', d['iterations'], 'coarse', p['setup.coarse']['avg_ms'], 'acoarse', p['apply.coarse']['avg_ms'])"
  done
done
