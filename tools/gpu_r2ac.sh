# W21 threshold re-tuned at 4 CTAs/SM (runtime env), cfg5 and cfg3
OUT=gpurun_out/${1:-r2ac}; mkdir -p $OUT
for v in 2048 1024 4096 512; do
  export BDDC_W21_MAX_SEP=$v
  for w in cfg5 cfg3; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_w21_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_w21_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('w21=$v $w', d['value'], 'setup', d['setup_ms'], 'solve', d['solve_ms'], 'coarse', p['setup.coarse']['avg_ms'], 'acoarse', p['apply.coarse']['avg_ms'])"
  done
done
