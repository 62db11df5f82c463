OUT=gpurun_out/${1:-r2p}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_cholesky" > $OUT/pytest_fused.log 2>&1; echo "fused pytest exit $?"; tail -3 $OUT/pytest_fused.log
for v in 1 0; do
  for w in cfg5 cfg3 cfg2_L4h; do
    BDDC_FUSED_CHOL=$v timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); p=d['phases']; print('fused=$v $w', d['value'], 'setup', d['setup_ms'], {k:(round(v['ms_total']/d['steps'],2), v.get('frac')) for k,v in p.items() if k in ('setup.SK','setup.Linv','setup.SKLinv')})"
  done
done
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
