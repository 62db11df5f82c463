OUT=gpurun_out/${1:-ab4}; mkdir -p $OUT
BDDC_SOLVE_512_SEP=128 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x -k "apply_matches or fused_pcg or l21 or scale" > $OUT/pytest_512.log 2>&1; echo "512 pytest exit $?"; tail -1 $OUT/pytest_512.log
for v in 0 2048 512 128; do
  export BDDC_SOLVE_512_SEP=$v
  for w in cfg5 cfg3 cfg2_Lh; do
    timeout 900 python bench.py --workload $w --steps 3 --warmup 2 --no-cpu-baseline > $OUT/bench_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('$OUT/bench_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', d['value'], 'solve', d['solve_ms'], 'acoarse', d['phases']['apply.coarse']['avg_ms'], d['phases']['apply.coarse']['frac'])"
  done
done
