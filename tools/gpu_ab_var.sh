# A/B of variant libraries (VARS) on workloads (W): bench lines + phase summary
OUT=gpurun_out/${1:-abvar}; mkdir -p $OUT
for rep in 1 2; do
for v in ${VARS:-default}; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for w in ${W:-cfg3}; do
    timeout 900 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_${v}_${w}_$rep.log 2>&1
    python - <<PY
import json
d=json.loads(open('$OUT/bench_${v}_${w}_$rep.log').read().strip().splitlines()[-1])
print('$v $w', d['value'], 'setup', d['setup_ms'], 'its', d.get('iterations'), {k[6:]: round(v['avg_ms'],3) for k,v in d['phases'].items() if k.startswith('setup')})
PY
  done
done
done
