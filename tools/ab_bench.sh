# A/B: the default library and variant libraries (BDDC_LIB) on the same box, cfg2 bench lines
mkdir -p gpurun_out/ab
for v in ${VARS:-default}; do
  if [ "$v" = default ]; then unset BDDC_LIB; else export BDDC_LIB=$PWD/paper_2001_07289_b200/libvar_$v.so; fi
  for rep in 1 2; do
    timeout 600 python bench.py --no-cpu-baseline ${BARGS} > gpurun_out/ab/bench_${v}_$rep.log 2>&1; echo "$v $rep exit $?"
  done
done
