# full-size pins + whole GPU suite on the committed sweep; ncu --set full of the operator sweep at cfg5
OUT=gpurun_out/${1:-r2s}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s -rxXs > $OUT/pytest_fullsize.log 2>&1; echo "fullsize exit $?"; grep "cfg" $OUT/pytest_fullsize.log | tail; tail -2 $OUT/pytest_fullsize.log
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs --deselect tests/test_gpu_fullsize.py > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
R=/tmp/ncu_reps; mkdir -p $R
for k in spmv_dot_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $R/$k python bench.py --workload cfg5 --steps 1 --warmup 3 --no-cpu-baseline > $OUT/full_$k.log 2>&1
  echo "full $k exit $?"
  python tools/ncu_summary.py $R/$k.ncu-rep > $OUT/summary_cfg5_$k.txt 2>&1
  python tools/ncu_lines.py $R/$k.ncu-rep 30 > $OUT/lines_cfg5_$k.txt 2>&1
  ncu -i $R/$k.ncu-rep --page details --csv > $OUT/details_cfg5_$k.csv 2>&1
done
cat $OUT/summary_*.txt
