# round 2: GPU tests, launch list of the default bench (cfg5) + --set full of the top kernels on
# cfg3, summarised on the box (the .ncu-rep files are too large to bring back)
D=gpurun_out/${1:-ncu_r2}; mkdir -p $D
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs > $D/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $D/pytest_gpu.log
BDDC_HOST_TIMING=1 timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $D/bench.log 2> $D/bench.err; echo "bench exit $?"
grep "bddc_setup host" $D/bench.err | tail -30
python -c "import json; d=json.loads(open('$D/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['setup_ms'], d['solve_ms'], d['cold_e2e'])"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 1200 \
  --log-file $D/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $D/list.log 2>&1
echo "list exit $?"; python tools/launch_shares.py $D/launches_cfg5.csv > $D/launch_shares_cfg5.txt 2>&1; head -30 $D/launch_shares_cfg5.txt
R=/tmp/ncu_reps; mkdir -p $R
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 20 -c 10 \
  -o $R/gemm_f64 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > $D/full_gemm.log 2>&1
echo "gemm exit $?"
python tools/ncu_summary.py $R/gemm_f64.ncu-rep > $D/summary_gemm_f64.txt 2>&1
ncu -i $R/gemm_f64.ncu-rep --page details --csv > $D/details_gemm_f64.csv 2>&1
for k in coop_factor_df_kernel coop_solve_df_kernel rh3d_kernel wfactor3d_kernel spmv_dot_kernel potrf trtri_from local_gamma1_lower; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o $R/$k python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > $D/full_$k.log 2>&1
  echo "full $k exit $?"
  python tools/ncu_summary.py $R/$k.ncu-rep > $D/summary_$k.txt 2>&1
  python tools/ncu_lines.py $R/$k.ncu-rep 30 > $D/lines_$k.txt 2>&1
  ncu -i $R/$k.ncu-rep --page details --csv > $D/details_$k.csv 2>&1
done
cat $D/summary_*.txt
du -sh $D
