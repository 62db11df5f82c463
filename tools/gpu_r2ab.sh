# final-code ncu evidence (4 CTAs/SM): DRAM bytes per launch at cfg5 (one pass), launch list of the default
# command, --set full of the coarse engine and the batched GEMM at cfg3 (summaries made on the box)
D=gpurun_out/${1:-r2ab}; mkdir -p $D
bash tools/ncu_dram_cfg5.sh ${1:-r2ab}/dram > $D/dram.log 2>&1; tail -12 $D/dram.log | cut -c1-250
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file $D/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $D/list.log 2>&1
echo "list exit $?"; python tools/launch_shares.py $D/launches_cfg5.csv > $D/launch_shares_cfg5.txt 2>&1; head -14 $D/launch_shares_cfg5.txt | cut -c1-120
R=/tmp/ncu_reps; mkdir -p $R
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 20 -c 10 \
  -o $R/gemm_f64 python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > $D/full_gemm.log 2>&1
echo "gemm exit $?"
python tools/ncu_summary.py $R/gemm_f64.ncu-rep > $D/summary_gemm_f64.txt 2>&1
for k in coop_factor_df_kernel coop_solve_df_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o $R/$k python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > $D/full_$k.log 2>&1
  echo "full $k exit $?"
  python tools/ncu_summary.py $R/$k.ncu-rep > $D/summary_$k.txt 2>&1
  python tools/ncu_lines.py $R/$k.ncu-rep 30 > $D/lines_$k.txt 2>&1
done
cat $D/summary_*.txt
