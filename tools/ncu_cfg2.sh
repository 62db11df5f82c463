# cfg2 (bench default): launch list (gpu__time_duration per kernel) + one --set full capture of
# each top kernel; summaries are written next to the reports (run on the GPU box)
mkdir -p gpurun_out/ncu2
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/ncu2/bench.log 2>&1; echo "bench exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ncu2/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2/list.log 2>&1
echo "list exit $?"
for k in coop_factor_df_kernel schur2d_kernel bt_solve_t_kernel coop_solve_df_kernel wfactor2d_kernel gemm_f64_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o gpurun_out/ncu2/$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2/full_$k.log 2>&1
  echo "full $k exit $?"
done
