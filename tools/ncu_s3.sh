# session 3: bench (clock sampling check) + launch list + --set full of the top setup kernels
D=${D:-gpurun_out/ncu3}; mkdir -p $D
timeout 600 python bench.py > $D/bench.log 2>&1; echo "bench exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $D/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $D/list.log 2>&1
echo "list exit $?"
for k in ${KS:-schur2d_kernel coop_factor_df_kernel wfactor2d_kernel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $D/$k python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $D/full_$k.log 2>&1
  echo "full $k exit $?"
done
