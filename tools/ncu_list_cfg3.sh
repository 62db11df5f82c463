mkdir -p gpurun_out/l3
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/l3/launches.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/l3/list.log 2>&1
echo "list exit $?"
