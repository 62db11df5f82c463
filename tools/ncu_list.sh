# launch list (per-kernel device time) of one bench workload: W=<workload>
mkdir -p gpurun_out/list
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/list/launches_${W:-cfg3}.csv python bench.py --workload ${W:-cfg3} --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/list/list_${W:-cfg3}.log 2>&1
echo "list exit $?"
