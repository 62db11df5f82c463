# coarse engine task profile (BDDC_COOP_TIMING) on cfg3 / cfg2, launch list of cfg3
OUT=gpurun_out/${1:-r2u}; mkdir -p $OUT
for w in cfg3 cfg2_L4h cfg2_Lh; do
  BDDC_COOP_TIMING=1 timeout 900 python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline > $OUT/coop_$w.log 2> $OUT/coop_$w.err; echo "coop $w exit $?"
  grep -A10 "simulated makespan\|coop factor" $OUT/coop_$w.err | tail -12
done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 3000 \
  --log-file $OUT/launches_cfg3.csv python bench.py --workload cfg3 --steps 2 --warmup 3 --no-cpu-baseline > $OUT/list.log 2>&1
echo "list exit $?"; python tools/launch_shares.py $OUT/launches_cfg3.csv > $OUT/launch_shares_cfg3.txt 2>&1; head -40 $OUT/launch_shares_cfg3.txt
