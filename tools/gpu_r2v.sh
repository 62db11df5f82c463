OUT=gpurun_out/${1:-r2v}; mkdir -p $OUT
BDDC_COOP_TIMING=1 timeout 1200 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-cpu-baseline > $OUT/coop_cfg5.log 2> $OUT/coop_cfg5.err; echo "coop exit $?"
grep "simulated makespan" $OUT/coop_cfg5.err | tail -1; grep -A10 "coop factor (dataflow)" $OUT/coop_cfg5.err | tail -10
