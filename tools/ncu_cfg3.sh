# cfg3 kernel launch list + full captures of the generic batched GEMM (3D setup)
mkdir -p gpurun_out/ncu3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/ncu3/launches.csv python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3/list.log 2>&1
echo "list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 40 -c 6 \
  -o gpurun_out/ncu3/gemm python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3/full.log 2>&1
echo "full exit $?"
