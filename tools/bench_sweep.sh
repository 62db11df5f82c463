# Runs bench.py over every BASELINE config workload (one GPU), logs under gpurun_out/sweep/
mkdir -p gpurun_out/sweep; : > gpurun_out/sweep/status.txt
for w in ${WORKLOADS:-cfg1 cfg2_L4h cfg2_Lh cfg2_L16h cfg2_LH cfg3 cfg4 cfg5}; do
  timeout $([ $w = cfg5 ] && echo 1800 || echo ${WT:-900}) python bench.py --workload $w --steps ${STEPS:-5} --warmup 3 > gpurun_out/sweep/$w.log 2>&1
  echo "$w exit $?" >> gpurun_out/sweep/status.txt
  nvidia-smi --query-gpu=memory.used --format=csv >> gpurun_out/sweep/status.txt
done
