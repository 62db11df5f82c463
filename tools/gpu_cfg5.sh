# cfg5 (256^3, 32^3 subdomains) on one GPU with aliased coarse fronts
mkdir -p gpurun_out/c5
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
( while true; do nvidia-smi --query-gpu=memory.used --format=csv,noheader >> gpurun_out/c5/mem.log; sleep 5; done ) &
MP=$!
timeout ${T5:-1500} python bench.py --workload cfg5 --steps ${S5:-1} --warmup ${W5:-1} --no-cpu-baseline > gpurun_out/c5/bench.log 2>&1; echo "cfg5 exit $?"
kill $MP
sort -n gpurun_out/c5/mem.log | tail -1
tail -c 3000 gpurun_out/c5/bench.log
