# cfg3: ncu --set full captures of the 3D interior elimination kernels
mkdir -p gpurun_out/ncu3s
for k in rh3d_kernel wfactor3d_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/ncu3s/$k python bench.py --workload cfg3 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu3s/$k.log 2>&1
  echo "$k exit $?"
done
