# cfg3: --set full of the dominant kernels (coarse dataflow factorization, batched GEMM, rh3d)
D=gpurun_out/ncu6; mkdir -p $D
for k in coop_factor_df_kernel rh3d_kernel local_gamma1_lower_kernel coop_solve_df_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 \
    -o $D/$k python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline > $D/full_$k.log 2>&1
  echo "full $k exit $?"
done
