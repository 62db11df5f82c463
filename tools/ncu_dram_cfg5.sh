# DRAM bytes per launch of the two coarse engines (and the top local kernels) at the default
# workload (cfg5): dram__bytes_read/write are collected in one pass (no kernel replay)
D=gpurun_out/${1:-dram_cfg5}; mkdir -p $D
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  -k regex:'coop_|gamma1|gamma2|bt_solve|spmv_dot|residual_kernel' -c 40 --log-file $D/dram_cfg5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $D/ncu.log 2>&1
echo "ncu exit $?"; tail -3 $D/ncu.log | cut -c1-300
python - <<PY
import csv, collections
rows = list(csv.reader(open('$D/dram_cfg5.csv')))
hdr = None; acc = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        acc[d['Kernel Name'].split('(')[0][-48:]][d['Metric Name'] + ' ' + d['Metric Unit']].append(float(d['Metric Value'].replace(',', '')))
for k, m in acc.items():
    print(k, {n: (len(v), sum(v) / len(v)) for n, v in m.items()})
PY
