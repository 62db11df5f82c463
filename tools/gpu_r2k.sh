# full GPU tests (incl. the checked build), the default bench line with the CPU legs, the
# reference arm, the launch list of the default command
OUT=gpurun_out/${1:-r2k}; mkdir -p $OUT
timeout 1800 python -m pytest tests -q -m gpu -x -rxXs > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $OUT/smoke.log
BDDC_HOST_TIMING=1 timeout 1200 python bench.py > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
python -c "import json; d=json.loads(open('$OUT/bench.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['setup_ms'], d['solve_ms'], d['cold_e2e'], d['cpu_baseline']['value'], d['roofline'], d['clocks'])"
timeout 900 python bench.py --impl reference > $OUT/ref.log 2>&1; echo "ref exit $?"; tail -c 400 $OUT/ref.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv -c 1500 \
  --log-file $OUT/launches_cfg5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/list.log 2>&1
echo "list exit $?"; python tools/launch_shares.py $OUT/launches_cfg5.csv > $OUT/launch_shares_cfg5.txt 2>&1; head -16 $OUT/launch_shares_cfg5.txt
