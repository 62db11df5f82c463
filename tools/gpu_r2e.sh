OUT=gpurun_out/${1:-r2e}; mkdir -p $OUT
timeout 900 python -m pytest tests/test_index_device.py -q -x -rxXs > $OUT/pytest_index.log 2>&1; echo "pytest exit $?"; tail -5 $OUT/pytest_index.log
for a in "20 2 1" "20 2 4" "20 2 16" "20 8 0" "20 8 8"; do timeout 300 ./tools/vmm_probe $a; done > $OUT/vmm.log 2>&1; cat $OUT/vmm.log
