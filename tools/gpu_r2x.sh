# final-state evidence: full-size pins (cfg2 / cfg3 / cfg4), whole GPU suite, smoke, default bench + reference arm
OUT=gpurun_out/${1:-r2x}; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s -rxXs > $OUT/pytest_fullsize.log 2>&1; echo "fullsize exit $?"; grep "^\.\?cfg" $OUT/pytest_fullsize.log; tail -2 $OUT/pytest_fullsize.log
timeout 1500 python -m pytest tests -q -m gpu -x -rxXs --deselect tests/test_gpu_fullsize.py > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $OUT/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"; tail -3 $OUT/smoke.log
timeout 1200 python bench.py > $OUT/bench_default.log 2> $OUT/bench_default.err; echo "bench exit $?"; tail -1 $OUT/bench_default.log | cut -c1-600
timeout 1200 python bench.py --impl reference > $OUT/bench_reference.log 2> $OUT/bench_reference.err; echo "ref exit $?"; tail -1 $OUT/bench_reference.log | cut -c1-600
