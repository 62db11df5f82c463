# GPU test suite + smoke (usage: bash tools/gpu_tests.sh <outdir> [pytest args])
OUT=gpurun_out/${1:-tests}; shift
mkdir -p $OUT
timeout 1500 python -m pytest tests -q -m gpu -rxXs "$@" > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -25 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?"
tail -2 $OUT/smoke.log
