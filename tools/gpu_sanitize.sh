# compute-sanitizer evidence (one tool per pass): smoke (cfg1) + the cfg3a/cfg2a apply and PCG tests
OUT=gpurun_out/${1:-sanitize}; mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/${tool}_smoke.log 2>&1
  echo "$tool smoke exit $?"; tail -3 $OUT/${tool}_smoke.log
done
for tool in memcheck racecheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 python -m pytest tests -q -m gpu -x \
    -k "test_apply_matches_reference and (cfg3a_p1_ref or cfg2a_p1_L4h or cfg4a_p1_spec)" > $OUT/${tool}_tests.log 2>&1
  echo "$tool tests exit $?"; tail -3 $OUT/${tool}_tests.log
done
