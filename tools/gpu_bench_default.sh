# default bench line (cfg5) with host-side cold-start timing, then the reference arm
OUT=gpurun_out/${1:-bench}; mkdir -p $OUT
nproc > $OUT/nproc.txt
BDDC_HOST_TIMING=1 timeout 1500 python bench.py > $OUT/bench.log 2> $OUT/bench.err; echo "bench exit $?"
grep "bddc_setup host" $OUT/bench.err | tail -30
tail -c 1500 $OUT/bench.log
timeout 600 python bench.py --impl reference > $OUT/ref.log 2>&1; echo "ref exit $?"; tail -c 600 $OUT/ref.log
