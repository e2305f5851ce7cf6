OUT=gpurun_out/r2t; mkdir -p $OUT
timeout 1500 python tools/flop_check.py capture $OUT/flops.json C1 C2 C3 C4 C5 > $OUT/flops.log 2>&1; echo flops_rc=$? >> $OUT/flops.log
cp $OUT/flops.json profiles/r02_flops.json 2>/dev/null
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo bench_rc=$? >> $OUT/bench.err
