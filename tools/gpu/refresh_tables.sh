OUT=gpurun_out/r02e; mkdir -p $OUT
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for c in C2 C3 C4 C5; do
  timeout 900 ncu --clock-control none --metrics $M --csv --log-file $OUT/stages_$c.csv python tools/prof_once.py $c > $OUT/stages_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sharded > $OUT/launches.log 2>&1
for c in C1 C2 C4; do timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2>$OUT/bench_$c.err; done
timeout 600 python bench.py > $OUT/bench_C3.json 2>$OUT/bench_C3.err
timeout 900 python bench.py --config C5 > $OUT/bench_C5.json 2>$OUT/bench_C5.err
