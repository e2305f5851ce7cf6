#!/bin/bash
# Round measurement on one B200 (run under gpurun): bench lines for every
# config, the ncu launch list of the default bench, per-stage metric tables
# (C2, C5) and one `ncu --set full` capture of the level-0 sweep (C2).
#   gpurun --timeout 2400 -- 'bash tools/profile_round.sh'
set -u
OUT=gpurun_out/round
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt
for c in C1 C2 C3 C4 C5; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 300 python bench.py --impl reference > $OUT/bench_reference_c2.json 2> $OUT/bench_reference_c2.err
# launch list (cold, serialised): shares only
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_bench_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  > $OUT/launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for c in C2 C5; do
  timeout 900 ncu --clock-control none --metrics $M --csv --log-file $OUT/stages_$c.csv \
    python tools/prof_once.py $c > $OUT/stages_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep4 -c 1 \
  -o $OUT/sweep4_c2 python tools/prof_once.py C2 > $OUT/sweep4_c2.log 2>&1
echo done > $OUT/DONE
