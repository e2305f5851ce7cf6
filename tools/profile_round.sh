#!/bin/bash
# Round measurement on one B200 (run under gpurun):
#   gpurun --timeout 3600 -- 'bash tools/profile_round.sh r02'
# bench lines for every config, the reference arm, the ncu launch list of the
# default bench, per-stage metric tables (C3, C5), one `ncu --set full`
# capture each of the level-0 sweep4 and prior_select (C3), the implemented
# FLOP counts per config and the C5 band-scaling bound.
set -u
TAG=${1:-round}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
for c in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
# launch list (cold, serialised): shares only
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-sharded > $OUT/launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for c in C2 C3 C5; do
  timeout 900 ncu --clock-control none --metrics $M --csv --log-file $OUT/stages_$c.csv \
    python tools/prof_once.py $c > $OUT/stages_$c.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep4_kernel -c 1 \
  -o $OUT/sweep4_c3 python tools/prof_once.py C3 > $OUT/sweep4_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prior_select -c 1 \
  -o $OUT/prior_select_c3 python tools/prof_once.py C3 > $OUT/prior_select_c3.log 2>&1
timeout 1500 python tools/flop_check.py capture $OUT/flops.json C1 C2 C3 C4 C5 > $OUT/flops.log 2>&1
timeout 900 python tools/band_scaling.py C5 2 4 8 > $OUT/bands.log 2>&1
echo done > $OUT/DONE
