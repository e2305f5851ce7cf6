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
# implemented FLOP counts first: bench.py's roofline reads profiles/r02_flops.json
timeout 1500 python tools/flop_check.py capture $OUT/flops.json C1 C2 C3 C4 C5 > $OUT/flops.log 2>&1
cp $OUT/flops.json profiles/r02_flops.json
for c in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
done
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
# launch list (cold, serialised): shares only
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_bench_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
  --no-sharded > $OUT/launches.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
for c in C2 C3 C4 C5; do
  timeout 900 ncu --clock-control none --metrics $M --csv --log-file $OUT/stages_$c.csv \
    python tools/prof_once.py $c > $OUT/stages_$c.log 2>&1
done
# ncu --set full captures: the .ncu-rep stays in /tmp on the box (gpurun_out/ is capped at
# 64 MiB); the raw-page summary + per-source-line breakdown come back as markdown
cap() {  # cap <config> <kernel regex> <name>
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$2 -c 1 -f \
    -o /tmp/$3 python tools/prof_once.py $1 > $OUT/$3.log 2>&1
  python tools/ncu_summary.py /tmp/$3.ncu-rep "$TAG $3: $2 on $1 (ncu --set full, one launch)" \
    > $OUT/$3_ncu.md 2>> $OUT/$3.log
  ncu -i /tmp/$3.ncu-rep --page source --csv > /tmp/$3_source.csv 2>/dev/null
  python tools/sass_stalls.py /tmp/$3_source.csv 25 > $OUT/$3_sass_stalls.txt 2>> $OUT/$3.log
}
cap C3 sweep4_kernel sweep4_c3
cap C5 sweep4_kernel sweep4_c5
cap C3 prior_select prior_select_c3
timeout 900 python tools/band_scaling.py C5 2 4 8 > $OUT/bands.log 2>&1
echo done > $OUT/DONE
