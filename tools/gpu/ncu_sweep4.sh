#!/bin/bash
# ncu --set full capture of the level-0 sweep4 kernel of one config; exports the raw and
# source pages as CSV (the .ncu-rep stays on the box: gpurun_out/ is capped at 64 MiB)
#   bash tools/gpu/ncu_sweep4.sh C3 tag [kernel-regex]
CFG=$1; TAG=$2; K=${3:-sweep4_kernel}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$K -c 1 -f \
  -o /tmp/$TAG python tools/prof_once.py $CFG > $OUT/run.log 2>&1
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i /tmp/$TAG.ncu-rep --page source --csv > $OUT/source.csv 2>/dev/null
python tools/ncu_summary.py /tmp/$TAG.ncu-rep "$TAG ($CFG, $K)" > $OUT/summary.md 2>/dev/null
ls -la $OUT
