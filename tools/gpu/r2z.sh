OUT=gpurun_out/r2z; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 C5 > $OUT/qt.log 2>&1
MSHBM_SWEEP4_TH=16 timeout 300 python tools/quick_time.py C2 C3 C5 > $OUT/qt16.log 2>&1
MSHBM_SWEEP4_TH=24 timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt24.log 2>&1
M=gpu__time_duration.sum
timeout 600 ncu --clock-control none --metrics $M -k regex:prior_select --csv --log-file $OUT/ps.csv python tools/prof_once.py C3 > /dev/null 2>&1
