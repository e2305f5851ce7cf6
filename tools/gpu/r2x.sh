OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 C4 C5 > $OUT/qt.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --clock-control none --metrics $M -k regex:prior_select --csv --log-file $OUT/ps.csv python tools/prof_once.py C3 > /dev/null 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
