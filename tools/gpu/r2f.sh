OUT=gpurun_out/r2f; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt.log 2>&1
MSHBM_SWEEP4_G=4 timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt_g4.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
timeout 600 ncu --clock-control none --metrics $M --csv --log-file $OUT/stages_C3.csv python tools/prof_once.py C3 > $OUT/stages_C3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep4_kernel -c 1 -o $OUT/sweep4_c3 python tools/prof_once.py C3 > $OUT/sweep4_c3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:prior_select -c 1 -o $OUT/psel_c3 python tools/prof_once.py C3 > $OUT/psel_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_sweep4.py -x -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
