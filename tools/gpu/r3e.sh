OUT=gpurun_out/r3e; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 C5 > $OUT/qt.log 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum
timeout 900 ncu --clock-control none --metrics $M --csv --log-file $OUT/stages_C5.csv python tools/prof_once.py C5 > $OUT/stages_C5.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_gpu_oracle.py -x -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
