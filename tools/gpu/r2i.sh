OUT=gpurun_out/r2j; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 C4 > $OUT/qt.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep4_kernel -c 1 -o $OUT/sweep4_c3 python tools/prof_once.py C3 > $OUT/sweep4_c3.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_sweep4.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
