OUT=gpurun_out/r2m; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 C4 C5 > $OUT/qt.log 2>&1
MSHBM_SWEEP4_B3=1 timeout 300 python tools/quick_time.py C3 C5 > $OUT/qt_b3.log 2>&1
MSHBM_SWEEP4_B3=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -s > $OUT/gpu_b3.log 2>&1; echo gpu_rc=$? >> $OUT/gpu_b3.log
