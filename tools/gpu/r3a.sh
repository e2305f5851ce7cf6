OUT=gpurun_out/r3a; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt.log 2>&1
MSHBM_NO_FORK=1 timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt_nofork.log 2>&1
