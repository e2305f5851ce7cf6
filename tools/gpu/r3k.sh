OUT=gpurun_out/r3k; mkdir -p $OUT
timeout 300 python tools/quick_time.py C1 C2 C3 C4 C5 > $OUT/qt.log 2>&1
MSHBM_NO_PRIO=1 timeout 300 python tools/quick_time.py C1 C2 C3 C4 C5 > $OUT/qt_noprio.log 2>&1
