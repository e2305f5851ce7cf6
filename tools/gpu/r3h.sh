OUT=gpurun_out/r3h; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C4 > $OUT/qt.log 2>&1
MSHBM_SWEEP4_G=4 timeout 300 python tools/quick_time.py C2 C4 > $OUT/qt_g4.log 2>&1
