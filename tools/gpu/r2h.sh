OUT=gpurun_out/r2h; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt.log 2>&1
MSHBM_S4_NOFENCE=1 timeout 300 python tools/quick_time.py C2 C3 > $OUT/qt_nf.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sweep4_kernel -c 1 -o $OUT/sweep4_c3 python tools/prof_once.py C3 > $OUT/sweep4_c3.log 2>&1
