OUT=gpurun_out/r2v; mkdir -p $OUT
timeout 300 python tools/quick_time.py C1 C2 C3 C4 C5 > $OUT/qt.log 2>&1
