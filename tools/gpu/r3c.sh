OUT=gpurun_out/r3c; mkdir -p $OUT
timeout 300 python tools/quick_time.py C2 C3 C5 > $OUT/qt.log 2>&1
timeout 900 python tools/band_scaling.py C5 2 4 8 > $OUT/bands.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
