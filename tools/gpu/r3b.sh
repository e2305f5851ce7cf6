OUT=gpurun_out/r3b; mkdir -p $OUT
timeout 300 python tools/quick_time.py C1 C2 C3 C4 C5 > $OUT/qt.log 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
