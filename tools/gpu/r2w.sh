OUT=gpurun_out/r2w; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -s > $OUT/full.log 2>&1; echo rc=$? >> $OUT/full.log
