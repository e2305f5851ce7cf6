mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s -m gpu > gpurun_out/r2/full2.log 2>&1; echo full_rc=$?
