mkdir -p gpurun_out/r2
timeout 1700 python -m pytest tests -q -m gpu -s > gpurun_out/r2/gpu4.log 2>&1; echo gpu_rc=$?
