mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke3.log 2>&1; echo smoke_rc=$?
timeout 1700 python -m pytest tests -x -q -m gpu -s > gpurun_out/r2/gpu3.log 2>&1; echo gpu_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2/bench3.json 2> gpurun_out/r2/bench3.err; echo bench_rc=$?
