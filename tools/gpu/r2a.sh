set -x
mkdir -p gpurun_out/r2a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo bench_rc=$?
timeout 2000 python -m pytest tests -q -m gpu -s --durations=30 > gpurun_out/r2a/gpu.log 2>&1; echo gpu_rc=$?
