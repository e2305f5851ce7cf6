set -x
mkdir -p gpurun_out/r2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -x -q -s -m gpu > gpurun_out/r2/full.log 2>&1; echo full_rc=$?
python bench.py --config C3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2/bench_c3.json 2> gpurun_out/r2/bench_c3.err; echo bench_rc=$?
