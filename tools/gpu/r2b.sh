set -x
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2b/smoke.log 2>&1; echo smoke_rc=$?
timeout 900 python -m pytest tests -x -q -m gpu -s > gpurun_out/r2b/gpu.log 2>&1; echo gpu_rc=$?
for c in C3 C2 C4; do timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-sharded > gpurun_out/r2b/bench_$c.json 2> gpurun_out/r2b/bench_$c.err; echo bench_$c=$?; done
