# full GPU check: smoke, all -m gpu tests, quick timings.  OUT=gpurun_out/$1
OUT=gpurun_out/${1:-full}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo smoke_rc=$? >> $OUT/smoke.log
timeout 300 python tools/quick_time.py C2 C3 C4 > $OUT/qt.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu > $OUT/gpu.log 2>&1; echo gpu_rc=$? >> $OUT/gpu.log
