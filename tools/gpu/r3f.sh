OUT=gpurun_out/r3f; mkdir -p $OUT
timeout 300 python tools/quick_time.py C3 C5 > $OUT/qt.log 2>&1
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:downsample --csv --log-file $OUT/ds.csv python tools/prof_once.py C5 > /dev/null 2>&1
