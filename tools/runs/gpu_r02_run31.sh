for spec in "abc 1 1024" "dgemm 0 1024" "abc 1 1536" "c 1 1024"; do timeout 120 python tools/cta_trace.py $spec 2>&1 | head -7; done > gpurun_out/r02_cta_trace4.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_small_launches.csv python tools/small_sizes.py 1024 abc1,dgemm0 > /dev/null 2>&1
