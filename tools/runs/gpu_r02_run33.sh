timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_c1_1024 python tools/run_once.py c 1 1024 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_abc1_1024b python tools/run_once.py abc 1 1024 > /dev/null 2>&1
