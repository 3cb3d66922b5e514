set -x
timeout 900 python bench.py > gpurun_out/r02_bench_final.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_final.csv python bench.py --steps 2 --warmup 1 --no-variants --no-e2e --no-cpu --no-classical > gpurun_out/r02_ncu_bench_final.log 2>&1
FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 1024 abc 2 32768 32768 1024 abc 1 32768 32768 1024 c 1 32768 32768 1024 dgemm 0 16384 16384 1024 dgemm 0 16384 16384 256 dgemm 0 32768 32768 1024 > gpurun_out/r02_cfg34_final.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_abc2_k256 python tools/run_once.py abc 2 16384 16384 256 > gpurun_out/r02_ncu_abc2_k256.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_abc2_cfg4 python tools/run_once.py abc 2 32768 32768 1024 > gpurun_out/r02_ncu_abc2_cfg4.log 2>&1
