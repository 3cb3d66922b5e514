set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest2.log 2>&1
for d in 0 1; do STRASSEN_B200_DYN=$d FMAX=2 REPS=3 timeout 300 python tools/fuse_probe.py naive 2 16384 16384 16384 c 2 16384 16384 16384 dgemm 0 16384 16384 16384 c 1 32768 32768 1024 > gpurun_out/r02_dyn$d.log 2>&1; done
FMAX=2 timeout 300 python tools/fuse_probe.py abc 2 16384 16384 16384 abc 2 32768 32768 1024 ab 2 16384 16384 16384 abc 1 1024 1024 1024 abc 2 1024 1024 1024 > gpurun_out/r02_default_f2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_cfg4_abc2 python tools/run_once.py abc 2 32768 32768 1024 > gpurun_out/r02_cfg4_abc2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_cfg4_c1 python tools/run_once.py c 1 32768 32768 1024 > gpurun_out/r02_cfg4_c1.log 2>&1
