set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest5.log 2>&1
timeout 300 python tools/small_sizes.py 1024,1536,2048,3072 dgemm0,abc1,naive1,abc2,c2 > gpurun_out/r02_small5.log 2>&1
FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 1024 abc 2 32768 32768 1024 c 2 16384 16384 256 c 1 32768 32768 1024 dgemm 0 16384 16384 256 dgemm 0 16384 16384 1024 > gpurun_out/r02_shortk_group.log 2>&1
STRASSEN_B200_UNIT_GROUP=0 FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 1024 abc 2 32768 32768 1024 c 2 16384 16384 256 c 1 32768 32768 1024 > gpurun_out/r02_shortk_nogroup.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_small_dgemm1024 python tools/run_once.py dgemm 0 1024 > gpurun_out/r02_small_dgemm1024.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_small_abc1_1024 python tools/run_once.py abc 1 1024 > gpurun_out/r02_small_abc1_1024.log 2>&1
