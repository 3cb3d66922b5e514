set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest14.log 2>&1
for gm in 2 3; do STRASSEN_B200_GROUP_MAX=$gm FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 512 abc 2 16384 16384 1024 abc 2 16384 16384 4096 abc 1 16384 16384 256 abc 1 16384 16384 1024 c 2 16384 16384 256 c 2 16384 16384 1024 abc 2 32768 32768 1024 c 1 32768 32768 1024 abc 1 32768 32768 1024 > gpurun_out/r02_group14_$gm.log 2>&1; done
