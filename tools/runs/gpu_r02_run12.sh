set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest12.log 2>&1
FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py c 2 16384 16384 16384 abc 2 16384 16384 16384 naive 2 16384 16384 16384 dgemm 0 16384 16384 16384 > gpurun_out/r02_big12.log 2>&1
for pm in 0 1; do STRASSEN_B200_PAIR=$pm FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 512 abc 2 16384 16384 1024 abc 2 16384 16384 2048 abc 1 16384 16384 256 abc 1 16384 16384 1024 c 2 16384 16384 512 > gpurun_out/r02_pair12_$pm.log 2>&1; done
