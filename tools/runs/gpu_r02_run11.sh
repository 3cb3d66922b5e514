set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest11.log 2>&1
for pm in 0 1; do STRASSEN_B200_PAIR=$pm FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 1024 abc 2 32768 32768 1024 c 2 16384 16384 256 c 2 16384 16384 1024 c 1 32768 32768 1024 abc 1 32768 32768 1024 abc 2 16384 16384 4096 c 2 16384 16384 16384 abc 2 16384 16384 16384 > gpurun_out/r02_pair_$pm.log 2>&1; done
