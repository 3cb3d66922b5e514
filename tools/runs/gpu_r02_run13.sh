set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest13.log 2>&1
for pm in 0 1; do STRASSEN_B200_PAIR=$pm FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 4096 abc 2 16384 16384 16384 c 2 16384 16384 4096 abc 1 16384 16384 4096 abc 2 32768 32768 1024 > gpurun_out/r02_pair13_$pm.log 2>&1; done
