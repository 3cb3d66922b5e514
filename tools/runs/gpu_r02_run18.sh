set -x
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest18.log 2>&1
FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py c 1 22528 22528 1024 c 1 20480 20480 1024 c 1 24576 24576 1024 > gpurun_out/r02_c1_22528.log 2>&1
