set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest7.log 2>&1
FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 1024 abc 2 32768 32768 1024 c 2 16384 16384 256 abc 2 16384 16384 16384 > gpurun_out/r02_shortk7.log 2>&1
timeout 1200 python tools/sweep.py square gpurun_out/r02_sweep_square.csv > gpurun_out/r02_sweep_square.log 2>&1
timeout 1200 python tools/sweep.py rankk gpurun_out/r02_sweep_rankk.csv > gpurun_out/r02_sweep_rankk.log 2>&1
timeout 900 python tools/sweep.py fixedk gpurun_out/r02_sweep_fixedk.csv > gpurun_out/r02_sweep_fixedk.log 2>&1
