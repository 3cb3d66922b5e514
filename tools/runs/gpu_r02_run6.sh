set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest6.log 2>&1
FMAX=2 REPS=3 timeout 600 python tools/fuse_probe.py abc 2 16384 16384 256 abc 2 16384 16384 1024 abc 2 32768 32768 1024 c 2 16384 16384 256 c 1 32768 32768 1024 abc 2 16384 16384 16384 > gpurun_out/r02_shortk6.log 2>&1
timeout 300 python tools/small_sizes.py 1024,1536,2048 dgemm0,abc1,abc2,naive2 > gpurun_out/r02_small6.log 2>&1
