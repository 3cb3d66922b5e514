set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest16.log 2>&1
timeout 300 python tools/small_sizes.py 1024,1536,2048 dgemm0,abc1,c1 > gpurun_out/r02_small16.log 2>&1
timeout 600 python tools/overhead_probe.py dgemm0,abc1 1536,1024 16,256,1024 > gpurun_out/r02_overhead16.log 2>&1
