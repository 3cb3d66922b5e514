set -x
timeout 300 python tools/small_sizes.py 1024,1536,2048,3072 > gpurun_out/r02_small_sk.log 2>&1
STRASSEN_B200_STREAMK=0 timeout 300 python tools/small_sizes.py 1024,1536,2048,3072 > gpurun_out/r02_small_nosk.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest4.log 2>&1
