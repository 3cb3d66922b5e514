#!/bin/bash
# host-side trims: ordering tests, host overhead, small sizes
timeout 900 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_narrow.py -q -m gpu -x 2>&1 | tail -4
timeout 300 python tools/host_overhead.py 256,512,768,1024 2>&1 | tee gpurun_out/r02_host_overhead48.log
N=30 timeout 300 python tools/small_sizes.py 256,512,768,1024 dgemm0,abc1,c1 2>&1 | sed 's/(executed.*kernels/kernels/' | tee gpurun_out/r02_small48.log
