#!/bin/bash
N=20 timeout 900 python tools/small_sizes.py 2048,2176,2304,2432,2560,2688,2816,2944,3072,3328,3584,3840,4096,4352,4608,5120 dgemm0 2>&1 | sed 's/(executed.*kernels/kernels/' | sed 's/| single.*//' | tee gpurun_out/r02_mid_scan.log
