#!/bin/bash
N=10 timeout 1200 python tools/small_sizes.py 2048,2304,2560,2816,3072,3328,3584,3840,4096,4352,4608,4864,5120,5632,6144 dgemm0,abc1,c1,abc2,naive2 2>&1 | sed 's/(executed.*kernels.*mm / mm /' | sed 's/| single.*//' | tee gpurun_out/r02_mid_scan_variants.log
