#!/bin/bash
for spec in "dgemm 0 1536" "dgemm 0 1792" "dgemm 0 2048" "dgemm 0 2560"; do timeout 120 python tools/cta_trace.py $spec 2>&1 | head -6; done 2>&1 | cut -c1-220 | tee gpurun_out/r02_cta_trace_mid.log
for nar in 0 1; do echo "== NARROW=$nar"; STRASSEN_B200_NARROW=$nar N=30 timeout 300 python tools/small_sizes.py 1536,1792,2048,2304,2560 dgemm0 2>&1 | grep -v cublas | sed 's/(executed.*kernels/kernels/'; done | tee gpurun_out/r02_mid_narrow_ab.log
