#!/bin/bash
for sk in 0 1; do
echo "=== COOP_SK=$sk"
for spec in "dgemm 0 1024" "abc 1 1024" "dgemm 0 1280"; do STRASSEN_B200_COOP_SK=$sk timeout 120 python tools/cta_trace.py $spec 2>&1 | head -8; done
done > gpurun_out/r02_cta_trace43.log 2>&1
cat gpurun_out/r02_cta_trace43.log | cut -c1-200
