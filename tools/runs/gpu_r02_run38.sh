#!/bin/bash
# CTA traces at HEAD for the small sizes (narrow tiles, fixup by piece 0)
for spec in "dgemm 0 1024" "abc 1 1024" "c 1 1024" "naive 1 1024" "dgemm 0 768" "abc 1 768"; do timeout 120 python tools/cta_trace.py $spec 2>&1 | head -8; done > gpurun_out/r02_cta_trace38.log 2>&1
cat gpurun_out/r02_cta_trace38.log | cut -c1-300
