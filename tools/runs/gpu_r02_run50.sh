#!/bin/bash
for spec in "abc 2 32768 32768 1024" "abc 2 16384 16384 1024" "abc 2 16384 16384 512" "abc 1 16384 16384 1024" "c 2 16384 16384 1024"; do timeout 200 python tools/cta_trace_epi.py $spec 2>&1 | tail -10; done | tee gpurun_out/r02_cta_trace_epilogue.log
