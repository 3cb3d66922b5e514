#!/bin/bash
# CUDA-graph capture probe; tiny-size traces; final ncu launch list + full capture of the bench's mm_kernel
timeout 300 python tools/graph_probe.py 256,512,768,1024 dgemm0,abc1,c1,abc2 2>&1 | tee gpurun_out/r02_graph_probe.log
for spec in "dgemm 0 512" "dgemm 0 640" "dgemm 0 768"; do timeout 120 python tools/cta_trace.py $spec 2>&1 | head -6; done 2>&1 | cut -c1-200 | tee gpurun_out/r02_cta_trace46.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench_final2.csv python bench.py --steps 2 --warmup 1 --no-variants --no-e2e --no-cpu --no-classical > gpurun_out/r02_ncu_bench_final2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_mm_naive2_16384_final python tools/run_once.py naive 2 16384 > gpurun_out/r02_ncu_mm_final.log 2>&1
ls -la gpurun_out/*.ncu-rep | tail -3
