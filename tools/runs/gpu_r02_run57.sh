#!/bin/bash
# final build: the N > 1 bench path on one GPU (1 x 1 grid), Python schedule and native entry point
timeout 1200 python bench.py --gpus 1 --summa --dim 32768 --steps 2 --warmup 1 > gpurun_out/r02_bench_summa1x1_32768_final.json 2> gpurun_out/r02_bench_summa_final.err; tail -c 700 gpurun_out/r02_bench_summa1x1_32768_final.json; echo
timeout 1200 python bench.py --gpus 1 --summa --native --dim 32768 --steps 2 --warmup 1 > gpurun_out/r02_bench_summa1x1_32768_native_final.json 2> gpurun_out/r02_bench_summa_native_final.err; tail -c 700 gpurun_out/r02_bench_summa1x1_32768_native_final.json; echo
