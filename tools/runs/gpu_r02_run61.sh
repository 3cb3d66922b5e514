#!/bin/bash
# final-build sweeps again (after the stream-K tail, fringe kernels and tile peeling)
timeout 1500 python tools/sweep.py square gpurun_out/r02f_sweep_square.csv > gpurun_out/r02f_sweep_square.log 2>&1
timeout 1500 python tools/sweep.py rankk gpurun_out/r02f_sweep_rankk.csv > gpurun_out/r02f_sweep_rankk.log 2>&1
timeout 1200 python tools/sweep.py fixedk gpurun_out/r02f_sweep_fixedk.csv > gpurun_out/r02f_sweep_fixedk.log 2>&1
tail -n 2 gpurun_out/r02f_sweep_square.log
