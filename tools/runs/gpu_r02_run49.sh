#!/bin/bash
# local-update rates at BASELINE config 5's per-rank panel shapes (SUMMA projection inputs)
FMAX=2 REPS=2 timeout 900 python tools/fuse_probe.py abc 2 65536 32768 8192 abc 2 32768 32768 8192 abc 2 32768 16384 8192 abc 2 46336 23168 8192 abc 2 32768 32768 4096 abc 2 32768 16384 4096 c 2 32768 16384 8192 naive 2 32768 16384 8192 2>&1 | cut -c1-160 | tee gpurun_out/r02_cfg5_local_shapes.log
