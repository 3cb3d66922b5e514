#!/bin/bash
# narrow tiles where a quadrant ends in at most half a tile: scan + full suite
N=10 timeout 1200 python tools/small_sizes.py 2304,2816,3328,3840,4352,4864,5376,5888,6400,6912,7424 c1,c2,naive2 2>&1 | grep -v cublas | sed 's/(executed.*kernels.*mm / mm /' | sed 's/| single.*//' | tee gpurun_out/r02_narrow_half_edge.log
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
