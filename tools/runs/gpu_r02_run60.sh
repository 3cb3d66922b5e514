#!/bin/bash
# peeling to whole quadrant tiles (remainder <= 8): A/B, then the full GPU suite
for p in 0 1; do echo "== TILE_PEEL=$p"; for spec in "dgemm 0 4097 4097 4097" "dgemm 0 4100 4100 4100" "c 2 4100 4100 4100" "abc 2 4104 4100 4099" "abc 1 4100 4100 4100" "naive 2 8200 8200 8200" "dgemm 0 2052 2052 2052" "c 2 2052 2052 2052" "dgemm 0 1028 1028 1028"; do STRASSEN_B200_TILE_PEEL=$p timeout 120 python tools/shape_ab.py $spec 2>&1 | sed 's/| cublas.*| launches/|/' | cut -c1-250; done; done | tee gpurun_out/r02_tile_peel_ab.log
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
