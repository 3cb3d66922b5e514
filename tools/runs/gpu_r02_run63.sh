#!/bin/bash
# fringe width 16: A/B at sizes 9..16 above whole tiles, then the parity suites
for p in 0 1; do echo "== TILE_PEEL=$p"; for spec in "c 2 4108 4108 4108" "naive 2 8208 8208 8208" "abc 2 4112 4106 4100" "dgemm 0 4112 4112 4112" "c 1 6160 6160 6160" "c 2 4100 4100 4100"; do STRASSEN_B200_TILE_PEEL=$p timeout 120 python tools/shape_ab.py $spec 2>&1 | sed 's/| cublas.*| launches/|/' | cut -c1-260; done; done | tee gpurun_out/r02_tile_peel16_ab.log
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
