#!/bin/bash
# narrow tiles: correctness first, then small-size A/B
set -x
timeout 900 python -m pytest tests -x -q -m gpu -k "robust or small or baseline_configs or fused or stream or split" 2>&1 | tail -15
for nar in 0 1; do
  echo "=== NARROW=$nar"
  STRASSEN_B200_NARROW=$nar timeout 300 python tools/small_sizes.py 1024,1536,2048 dgemm0,abc1,ab1,naive1,c1,abc2,naive2,c2 2>&1 | tail -30
done
