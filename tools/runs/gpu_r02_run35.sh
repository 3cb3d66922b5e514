#!/bin/bash
# narrow tiles vs wide: which (variant, level, size) gain
for nar in 0 1; do
  echo "=== NARROW=$nar"
  STRASSEN_B200_NARROW=$nar N=30 timeout 600 python tools/small_sizes.py 768,1000,1024,1280,1536,2000,2048,2560,3072 dgemm0,abc1,c1,abc2,c2 2>&1 | grep -v "^+" | sed 's/(executed.*kernels/kernels/'
done
