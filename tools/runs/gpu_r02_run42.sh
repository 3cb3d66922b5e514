#!/bin/bash
# k-chunk grids with the cooperative fixup vs stream-K (single-owner) for small DGEMM
STRASSEN_B200_COOP=0 timeout 600 python tools/coop_check.py > gpurun_out/coop0.txt 2>&1
STRASSEN_B200_COOP=1 timeout 600 python tools/coop_check.py > gpurun_out/coop1.txt 2>&1
echo "lines: $(wc -l < gpurun_out/coop1.txt)  BAD: $(grep -c BAD gpurun_out/coop1.txt)  diff lines: $(diff gpurun_out/coop0.txt gpurun_out/coop1.txt | grep -c '^[<>]')"
for sk in 1 0; do
  echo "=== STREAMK=$sk"
  STRASSEN_B200_STREAMK=$sk N=30 timeout 600 python tools/small_sizes.py 512,640,768,896,1000,1024,1152,1280,1536,1792,2048 dgemm0 2>&1 | sed 's/(executed.*kernels/kernels/'
done 2>&1 | tee gpurun_out/r02_coop_kchunk.log
