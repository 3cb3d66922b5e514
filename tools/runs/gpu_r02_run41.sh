#!/bin/bash
# A/B in one run, alternating: previous library vs cooperative-fixup build
STRASSEN_B200_COOP=0 timeout 600 python tools/coop_check.py > gpurun_out/coop0.txt 2>&1
STRASSEN_B200_COOP=1 timeout 600 python tools/coop_check.py > gpurun_out/coop1.txt 2>&1
echo "lines: $(wc -l < gpurun_out/coop1.txt)  BAD: $(grep -c BAD gpurun_out/coop1.txt)  diff lines: $(diff gpurun_out/coop0.txt gpurun_out/coop1.txt | grep -c '^[<>]')"
for rep in 1 2; do
for lib in libstrassen_b200_prev.so libstrassen_b200.so; do
  echo "=== $lib rep $rep"
  STRASSEN_B200_LIB=$lib N=30 timeout 600 python tools/small_sizes.py 768,1024,1280 dgemm0,abc1,c1 2>&1 | grep -v cublas | sed 's/(executed.*kernels/kernels/'
done; done 2>&1 | tee gpurun_out/r02_coop_ab2.log
for rep in 1 2; do
for lib in libstrassen_b200.so libstrassen_b200_prev.so; do
  echo "== $lib rep $rep"
  STRASSEN_B200_LIB=$lib FMAX=2 REPS=3 timeout 300 python tools/fuse_probe.py naive 2 16384 16384 16384 abc 1 16384 16384 16384 2>&1 | cut -c1-110
done; done 2>&1 | tee gpurun_out/r02_coop_regress2.log
