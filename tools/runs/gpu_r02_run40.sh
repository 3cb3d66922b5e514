#!/bin/bash
# cooperative fixup: bitwise equality with the single-owner fixup, then A/B timings
STRASSEN_B200_COOP=0 timeout 600 python tools/coop_check.py > gpurun_out/coop0.txt 2>&1
STRASSEN_B200_COOP=1 timeout 600 python tools/coop_check.py > gpurun_out/coop1.txt 2>&1
echo "lines: $(wc -l < gpurun_out/coop1.txt)  BAD: $(grep -c BAD gpurun_out/coop1.txt)  diff lines: $(diff gpurun_out/coop0.txt gpurun_out/coop1.txt | grep -c '^[<>]')"
diff gpurun_out/coop0.txt gpurun_out/coop1.txt | head -10
tail -3 gpurun_out/coop1.txt
for coop in 0 1; do
  echo "=== COOP=$coop"
  STRASSEN_B200_COOP=$coop N=30 timeout 600 python tools/small_sizes.py 768,1024,1280,1536,2048 dgemm0,abc1,c1,naive1 2>&1 | sed 's/(executed.*kernels/kernels/'
done 2>&1 | tee gpurun_out/r02_coop_ab.log
for lib in libstrassen_b200_prev.so libstrassen_b200.so; do
  echo "== $lib"
  STRASSEN_B200_LIB=$lib FMAX=2 REPS=3 timeout 300 python tools/fuse_probe.py naive 2 16384 16384 16384 abc 1 16384 16384 16384 dgemm 0 16384 16384 16384 abc 2 16384 16384 1024 2>&1 | cut -c1-110
done 2>&1 | tee gpurun_out/r02_coop_regress.log
