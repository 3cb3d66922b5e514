#!/bin/bash
# final-build ncu --set full captures of the other 16384^3 configurations' mm_kernel
for spec in "abc 1" "abc 2" "c 2" "dgemm 0" "ab 2"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_mm_$1$2_16384_final python tools/run_once.py $1 $2 16384 > gpurun_out/r02_ncu_mm_$1$2.log 2>&1
  python tools/ncu_top.py gpurun_out/r02_ncu_mm_$1$2_16384_final.ncu-rep 2>&1 | head -60 > gpurun_out/r02_ncu_mm_kernel_$1$2_16384_final.txt
  rm -f gpurun_out/r02_ncu_mm_$1$2_16384_final.ncu-rep
done
grep -H "Duration\|dram__bytes_read.sum  \|dram__bytes_write.sum  \|dmma.avg.pct" gpurun_out/r02_ncu_mm_kernel_*_final.txt
