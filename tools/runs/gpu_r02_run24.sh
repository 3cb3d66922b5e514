for rep in 1 2; do
for lib in libstrassen_b200_cd8b6d6.so libstrassen_b200.so; do
  echo "== $lib rep $rep"
  STRASSEN_B200_LIB=$lib FMAX=2 REPS=3 timeout 300 python tools/fuse_probe.py dgemm 0 16384 16384 16384 c 2 16384 16384 16384 naive 2 16384 16384 16384 2>&1 | cut -c1-110
done; done > gpurun_out/r02_regress_ab4.log 2>&1
