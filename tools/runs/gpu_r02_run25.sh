set -x
for rep in 1 2; do
for lib in libstrassen_b200_cd8b6d6.so libstrassen_b200.so; do
  echo "== $lib rep $rep"
  STRASSEN_B200_LIB=$lib FMAX=2 REPS=3 timeout 300 python tools/fuse_probe.py dgemm 0 16384 16384 16384 c 2 16384 16384 16384 2>&1 | cut -c1-110
done; done > gpurun_out/r02_regress_ab5.log 2>&1
timeout 300 python tools/small_sizes.py 1024,2048 abc1,naive2,abc2 > gpurun_out/r02_small25.log 2>&1
STRASSEN_B200_LIB=libstrassen_b200_cd8b6d6.so timeout 300 python tools/small_sizes.py 1024,2048 abc1,naive2,abc2 > gpurun_out/r02_small25_old.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest25.log 2>&1
