for lib in libstrassen_b200_prev.so libstrassen_b200.so; do
  echo "== $lib"
  STRASSEN_B200_LIB=$lib FMAX=2 REPS=3 timeout 300 python tools/fuse_probe.py naive 2 16384 16384 16384 c 2 16384 16384 16384 dgemm 0 16384 16384 16384 2>&1 | cut -c1-110
  STRASSEN_B200_LIB=$lib timeout 300 python tools/small_sizes.py 1024,1536,2048 dgemm0,abc1,naive1 2>&1 | cut -c1-110
done > gpurun_out/r02_fixup0_ab.log 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_gputest30.log 2>&1
