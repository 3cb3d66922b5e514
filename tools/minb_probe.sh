# level-2 register stream pass: launch-bound min-blocks 4 (current build) vs 1
run() { for sz in 1024 2048 3072 8192 16384; do for vl in "naive 2" "abc 2"; do
  echo "$1 $sz $vl $(PROFILE=1 python tools/run_once.py $vl $sz | grep totals)"; done; done; }
run MINB4
touch paper_1605_01078_b200/csrc/kernels.cu
make -C paper_1605_01078_b200/csrc NVCC="/usr/local/cuda/bin/nvcc -DSTREAM_FIXED_MINB2=1" > /dev/null 2>&1 || echo build-failed
run MINB1
