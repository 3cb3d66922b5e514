set -x
timeout 1200 python -m pytest tests/test_baseline_configs.py -m gpu -x -q -s > gpurun_out/r02_baseline_tests.log 2>&1
timeout 600 python tools/fuse_probe.py > gpurun_out/r02_fuse_probe.log 2>&1
for c in 4,4 4,2 2,4 2,2 1,1; do
  STRASSEN_B200_PROFILE_ONLY_COMBO=$c timeout 300 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_combo_${c/,/} python tools/run_once.py abc 2 8192 > gpurun_out/r02_combo_${c/,/}.log 2>&1
done
