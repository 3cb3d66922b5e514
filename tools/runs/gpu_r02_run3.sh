set -x
timeout 900 python -m pytest tests/test_gpu_robustness.py tests/test_gpu_parity.py tests/test_baseline_configs.py -m gpu -x -q > gpurun_out/r02_gputest3.log 2>&1
for s2 in 0 1; do STRASSEN_B200_SEP2=$s2 FMAX=2,1 REPS=3 timeout 600 python tools/fuse_probe.py abc 1 16384 16384 16384 abc 2 16384 16384 16384 abc 2 32768 32768 1024 abc 2 16384 16384 1024 abc 2 16384 16384 256 abc 1 32768 32768 1024 > gpurun_out/r02_sep2_$s2.log 2>&1; done
