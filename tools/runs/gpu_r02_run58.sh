#!/bin/bash
# fringe kernels for dynamic peeling: parity suites that cover odd sizes, then odd-size timings A/B
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_baseline_configs.py tests/test_level3.py -q -m gpu -x 2>&1 | tail -4
for f in 0 1; do echo "== FRINGE=$f"; for spec in "c 2 4097 4097 4097" "naive 2 4097 4097 4097" "abc 1 4097 4097 4097" "abc 2 4097 4097 4097" "c 2 9999 9999 9999" "abc 2 9999 9999 9999" "c 1 1001 1001 1001" "abc 2 4099 4098 4097"; do STRASSEN_B200_FRINGE=$f timeout 120 python tools/shape_ab.py $spec 2>&1 | sed 's/| cublas.*| launches/|/' | cut -c1-330; done; done | tee gpurun_out/r02_fringe_ab.log
