set -x
timeout 1200 python tools/sweep.py rankk gpurun_out/r02_sweep_rankk.csv > gpurun_out/r02_sweep_rankk.log 2>&1
timeout 900 python tools/sweep.py fixedk gpurun_out/r02_sweep_fixedk.csv > gpurun_out/r02_sweep_fixedk.log 2>&1
timeout 1200 python tools/sweep.py square gpurun_out/r02_sweep_square.csv > gpurun_out/r02_sweep_square.log 2>&1
