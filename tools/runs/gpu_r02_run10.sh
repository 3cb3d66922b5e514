set -x
timeout 900 python bench.py > gpurun_out/r02_bench.log 2>&1
timeout 600 python bench.py --gpus 1 --summa --dim 32768 --steps 2 --warmup 1 --no-e2e > gpurun_out/r02_bench_summa1.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-variants --no-e2e --no-cpu --no-classical > gpurun_out/r02_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mm_kernel -c 1 -f -o gpurun_out/r02_ncu_mm_naive2_16384 python tools/run_once.py naive 2 16384 > gpurun_out/r02_ncu_mm.log 2>&1
