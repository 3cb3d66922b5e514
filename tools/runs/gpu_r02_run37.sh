#!/bin/bash
# re-entry baseline at HEAD: full GPU suite, smoke, bench line, reference arm, small sizes, short-k
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -8 | tee gpurun_out/r02_gputest37.log
timeout 300 python __graft_entry__.py 2>&1 | tail -8
timeout 900 python bench.py > gpurun_out/r02_bench37.json 2> gpurun_out/r02_bench37.err; tail -c 3000 gpurun_out/r02_bench37.json
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 2>&1 | tail -2 | tee gpurun_out/r02_bench37_ref.json
N=30 timeout 300 python tools/small_sizes.py 768,1024,1536,2048 dgemm0,abc1,ab1,c1 2>&1 | sed 's/(executed.*kernels/kernels/' | tee gpurun_out/r02_small37.log
