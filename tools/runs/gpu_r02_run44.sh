#!/bin/bash
# full GPU suite + smoke + bench at the cooperative-fixup build
timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -8 | tee gpurun_out/r02_gputest44.log
timeout 300 python __graft_entry__.py 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/r02_bench44.json 2> gpurun_out/r02_bench44.err; tail -c 600 gpurun_out/r02_bench44.json
timeout 300 python tools/stress.py 150 11 2>&1 | tail -3 | tee gpurun_out/r02_stress44.log
