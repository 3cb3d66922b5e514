#!/bin/bash
# full GPU suite with narrow tiles planned, stress, small sizes
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -8
timeout 300 python tools/stress.py 200 7 2>&1 | tail -5
N=30 timeout 300 python tools/small_sizes.py 768,1024,1280,2048,2560 dgemm0,abc1,c1,naive1,c2,naive2 2>&1 | sed 's/(executed.*kernels/kernels/'
