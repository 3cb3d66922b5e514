timeout 600 python tools/overhead_probe.py dgemm0,abc1 1536,1024,1000,1152 16,64,256,512,1024,1536 > gpurun_out/r02_overhead.log 2>&1
STRASSEN_B200_PERSISTENT=0 timeout 300 python tools/overhead_probe.py dgemm0 1536,1024 16,256,1024 > gpurun_out/r02_overhead_nopersist.log 2>&1
STRASSEN_B200_STREAMK=0 timeout 300 python tools/overhead_probe.py dgemm0,abc1 1024 256,1024 > gpurun_out/r02_overhead_nosk.log 2>&1
