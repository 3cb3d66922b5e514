"""Analyse a pipeline trace (SB_TRACE=<cta> SB_TRACE_OUT=file): per k-step
clock64 stamps: 0/1 producer issue start/end, 2 summer st_empty wait start,
3 raw_full wait start, 4 sum start, 5 sum end, 6 consumer st_full wait start,
7 consumer MMA start."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(1024, 8).astype(np.int64)
n = int((t[:, 7] > 0).sum())
t = t[:n]
t0 = t[t > 0].min()
t = np.where(t > 0, t - t0, 0)
mma_period = np.diff(t[:, 7])
print(f"steps traced {n}; median consumer period {np.median(mma_period):.0f} clk")
print(f"consumer wait for stage (7-6): median {np.median(t[1:,7]-t[1:,6]):.0f}  mean {np.mean(t[1:,7]-t[1:,6]):.0f}")
print(f"summer st_empty wait (3-2): median {np.median(t[:,3]-t[:,2]):.0f}")
print(f"summer raw_full wait (4-3): median {np.median(t[:,4]-t[:,3]):.0f}  mean {np.mean(t[:,4]-t[:,3]):.0f}")
print(f"summer sum time (5-4):      median {np.median(t[:,5]-t[:,4]):.0f}  mean {np.mean(t[:,5]-t[:,4]):.0f}")
print(f"producer issue span (1-0):  median {np.median(t[:,1]-t[:,0]):.0f}")
print(f"issue-end -> sum start (TMA latency proxy, 4-1): median {np.median(t[:,4]-t[:,1]):.0f}")
print(f"producer lead over consumer (7-0): median {np.median(t[:,7]-t[:,0]):.0f}")
for i in list(range(0, 6)) + list(range(n // 2, n // 2 + 6)):
    print(i, t[i].tolist())
