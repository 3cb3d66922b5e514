import sys, time, numpy as np, torch
sys.path.insert(0,'.')
import paper_1605_01078_b200 as S
m=n=k=8200
a=torch.rand(k,m,dtype=torch.float64).pin_memory().numpy().T
b=torch.rand(n,k,dtype=torch.float64).pin_memory().numpy().T
c=torch.rand(n,m,dtype=torch.float64).pin_memory().numpy().T
ctx=S.Ctx()
for _ in range(2): ctx.gemm("naive",2,1.0,a,b,c)
t0=time.perf_counter()
for _ in range(3): ctx.gemm("naive",2,1.0,a,b,c)
t=(time.perf_counter()-t0)/3
print("host naive2 8200^3: %.1f ms  %.1f TF/s  launches %d"%(t*1e3, 2*m*n*k/t/1e12, ctx.last_launches()))
