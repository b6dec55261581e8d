import time, sys, torch, numpy as np
sys.path.insert(0,'.')
import paper_1703_01325_b200 as b2
n,bs,rp,ci,vals=b2.reservoir_block_grid(128,128,128,3,seed=0)
a=b2.BcsrMatrix(bs,n,n,rp,ci,vals); f=b2.build_preconditioner(a,0); op=b2.DeviceOperator(a)
bb=torch.from_numpy(b2.synthetic.ones_rhs(n,bs,rp,ci,vals)).cuda(); cfg=b2.SolverConfig(restart=30, rel_tol=1e-6)
for rep in range(5):
    torch.cuda.synchronize(); t=time.perf_counter(); _,st=b2.bicgstab(op,bb,M=f,cfg=cfg); torch.cuda.synchronize(); print(rep, round((time.perf_counter()-t)*1e3,1), st.iterations, flush=True)
rhs=torch.randn(n*bs,dtype=torch.float64,device='cuda'); out=torch.empty_like(rhs)
for _ in range(3): b2.apply_preconditioner(f,rhs,out=out)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(20): b2.apply_preconditioner(f,rhs,out=out)
torch.cuda.synchronize(); print("apply ms", (time.perf_counter()-t)/20*1e3)
for _ in range(3): op.matvec(rhs,out=out)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(20): op.matvec(rhs,out=out)
torch.cuda.synchronize(); print("spmv ms", (time.perf_counter()-t)/20*1e3)
