import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2311_14206_b200 as sk
from tools.c4_problem import c4_complex_csr
ctx = sk.default_context()
dims=(32,32,32,64); N=int(np.prod(dims))
off,col,val=c4_complex_csr(dims,-0.8,2,sk.uniform_stream)
A=sk.SparseMatrix.from_complex(N,N,off,col,val)
b=sk.gaussian_vector(2*N,4)
cfg=sk.SolverConfig(m=80,k=20,t=3,s=200,tol=1e-8)
S=sk.SketchOperator.subsampled_dct(2*N,200,cfg.sketch_seed)
import torch
bd=torch.from_numpy(b).cuda()
for i in range(3):
    r=sk.solve(A,bd,cfg,sketch=S)
ctx.synchronize()
ctx.set_timing(True); ctx.timing_reset()
t=time.perf_counter(); r=sk.solve(A,bd,cfg,sketch=S); ctx.synchronize(); dt=time.perf_counter()-t
print("wall ms", dt*1e3, r.report.iterations, {k:round(v,2) for k,v in r.report.phases.items()})
names=("spmv_arnoldi","update","sketch","update_sketch","sketch_fold","tallskinny","recycle_gemm","col_norms","correction","residual","copy_norm","axpy","fold_partials")
for nm in names:
    c,ms=ctx.timing(nm)
    if c: print(nm,c,round(ms,3))
