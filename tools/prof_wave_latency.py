import sys, json; sys.path.insert(0,'/root/repo')
import numpy as np, scipy.sparse as sp, torch
from paper_1604_01713_b200 import device as D
from paper_1604_01713_b200.sparse_core import CsrMatrix
from paper_1604_01713_b200.precond import ilu0
out={}
for n in (2000, 20000):
    T=sp.diags([np.full(n-1,-1.0),np.full(n,3.0),np.full(n-1,-1.0)],[-1,0,1],format='csr')
    F=ilu0(CsrMatrix.from_scipy(T)); lu=F.device_lu()
    X=D.empty_block(n,8); X.copy_(torch.randn(n,8,device='cuda',dtype=torch.float64)); Y=D.empty_block(n,8)
    for _ in range(2): lu.solve(X,Y,upper=False)
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(); lu.solve(X,Y,upper=False); e1.record(); torch.cuda.synchronize()
    out[n]=dict(ms=e0.elapsed_time(e1), levels=lu.lower_sched.levels, us_per_level=e0.elapsed_time(e1)*1e3/lu.lower_sched.levels)
print(json.dumps(out))
