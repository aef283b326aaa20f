import sys, json; sys.path.insert(0,'/root/repo')
import torch, bench
from paper_1604_01713_b200 import device as D
dev=torch.device("cuda",0)
_, op, rs, fact, _ = bench._setup_step(256, dev)
out={}
for timing in (False, True, False, True):
    for _ in range(3): bench._one_step(fact, op, rs)
    torch.cuda.synchronize()
    D.LaunchLog.reset(timing=timing)
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): bench._one_step(fact, op, rs)
    e1.record(); torch.cuda.synchronize()
    out.setdefault(str(timing),[]).append(round(e0.elapsed_time(e1)/20,3))
    D.LaunchLog.reset(timing=False)
print(json.dumps(out))
