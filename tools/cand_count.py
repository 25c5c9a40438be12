import torch, sys, numpy as np
sys.path.insert(0,'.')
from paper_2605_21649_b200.workload import make_workload
# count candidates z > zmax - 1 per head for the full 1M randn workload, on the GPU with torch
dev=torch.device('cuda')
n=(1<<20); Hq,Hkv=32,8
wl=make_workload(1,n,Hq,Hkv,seed=1,device=dev)
K=wl.K[wl.page_table[0].long()].float()   # [M][Hkv][P][d]
q=wl.q[0].float()
for alpha in [1.5, 2.0, 1.25]:
    a=alpha-1
    res=[]
    for h in range(0,Hq,8):
        s=torch.einsum('mpd,d->mp', K[:, h//4], q[h]).flatten()/128**0.5
        z=a*s; zm=z.max()
        res.append(int((z>zm-1).sum()))
    print(alpha, res)
