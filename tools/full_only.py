import torch, sys, time
sys.path.insert(0,'.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload
dev=torch.device('cuda')
n=(1<<20); Hq,Hkv=32,8
alpha=float(sys.argv[1]) if len(sys.argv)>1 else 1.5
wl=make_workload(1,n,Hq,Hkv,seed=1,device=dev)
c=ekv.PagedCache.allocate_meta(wl.K,wl.V,wl.page_table,wl.seq_lens); ekv.rebuild_page_stats(c)
ws=ekv.alloc_workspace(c,Hq,None)
for i in range(3):
    o,t,s=ekv.full_attend(c,wl.q,ekv.attn_params(alpha),workspace=ws)
torch.cuda.synchronize()
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(5): ekv.full_attend(c,wl.q,ekv.attn_params(alpha),workspace=ws)
e1.record(); torch.cuda.synchronize()
print('full us', e0.elapsed_time(e1)*1e3/5, 'supp', s.tolist()[0][:8])
