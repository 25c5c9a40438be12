import ctypes, torch, sys, math
sys.path.insert(0,'.')
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload, new_tokens
dev=torch.device('cuda')
n=(1<<20)-200; Hq,Hkv=32,8
wl=make_workload(1,n,Hq,Hkv,seed=1,device=dev,spare_tokens=200)
c=ekv.PagedCache.allocate_meta(wl.K,wl.V,wl.page_table,wl.seq_lens); ekv.rebuild_page_stats(c)
sel=ekv.select_params('topk',656); attn=ekv.attn_params(1.5); ws=ekv.alloc_workspace(c,Hq,sel)
st=ekv.DecodeStats(1,Hq,dev)
L=ekv.lib(); L.entmaxkv_debug_stamps.argtypes=[ctypes.c_void_p, ctypes.c_void_p]
buf=(ctypes.c_ulonglong*256)(); nc=ctypes.c_int()
for it in range(5):
    ekv.decode(c,wl.q,sel,attn,ws,stats=st); torch.cuda.synchronize()
L.entmaxkv_debug_stamps(buf, ctypes.byref(nc))
for k,name in [(0,'tau'),(1,'topk'),(6,'tau-solver')]:
    v=[buf[k*32+i] for i in range(8)]
    b0=buf[0*32+2] if k==6 else v[0]
    print(name, [ (v[i]-b0)/1000 if v[i] else None for i in range(8)])
print('tau ncand (block 0)', buf[14], 'newton its', buf[13], 'amb', buf[12], 'listed', buf[11])
v=[buf[2*32+i] for i in range(16)]
print('K4 producer', [ (x-v[0])/1000 if x else None for x in v[:13]])
w=[buf[3*32+i] for i in range(32)]
print('K4 consumer stage arrivals', [ (x-v[0])/1000 if x else None for x in w[:16]])
print('K4 consumer stage done    ', [ (x-v[0])/1000 if x else None for x in w[16:32]])
w=[buf[4*32+i] for i in range(32)]
print('score consumer arrivals', [ (x-w[0])/1000 if x else None for x in w[:16]])
print('score consumer done    ', [ (x-w[0])/1000 if x else None for x in w[16:32]])
v=[buf[0*32+i] for i in range(8)]; cl=[buf[0*32+16+i] for i in range(8)]
i0=0; i1=max(i for i in range(8) if v[i])
print('tau kernel SM clock MHz ~', (cl[i1]-cl[i0])/((v[i1]-v[i0])/1e3)/1e6*1e6/1e6 if v[i1]>v[i0] else None, 'cycles per phase', [cl[i]-cl[i0] for i in range(8) if v[i]])
