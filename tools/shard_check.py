"""Multi-process check of the sequence-sharded decode through TorchComm (torchrun):
every rank decodes its striped share; rank 0 compares the replicated output with the
1-GPU decode of the whole sequence.  EKV_SAME_DEVICE=1 puts every rank on cuda:0 and uses
gloo (host-staged collectives) so that the multi-process path runs on a one-GPU box.
usage: torchrun --nproc-per-node N tools/shard_check.py [n_tokens] [k] [alpha]"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_21649_b200 import binding as ekv  # noqa: E402
from paper_2605_21649_b200 import sharding  # noqa: E402
from paper_2605_21649_b200.workload import make_workload  # noqa: E402

same = os.environ.get("EKV_SAME_DEVICE") == "1"
dist.init_process_group("gloo" if same else "nccl", init_method="env://")
rank, world = dist.get_rank(), dist.get_world_size()
local = 0 if same else int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 40000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 100
alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 1.5
Hq, Hkv = 32, 8
wl = make_workload(1, n, Hq, Hkv, seed=3, kind="planted", device=dev)
cache = sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, rank, world)
sel, attn = ekv.select_params("topk", k), ekv.attn_params(alpha)
ws = ekv.shard_workspace(cache, Hq, sel, world)
st = ekv.DecodeStats(1, Hq, dev, delta_bar=False)
if os.environ.get("EKV_PEER") == "1":        # in-kernel collectives over CUDA IPC buffers (N2)
    comm = sharding.ipc_peer_comm(ekv.peer_buffer_size(cache, Hq, sel, world))
else:
    comm = sharding.TorchComm()
out = None
for _ in range(3):
    out = ekv.decode_sharded(cache, wl.seq_lens.to(torch.int32).to(dev), wl.q.to(dev), sel, attn, comm, ws, stats=st)
torch.cuda.synchronize()
ok = True
if rank == 0:
    full = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table.to(dev), wl.seq_lens.to(dev))
    ekv.rebuild_page_stats(full)
    st1 = ekv.DecodeStats(1, Hq, dev, delta_bar=False)
    ref = ekv.decode(full, wl.q.to(dev), sel, attn, ekv.alloc_workspace(full, Hq, sel), stats=st1)
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    same_supp = bool((st.supp_count == st1.supp_count).all().item())
    dtau = (st.tau - st1.tau).abs().max().item()
    ok = err <= 2e-3 and same_supp and dtau <= 1e-6
    print(f"shard_check world={world} n={n} k={k} alpha={alpha}: max|out-out_1gpu|={err:.2e} "
          f"supports equal={same_supp} max|dtau|={dtau:.2e} -> {'OK' if ok else 'FAIL'}", flush=True)
flag = torch.tensor([0 if ok else 1])
dist.all_reduce(flag)
dist.destroy_process_group()
sys.exit(int(flag.item()))
