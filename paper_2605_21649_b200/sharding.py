"""Sequence sharding plumbing: page striping of a cache over ranks and the
communicator adapters the library calls back for its collectives (include/entmaxkv.h,
ekv_comm).  Argument marshalling and data movement only -- every step of the decode runs in
the library's kernels; the collectives are torch.distributed's (NCCL on GPUs).

Striping: rank r of W holds the global pages p = r + i W as local pages i = 0, 1, ...  Only
the global last page can be partial, and it is its owner's last local page, so each rank's
pages form an ordinary cache of L_r tokens.
"""
from __future__ import annotations

import threading

import torch

from . import binding as ekv

_DT = {0: torch.float32, 1: torch.float64}


def local_pages(n_tokens: int, rank: int, world: int, P: int = 16):
    """Global page ids owned by `rank` (ascending) and the local token count L_r."""
    M = (n_tokens + P - 1) // P
    pages = list(range(rank, M, world))
    L = sum(min(P, n_tokens - p * P) for p in pages)
    return pages, L


def shard_cache(K, V, page_table, seq_lens, rank: int, world: int, spare_pages: int = 0, bound="kv", stat="f32"):
    """Rank `rank`'s local cache of a global paged cache (K/V [n_phys][Hkv][P][d], page_table
    [B][maxp], seq_lens [B]; host or device tensors): its pages gathered into a local pool
    (local page i -> local physical page), metadata rebuilt by the library on the device."""
    B = page_table.shape[0]
    P = K.shape[2]
    dev = torch.device("cuda", torch.cuda.current_device()) if not K.is_cuda else K.device
    lens = [int(x) for x in seq_lens.tolist()]
    per_b = [local_pages(L, rank, world, P) for L in lens]
    mloc = max(1, max(len(p) for p, _ in per_b) + spare_pages)
    phys = []
    table = torch.zeros(B, mloc, dtype=torch.int32)
    for b, (pages, _) in enumerate(per_b):
        gp = page_table[b, pages].long().cpu() if pages else torch.zeros(0, dtype=torch.long)
        base = len(phys)
        phys.extend(gp.tolist())
        table[b, :len(pages)] = torch.arange(base, base + len(pages), dtype=torch.int32)
        # spare local pages for appends map to fresh zero pages
        for i in range(len(pages), mloc):
            table[b, i] = -1
    idx = torch.tensor(phys if phys else [0], dtype=torch.long)
    Kl = K[idx.to(K.device)].to(dev).contiguous()
    Vl = V[idx.to(V.device)].to(dev).contiguous()
    n_used = Kl.shape[0]
    extra = int((table < 0).sum())
    if extra:
        z = torch.zeros((extra,) + tuple(Kl.shape[1:]), dtype=Kl.dtype, device=dev)
        Kl, Vl = torch.cat([Kl, z]), torch.cat([Vl, z.clone()])
        table[table < 0] = torch.arange(n_used, n_used + extra, dtype=torch.int32)
    cache = ekv.PagedCache.allocate_meta(Kl, Vl, table.to(dev), torch.tensor([L for _, L in per_b], dtype=torch.int32,
                                                                             device=dev), bound=bound, stat=stat)
    ekv.rebuild_page_stats(cache)
    return cache


class _CommBase:
    """Maps the workspace pointers the library passes back to views of the workspace tensor."""

    def __init__(self, rank: int, world: int):
        self.rank, self.world = rank, world
        self.ws = None
        self.stream = None
        self.error = None
        self.c_allreduce = ekv.ALLREDUCE_FN(self._allreduce)
        self.c_allgather = ekv.ALLGATHER_FN(self._allgather)

    def bind(self, ws, stream):
        self.ws, self.stream, self.error = ws, stream, None

    def unbind(self):
        self.ws = None

    def _view(self, ptr, nbytes, dtype=torch.uint8):
        off = int(ptr) - self.ws.data_ptr()
        if off < 0 or off + nbytes > self.ws.numel():
            raise ValueError("collective buffer outside the bound workspace")
        return self.ws[off:off + nbytes].view(dtype)

    def _allreduce(self, buf, count, dtype, op, user, stream):
        try:
            dt = _DT[int(dtype)]
            t = self._view(buf, int(count) * torch.tensor([], dtype=dt).element_size(), dt)
            self.all_reduce(t, int(op))
            return 0
        except Exception as e:  # reported after the call returns
            self.error = e
            return 1

    def _allgather(self, send, recv, nbytes, user, stream):
        try:
            nb = int(nbytes)
            self.all_gather(self._view(send, nb), self._view(recv, nb * self.world))
            return 0
        except Exception as e:
            self.error = e
            return 1


class TorchComm(_CommBase):
    """Collectives through torch.distributed (NCCL for CUDA tensors), on the call's stream."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        super().__init__(dist.get_rank(group), dist.get_world_size(group))

    def _host_staged(self):
        # gloo (tests: several ranks sharing one GPU) has no device all-gather: stage on the host
        return self.dist.get_backend(self.group) == "gloo"

    def all_reduce(self, t, op):
        d = self.dist
        rop = d.ReduceOp.MAX if op == 1 else d.ReduceOp.SUM
        if self._host_staged():
            self.stream.synchronize()
            h = t.cpu()
            d.all_reduce(h, op=rop, group=self.group)
            t.copy_(h)
            torch.cuda.synchronize()
            return
        with torch.cuda.stream(self.stream):
            d.all_reduce(t, op=rop, group=self.group)

    def all_gather(self, send, recv):
        if self._host_staged():
            self.stream.synchronize()
            parts = [torch.empty_like(send, device="cpu") for _ in range(self.world)]
            self.dist.all_gather(parts, send.cpu(), group=self.group)
            recv.copy_(torch.cat(parts))
            torch.cuda.synchronize()
            return
        with torch.cuda.stream(self.stream):
            self.dist.all_gather_into_tensor(recv, send, group=self.group)


class LoopbackGroup:
    """W virtual ranks in one process (one thread each, e.g. on one GPU): the collectives
    rendezvous on a barrier and reduce the ranks' buffers with torch ops.  For tests of the
    sharded protocol where only one device is available."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world

    def comm(self, rank: int):
        return LoopbackComm(self, rank)


class LoopbackComm(_CommBase):
    def __init__(self, group: LoopbackGroup, rank: int):
        self.g = group
        super().__init__(rank, group.world)

    def _exchange(self, t):
        self.stream.synchronize()
        self.g.slots[self.rank] = t
        self.g.barrier.wait()
        vals = [x.clone() for x in self.g.slots]
        self.g.barrier.wait()
        return vals

    def all_reduce(self, t, op):
        vals = self._exchange(t)
        r = vals[0]
        for v in vals[1:]:
            r = torch.maximum(r, v) if op == 1 else r + v
        t.copy_(r)
        torch.cuda.synchronize()

    def all_gather(self, send, recv):
        vals = self._exchange(send)
        recv.copy_(torch.cat(vals))
        torch.cuda.synchronize()


# ----------------------------------------------------------------------------- in-kernel collectives (N2)
class PeerComm(_CommBase):
    """Rank `rank` of an in-kernel collective group: `peers` = every rank's exchange buffer
    (device pointers as mapped in this process).  The library exchanges its partials inside
    its kernels (include/entmaxkv.h, ekv_comm.peers); no callback is ever made."""

    def __init__(self, rank: int, world: int, peers, keep=None):
        super().__init__(rank, world)
        self.peers = [int(p) for p in peers]
        self._keep = keep          # keeps the buffers (and any IPC mappings) alive

    def all_reduce(self, t, op):   # pragma: no cover - never called in peer mode
        raise RuntimeError("in-kernel collective mode makes no callbacks")

    all_gather = all_reduce


class LocalPeerGroup:
    """W virtual ranks sharing one GPU (tests): the W exchange buffers are plain zeroed device
    buffers of this process; each rank's step must run on its own stream so that the ranks'
    kernels run concurrently."""

    def __init__(self, world: int, nbytes: int, device=None):
        self.world = world
        self.bufs = [torch.zeros(int(nbytes), dtype=torch.uint8, device=device or "cuda") for _ in range(world)]

    def comm(self, rank: int) -> PeerComm:
        return PeerComm(rank, self.world, [b.data_ptr() for b in self.bufs], keep=self.bufs)

    def reset(self):
        for b in self.bufs:
            b.zero_()


def ipc_peer_comm(nbytes: int, group=None) -> PeerComm:
    """One rank per process (one GPU each, or several sharing a GPU): allocate this rank's
    zeroed exchange buffer, share its CUDA IPC handle through torch.distributed (any backend)
    and open every peer's buffer in this process (peer access over NVLink / NVSwitch is
    enabled by the IPC mapping).  Collective over `group`."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buf = torch.zeros(int(nbytes), dtype=torch.uint8, device="cuda")
    torch.cuda.synchronize()
    handle = buf.untyped_storage()._share_cuda_()
    off = int(handle[3])
    handles = [None] * world
    dist.all_gather_object(handles, (handle, off, buf.data_ptr() - buf.untyped_storage().data_ptr()), group=group)
    keep, peers = [buf], []
    for r, (h, off_r, view_off) in enumerate(handles):
        if r == rank:
            peers.append(buf.data_ptr())
            continue
        st = torch.UntypedStorage._new_shared_cuda(*h)
        keep.append(st)
        peers.append(st.data_ptr() + view_off)
    dist.barrier(group=group)
    return PeerComm(rank, world, peers, keep=keep)
