"""Shared helpers for the GPU parity tests: build a device cache through the
library (rebuild_page_stats) and an independent host cache for the oracle from
the SAME seeded workload tensors (the oracle computes its own metadata)."""
import numpy as np
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload


def device_cache(wl, bound="kv", stat="f32"):
    dev = torch.device("cuda")
    c = ekv.PagedCache.allocate_meta(wl.K.to(dev), wl.V.to(dev), wl.page_table.to(dev), wl.seq_lens.to(dev),
                                     bound=bound, stat=stat)
    ekv.rebuild_page_stats(c)
    return c


def host_cache(wl, stats=True, bound="kv", stat="f32"):
    hc = oracle.HostCache(wl.K.float().cpu().numpy(), wl.V.float().cpu().numpy(), wl.page_table.cpu().numpy(),
                          wl.seq_lens.cpu().numpy())
    if stats:
        hc.build_stats(bound=bound, stat=stat)
    return hc


def make_pair(B, seq_lens, Hq, Hkv, dtype=torch.bfloat16, seed=0, kind="randn", spare_tokens=0, bound="kv",
              stat="f32"):
    wl = make_workload(B, seq_lens, Hq, Hkv, dtype=dtype, seed=seed, kind=kind, spare_tokens=spare_tokens)
    return wl, device_cache(wl, bound, stat), host_cache(wl, bound=bound, stat=stat)


def meta_f32(dc):
    """The device cache's stored metadata as fp32 arrays (e4m3 bounds decoded)."""
    kmin, kmax = dc.bounds_f32()
    return {"kmin": kmin.cpu().numpy(), "kmax": kmax.cpu().numpy(), "ksum": dc.ksum.cpu().numpy(),
            "ksumsq": dc.ksumsq.cpu().numpy(), "kavg": dc.kavg.float().cpu().numpy(),
            "kvar": dc.kvar.float().cpu().numpy()}


def q_host(wl):
    return wl.q.float().cpu().numpy()


def tol_for(dtype):
    return 2e-3 if dtype == torch.bfloat16 else 1e-5
