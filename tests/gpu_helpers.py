"""Shared helpers for the GPU parity tests: build a device cache through the
library (rebuild_page_stats) and an independent host cache for the oracle from
the SAME seeded workload tensors (the oracle computes its own metadata)."""
import numpy as np
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200.workload import make_workload


def device_cache(wl):
    dev = torch.device("cuda")
    c = ekv.PagedCache.allocate_meta(wl.K.to(dev), wl.V.to(dev), wl.page_table.to(dev), wl.seq_lens.to(dev))
    ekv.rebuild_page_stats(c)
    return c


def host_cache(wl, stats=True):
    hc = oracle.HostCache(wl.K.float().cpu().numpy(), wl.V.float().cpu().numpy(), wl.page_table.cpu().numpy(),
                          wl.seq_lens.cpu().numpy())
    if stats:
        hc.build_stats()
    return hc


def make_pair(B, seq_lens, Hq, Hkv, dtype=torch.bfloat16, seed=0, kind="randn", spare_tokens=0):
    wl = make_workload(B, seq_lens, Hq, Hkv, dtype=dtype, seed=seed, kind=kind, spare_tokens=spare_tokens)
    return wl, device_cache(wl), host_cache(wl)


def q_host(wl):
    return wl.q.float().cpu().numpy()


def tol_for(dtype):
    return 2e-3 if dtype == torch.bfloat16 else 1e-5
