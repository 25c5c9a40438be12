"""CPU, world size 2 (gloo): the sequence-sharding protocol of entmaxkv_decode_sharded
(include/entmaxkv.h) executed with real torch.distributed collectives, every
rank's local quantities computed by the CPU oracle from its striped pages only.  Pins the
protocol itself -- striping, the all-gather merge of local top-k lists with R3's tie-break,
the max all-reduce of z_max, the multisection rounds on F(x) = sum (z - x)_+^beta with the
"no z strictly inside the bracket" stop, the power-sum closed form for tau and the
numerator/denominator all-reduce -- against the oracle's UNSHARDED decode:
identical global page sets, identical supports, tau and outputs to fp64 rounding."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2605_21649_b200.sharding import local_pages
from paper_2605_21649_b200.workload import make_workload

T_PROBES = 62            # interior probes per round (kernels_shard.cuh kShT)
NP = T_PROBES + 2


def probe_x(lo, hi, t):
    if t == 0:
        return lo
    if t == NP - 1:
        return hi
    return lo + (hi - lo) * (t / (NP - 1))


def sharded_head(hc, q, b, kvh, alpha, k, rank, world):
    """One query head through the protocol; returns (global pages, tau, supp, out)."""
    a = alpha - 1.0
    beta = 1.0 / a
    ib = int(round(beta))
    L = int(hc.seq_lens[b])
    mine, _ = local_pages(L, rank, world)
    box_all, _, _ = hc.score_pages(q, b, kvh, modes=1)        # per-page values need only the page
    lbox = box_all[mine]
    # 1. local top-k -> all-gather (score, global page) -> merge, tie-break lower global page
    lsel = oracle.topk(lbox, k) if len(mine) else np.zeros(0, np.int32)
    send = np.full((k, 2), [-np.inf, -1.0])
    for i, lp in enumerate(lsel):
        send[i] = [lbox[lp], mine[lp]]
    recv = [torch.zeros(k, 2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(recv, torch.from_numpy(send))
    cand = [(float(s), int(g)) for r_ in recv for s, g in r_.numpy() if g >= 0]
    cand.sort(key=lambda x: (-np.float32(x[0]), x[1]))
    gsel = sorted(g for _, g in cand[:min(k, len(cand))])
    my_sel = [g for g in gsel if g % world == rank]
    # 2. local token scores of the share (the oracle's canonical score), max all-reduce
    att = hc.attend(q, b, kvh, np.arange(hc.n_pages(b), dtype=np.int32), alpha, want_s=True)
    s_all = att["s"]
    toks = [j for g in my_sel for j in range(g * hc.P, min((g + 1) * hc.P, L))]
    z = np.array([a * float(s_all[j]) for j in toks], np.float64)
    zl = np.array([z.max() if z.size else -np.inf])
    zt = torch.from_numpy(zl)
    dist.all_reduce(zt, op=dist.ReduceOp.MAX)
    zmax = float(zt[0])
    lo, hi = zmax - 1.0 - 1e-12 * max(1.0, abs(zmax)), zmax
    zc = z[z > lo]
    # 3. multisection rounds
    for _ in range(14):
        part = np.zeros((NP, 3))
        for t in range(NP):
            x = probe_x(lo, hi, t)
            d = zc - x
            part[t] = [np.sum(d[d > 0] ** ib), np.sum(d > 0), np.sum(d >= 0)]
        pt = torch.from_numpy(part)
        dist.all_reduce(pt)
        part = pt.numpy()
        t1 = max(t for t in range(NP) if part[t, 0] >= 1.0)
        t2 = min(t1 + 1, NP - 1)
        lo, hi, cgt, cge = probe_x(lo, hi, t1), probe_x(lo, hi, t2), part[t1, 1], part[t2, 2]
        if cgt == cge:
            break
    else:
        raise AssertionError("multisection did not converge")
    # 4. power sums at lo -> tau
    w = zc[zc > lo] - lo
    S = torch.from_numpy(np.array([np.sum(w ** m) for m in range(5)]))
    dist.all_reduce(S)
    S = S.numpy()
    if ib == 1:
        delta = (S[1] - 1.0) / S[0]
    else:
        delta = (S[1] - np.sqrt(max(0.0, S[1] ** 2 - S[0] * (S[2] - 1.0)))) / S[0]
    tau = lo + delta
    # 5. numerator / denominator
    num = np.zeros(hc.dv + 1)
    row = hc.page_table[b]
    for j, zj in zip(toks, z):
        if zj > lo:
            p = (zj - tau) ** ib
            num[:hc.dv] += p * hc.V[row[j // hc.P], kvh, j % hc.P].astype(np.float64)
            num[hc.dv] += p
    nt = torch.from_numpy(num)
    dist.all_reduce(nt)
    nt = nt.numpy()
    return gsel, tau, int(S[0]), nt[:hc.dv] / nt[hc.dv]


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = make_workload(1, 5000, 4, 1, dtype=torch.float32, seed=5, kind="planted")
        hc = oracle.HostCache(wl.K.numpy(), wl.V.numpy(), wl.page_table.numpy(), wl.seq_lens.numpy())
        hc.build_stats()
        q = wl.q.numpy()
        out = []
        for alpha, k in ((1.5, 20), (2.0, 7), (1.5, 313)):
            for h in range(4):
                gsel, tau, supp, o = sharded_head(hc, q[0, h], 0, 0, alpha, k, rank, world)
                ref = oracle.decode_head(hc, q[0, h], 0, 0, alpha, k_pages=k)
                out.append((gsel == ref["pages"].tolist(), supp == ref["supp"],
                            abs(tau - ref["tau"]) <= 1e-9 * max(1.0, abs(ref["tau"])),
                            float(np.max(np.abs(o - ref["o"])))))
        results[rank] = out
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_local_pages_striping():
    for n in (1, 15, 16, 17, 5000, 4096):
        for world in (1, 2, 3, 4, 8):
            seen, tot = [], 0
            for r in range(world):
                pages, L = local_pages(n, r, world)
                assert pages == sorted(pages) and all(p % world == r for p in pages)
                # only the global last page may be partial, and it is its owner's last page
                M = (n + 15) // 16
                if M - 1 in pages:
                    assert pages[-1] == M - 1
                seen += pages
                tot += L
            assert sorted(seen) == list(range((n + 15) // 16)) and tot == n


def test_sharded_protocol_world2_gloo():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    for r in range(world):
        for same_pages, same_supp, tau_ok, err in results[r]:
            assert same_pages and same_supp and tau_ok
            assert err <= 1e-9
