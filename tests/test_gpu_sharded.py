"""GPU: sequence-sharded decode (include/entmaxkv.h entmaxkv_decode_sharded)
against the CPU oracle's UNSHARDED decode of the same sequence.  One GPU is available, so the
W ranks are virtual: one thread per rank, each with its own striped local cache and stream;
the collectives rendezvous in-process (sharding.LoopbackGroup).  Bars as for the 1-GPU path:
global page sets identical (checked via |C_page| and the exact outputs), supports bit-exact,
outputs max-abs <= 2e-3 (bf16), |tau - tau_oracle| <= 1e-6 max(1, |tau|)."""
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200 import sharding
from gpu_helpers import host_cache, q_host
from paper_2605_21649_b200.workload import make_workload

pytestmark = pytest.mark.gpu


def run_sharded(wl, world, k, alpha):
    B, Hq = wl.q.shape[0], wl.q.shape[1]
    grp = sharding.LoopbackGroup(world)
    outs, stats, errs = [None] * world, [None] * world, []
    gl = wl.seq_lens.to(torch.int32).cuda()
    caches = [sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, r, world) for r in range(world)]
    torch.cuda.synchronize()
    sel = ekv.select_params("topk", k)
    attn = ekv.attn_params(alpha)

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            ws = ekv.shard_workspace(caches[r], Hq, sel, world)
            st = ekv.DecodeStats(B, Hq, "cuda", delta_bar=False)
            with torch.cuda.stream(s):
                o = ekv.decode_sharded(caches[r], gl, wl.q.cuda(), sel, attn, grp.comm(r), ws, stats=st, stream=s)
            s.synchronize()
            outs[r], stats[r] = o.cpu().numpy(), st
        except Exception as e:  # pragma: no cover
            errs.append(e)
            grp.barrier.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return outs, stats


@pytest.mark.parametrize("world", [1, 2, 4])
@pytest.mark.parametrize("alpha,k", [(1.5, 64), (2.0, 300), (1.25, 40)])
def test_sharded_matches_unsharded_oracle(world, alpha, k):
    B, Hq, Hkv = 2, 8, 2
    wl = make_workload(B, [20000, 9011], Hq, Hkv, seed=41, kind="planted")
    outs, stats = run_sharded(wl, world, k, alpha)
    hc = host_cache(wl)
    qh = q_host(wl)
    G = Hq // Hkv
    for b in range(B):
        M = (int(wl.seq_lens[b]) + 15) // 16
        for h in range(Hq):
            ref = oracle.decode_head(hc, qh[b, h], b, h // G, alpha, k_pages=k)
            for r in range(world):                  # replicated output on every rank
                np.testing.assert_allclose(outs[r][b, h], ref["o"], atol=2e-3, rtol=0,
                                           err_msg=f"rank {r} b={b} h={h}")
                st = stats[r]
                assert int(st.supp_count[b, h]) == ref["supp"], (r, b, h)
                assert abs(float(st.tau[b, h]) - ref["tau"]) <= 1e-6 * max(1.0, abs(ref["tau"])), (r, b, h)
                assert int(st.n_sel[b, h]) == min(k, M) == len(ref["pages"])


def test_sharded_rejects_non_integer_beta():
    wl = make_workload(1, 4000, 4, 1, seed=1, kind="randn")
    c = sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, 0, 1)
    sel = ekv.select_params("topk", 8)
    ws = ekv.shard_workspace(c, 4, sel, 1)
    with pytest.raises(ekv.EkvError) as ei:
        ekv.decode_sharded(c, wl.seq_lens.to(torch.int32).cuda(), wl.q.cuda(), sel, ekv.attn_params(1.7),
                           sharding.LoopbackGroup(1).comm(0), ws)
    assert ei.value.status == ekv.EKV_ERR_UNSUPPORTED


def test_torchcomm_two_processes_share_one_gpu():
    """The multi-process path (torchrun, TorchComm callbacks, one process per rank) on the
    one available GPU: gloo with host-staged collectives, compared with the 1-GPU decode."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, EKV_SAME_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tools", "shard_check.py"), "40000", "100", "1.5"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "-> OK" in r.stdout
