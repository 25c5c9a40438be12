"""GPU: sequence-sharded decode with IN-KERNEL collectives (include/entmaxkv.h
ekv_comm.peers): the ranks exchange top-k lists, z_max, the multisection partials, the power
sums and numerator / denominator by remote stores + flags inside their kernels, with no
callback and no host read.  One GPU is available, so the W ranks are virtual: W local caches,
W workspaces and W exchange buffers on the one device, each rank's step on its own stream so
that the ranks' kernels run concurrently (they wait on each other's flags).  Bars as for the
1-GPU path, against the CPU oracle's UNSHARDED decode: outputs max-abs <= 2e-3, supports
bit-exact, |tau - tau_oracle| <= 1e-6 max(1, |tau|), global |C_page| = min(k, M)."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle
from paper_2605_21649_b200 import binding as ekv
from paper_2605_21649_b200 import sharding
from gpu_helpers import host_cache, q_host
from paper_2605_21649_b200.workload import make_workload

pytestmark = pytest.mark.gpu


class Ranks:
    """W virtual ranks of one sequence-sharded cache on cuda:0 with in-kernel collectives."""

    def __init__(self, wl, world, k, alpha):
        self.wl, self.world = wl, world
        B, Hq = wl.q.shape[0], wl.q.shape[1]
        self.gl = wl.seq_lens.to(torch.int32).cuda()
        self.q = wl.q.cuda()
        self.caches = [sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, r, world) for r in range(world)]
        self.sel, self.attn = ekv.select_params("topk", k), ekv.attn_params(alpha)
        self.ws = [ekv.shard_workspace(c, Hq, self.sel, world) for c in self.caches]
        self.grp = sharding.LocalPeerGroup(world, ekv.peer_buffer_size(self.caches[0], Hq, self.sel, world))
        self.streams = [torch.cuda.Stream() for _ in range(world)]
        self.stats = [ekv.DecodeStats(B, Hq, "cuda", delta_bar=False) for _ in range(world)]
        self.outs = [torch.empty(B, Hq, 128, dtype=torch.float32, device="cuda") for _ in range(world)]
        torch.cuda.synchronize()

    def step(self):
        # every rank's whole step is enqueued before any completes: the ranks run concurrently
        for r in range(self.world):
            ekv.decode_sharded(self.caches[r], self.gl, self.q, self.sel, self.attn, self.grp.comm(r), self.ws[r],
                               out=self.outs[r], stats=self.stats[r], stream=self.streams[r])
        torch.cuda.synchronize()


def _warm(alpha, dtype=torch.bfloat16):
    # load every kernel once (world 1: no cross-stream wait) before ranks wait on each other
    wl = make_workload(1, 3000, 8, 2, seed=5, kind="planted", dtype=dtype)
    Ranks(wl, 1, 16, alpha).step()


def _check(rk, k, alpha):
    wl = rk.wl
    B, Hq = wl.q.shape[0], wl.q.shape[1]
    Hkv = wl.K.shape[1]
    G = Hq // Hkv
    hc, qh = host_cache(wl), q_host(wl)
    for b in range(B):
        M = (int(wl.seq_lens[b]) + 15) // 16
        for h in range(Hq):
            ref = oracle.decode_head(hc, qh[b, h], b, h // G, alpha, k_pages=k)
            for r in range(rk.world):
                np.testing.assert_allclose(rk.outs[r][b, h].cpu().numpy(), ref["o"], atol=2e-3, rtol=0,
                                           err_msg=f"rank {r} b={b} h={h}")
                st = rk.stats[r]
                assert int(st.supp_count[b, h]) == ref["supp"], (r, b, h)
                assert abs(float(st.tau[b, h]) - ref["tau"]) <= 1e-6 * max(1.0, abs(ref["tau"])), (r, b, h)
                assert int(st.n_sel[b, h]) == min(k, M) == len(ref["pages"])


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("alpha,k", [(1.5, 64), (2.0, 300), (1.25, 40)])
def test_peer_sharded_matches_unsharded_oracle(world, alpha, k):
    _warm(alpha)
    wl = make_workload(2, [20000, 9011], 8, 2, seed=41, kind="planted")
    rk = Ranks(wl, world, k, alpha)
    for _ in range(3):                           # the exchange counters advance across calls
        rk.step()
    _check(rk, k, alpha)
    for r in range(1, world):                    # replicated bits
        assert torch.equal(rk.outs[r], rk.outs[0]) and torch.equal(rk.stats[r].tau, rk.stats[0].tau)


def test_peer_sharded_matches_callback_mode():
    """Same step through the host-callback collectives (LoopbackGroup) and in-kernel: equal."""
    _warm(1.5)
    wl = make_workload(1, 50000, 32, 8, seed=43, kind="llama")
    rk = Ranks(wl, 4, 100, 1.5)
    rk.step()
    import test_gpu_sharded as cb
    outs, stats = cb.run_sharded(wl, 4, 100, 1.5)
    for r in range(4):
        np.testing.assert_allclose(rk.outs[r].cpu().numpy(), outs[r], atol=1e-6, rtol=0)
        assert torch.equal(rk.stats[r].supp_count.cpu(), stats[r].supp_count.cpu())
        assert torch.allclose(rk.stats[r].tau.cpu(), stats[r].tau.cpu(), atol=1e-12, rtol=0)


def test_peer_sharded_graph_capture():
    """Each rank's step captured into its own CUDA graph (no host read inside), the W graphs
    replayed concurrently: the exchange counters advance on the device, results equal eager."""
    _warm(1.5)
    world = 2
    wl = make_workload(1, 30000, 8, 2, seed=47, kind="planted")
    rk = Ranks(wl, world, 80, 1.5)
    rk.step()
    ref = [o.clone() for o in rk.outs]
    graphs = []
    for r in range(world):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=rk.streams[r]):
            ekv.decode_sharded(rk.caches[r], rk.gl, rk.q, rk.sel, rk.attn, rk.grp.comm(r), rk.ws[r], out=rk.outs[r],
                               stats=rk.stats[r], stream=rk.streams[r])
        graphs.append(g)
    torch.cuda.synchronize()
    for _ in range(3):
        for r in range(world):
            with torch.cuda.stream(rk.streams[r]):
                graphs[r].replay()
        torch.cuda.synchronize()
        for r in range(world):
            assert torch.equal(rk.outs[r], ref[r])


def test_peer_sharded_capacity_overflow_every_rank():
    """A row over 8192 candidates on one rank is marked on EVERY rank in the same exchange
    (NaN out / tau, supp -1, EKV_STATUS_CAPACITY in every rank's status word)."""
    from test_gpu_capacity import flat_workload
    _warm(1.25)
    wl = flat_workload(20000, Hq=4)
    rk = Ranks(wl, 2, 1100, 1.25)                # ~8800 candidates per rank > 8192
    rk.step()
    for r in range(2):
        assert bool((rk.stats[r].supp_count.cpu() == -1).all())
        assert bool(torch.isnan(rk.outs[r].cpu()).all())
        flags = ekv.workspace_status(rk.caches[r], 4, rk.sel, rk.ws[r])
        assert flags & ekv.EKV_STATUS_CAPACITY


def test_peer_two_processes_ipc():
    """Two processes (torchrun), one exchange buffer each, shared by CUDA IPC: the multi-process
    form of the in-kernel mode, on the one GPU (gloo only for the handle exchange)."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    env = dict(os.environ, EKV_SAME_DEVICE="1", EKV_PEER="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(root, "tools", "shard_check.py"), "40000", "100", "1.5"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "-> OK" in r.stdout
