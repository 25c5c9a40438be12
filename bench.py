#!/usr/bin/env python
"""Benchmark of the EntmaxKV sparse decode step on B200.

Default workload (BASELINE.json configs[3], the 1M-context config the metric is quoted on;
it fits one GPU): one 1,048,576-token sequence, Llama-3.1-8B attention shape (32 q / 8 KV
heads, d = 128), bf16, page 16, alpha = 1.5, top-k 1 % of the pages (k = 656), on the
north star's synthetic Llama-shaped cache with planted heavy-hitter keys (DESIGN.md
"Input recipe"; `--workload randn` = the paper's efficiency workload).

One step = append the new token's k/v (a0) + page scoring (a1) + top-k selection (a2) +
exact sparse alpha-entmax attention (a3) + the certified delta_bar (a4), replayed from a
CUDA graph.  Inputs are larger than L2 (K/V 4 GiB, metadata 1.5 GiB): no flush needed.

Beside the headline the JSON line carries: the dominant kernel's roofline, the step-level
HBM fraction, the full-cache entmax baselines (a5) on the same cache, the selection quality
(exact delta and support recall rho vs full-cache entmax, eval mode), a budget sweep, the
Gaussian selector on the same cache, the e2e public-API time (graph and eager), the CPU
oracle on the same cache (threaded over the host cores; also its max-abs vs the GPU output
of the timed state), clocks.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run (N ranks, one
per GPU).  N > 1: configs[3]'s multi-GPU form, ONE 1M sequence sequence-sharded over the N
GPUs (strong scaling; time = max over ranks); the batch-sharded weak-scaling line beside it.
"""
import argparse
import concurrent.futures as cf
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs per decode step (sparse vs full entmax) at 128K–1M ctx; HBM GB/s vs peak"
NOMINAL_HBM_GBS = 8000.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--budget", type=float, default=0.01)
    ap.add_argument("--alpha", type=float, default=1.5)
    ap.add_argument("--policy", default="topk", choices=["topk", "gauss"])
    ap.add_argument("--workload", default="llama", choices=["llama", "planted", "randn"])
    ap.add_argument("--bounds", default="kv", choices=["kv", "e4m3"],
                    help="stored page bounds: KV dtype (exact) or outward-rounded fp8 e4m3 (N3, R24)")
    ap.add_argument("--stats", default="f32", choices=["f32", "bf16"], help="stored kavg/kvar dtype")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="headline + roofline only (profiling runs)")
    argv = json.loads(os.environ["EKV_BENCH_ARGV"]) if "EKV_BENCH_ARGV" in os.environ else None
    return ap.parse_args(argv)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def ncu_traffic(kernel_prefix):
    """dram__bytes_read.sum + dram__bytes_write.sum (bytes) of one launch of the kernel, from the
    newest committed ncu --set full capture summary (profiles/r*_ncu_full_top_kernels.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_top_kernels.json")))
    if not files:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    try:
        for k in json.load(open(files[-1])):
            if k["Kernel Name"][0].split("(")[0].replace("void ", "").startswith(kernel_prefix):
                rd, wr = k["dram__bytes_read.sum"], k["dram__bytes_write.sum"]
                return float(rd[0]) * scale[rd[1]] + float(wr[0]) * scale[wr[1]]
    except Exception:
        return None
    return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = max(mx, float(r[1]))
                for n, v in zip(names, r[2:6]):
                    if v.lower() == "active":
                        reasons.add(n)
            except Exception:
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
HQ, HKV, D, P = 32, 8, 128, 16


def workload_for(args, rank, device, n_tokens=None, spare=0):
    from paper_2605_21649_b200.workload import make_workload
    n = args.n if n_tokens is None else n_tokens
    return make_workload(1, n, HQ, HKV, seed=1000 + rank, device=device, kind=args.workload, spare_tokens=spare)


def k_pages_for(args):
    return max(1, math.ceil(args.budget * ((args.n + P - 1) // P)))


# ----------------------------------------------------------------------------- CPU oracle
def host_group_caches(K, V, page_table, seq_len, bound="kv", stat="f32"):
    """One oracle cache per KV group of sequence 0 (pages gathered in logical order; the oracle
    computes its own metadata).  Cache state, not per-step work."""
    import numpy as np
    import torch

    import oracle
    M = (seq_len + P - 1) // P
    phys = page_table[0, :M].long()
    caches = []
    for kv in range(K.shape[1]):
        Kh = K[phys, kv].float().cpu().numpy()[:, None]
        Vh = V[phys, kv].float().cpu().numpy()[:, None]
        hc = oracle.HostCache(Kh, Vh, np.arange(M, dtype=np.int32)[None], np.array([seq_len], np.int32))
        hc.build_stats(bound=bound, stat=stat)
        caches.append(hc)
        del Kh, Vh
        torch.cuda.empty_cache() if torch.cuda.is_available() else None
    return caches


def oracle_step(caches, qh, alpha, k_pages, threads, heads=None):
    """The oracle's decode step (score all pages -> top-k -> exact sparse entmax) for the given
    query heads, one head per task on `threads` threads (ctypes releases the GIL)."""
    import oracle
    G = HQ // HKV
    heads = list(range(HQ)) if heads is None else heads

    def one(h):
        return h, oracle.decode_head(caches[h // G], qh[0, h], 0, 0, alpha, k_pages=k_pages)

    if threads <= 1:
        return dict(one(h) for h in heads)
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        return dict(ex.map(one, heads))


def time_oracle(caches, qh, alpha, k_pages, threads, reps, heads=None):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        oracle_step(caches, qh, alpha, k_pages, threads, heads)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (as it stands) decoding the same 1M-token cache, the
    whole 32-head step per step, threaded over the host's cores; W untimed + K timed steps."""
    import torch
    if world > 1 and rank != 0:
        return
    dev = torch.device("cuda") if torch.cuda.is_available() else torch.device("cpu")
    k_pages = k_pages_for(args)
    wl = workload_for(args, 0, dev)
    caches = host_group_caches(wl.K, wl.V, wl.page_table, int(wl.seq_lens[0]), args.bounds, args.stats)
    qh = wl.q.float().cpu().numpy()
    del wl
    cores = os.cpu_count() or 1
    threads = min(cores, HQ)
    for _ in range(args.warmup):
        oracle_step(caches, qh, args.alpha, k_pages, threads)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle_step(caches, qh, args.alpha, k_pages, threads)
        ts.append(time.perf_counter() - t0)
    us = statistics.median(ts) * 1e6
    line = {"impl": "reference", "metric": METRIC, "value": us, "unit": "us", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C4: 1 seq x {args.n} ctx, 32q/8kv, d=128, P=16, alpha={args.alpha}, top-k "
                                   f"{args.budget:.0%} (k={k_pages}), {args.workload}, page bounds {args.bounds}, "
                                   f"stats {args.stats}"},
            "cpu_baseline": {"value": us, "unit": "us", "cores": threads, "kind": "oracle",
                             "sample": f"the whole step (32 query heads: score all {len(caches[0].page_table[0])} pages, "
                                       f"top-k, exact sparse entmax), one head per thread on {threads} of {cores} "
                                       f"host cores; median of {args.steps} steps after {args.warmup} warm-up"},
            "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- timing helpers
def make_timer(stream):
    import torch

    def time_graph(fn, reps, warm=3):
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            fn()
        stream.synchronize()
        with torch.cuda.graph(gg, stream=stream):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for _ in range(warm):
                gg.replay()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(reps):
                gg.replay()
            b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / reps
    return time_graph


def union_pages(pi, ns):
    import torch
    G = HQ // HKV
    u = 0
    for gk in range(HKV):
        rows = [pi[0, gk * G + j, :int(ns[0, gk * G + j])] for j in range(G)]
        u += int(torch.unique(torch.cat(rows)).numel())
    return u


def quality(ekv, cache, q, sel, attn, dev):
    """Exact delta and support recall rho vs full-cache entmax (eval mode, untimed)."""
    import torch
    ste = ekv.DecodeStats(1, HQ, dev, delta_bar=True, eval_exact=True, gauss=sel.policy == ekv.EKV_GAUSS)
    ekv.decode(cache, q, sel, attn, ekv.alloc_workspace(cache, HQ, sel), stats=ste)
    torch.cuda.synchronize()
    rec, sup = ste.recovered.double(), ste.full_supp.double()
    rho = rec / sup.clamp_min(1)
    return {"rho_pooled": float((rec.sum() / sup.sum()).item()), "rho_min": float(rho.min().item()),
            "rho_mean": float(rho.mean().item()), "delta_mean": float(ste.delta.mean().item()),
            "delta_max": float(ste.delta.max().item()), "supp_full_mean": float(sup.mean().item()),
            "delta_bar_mean": float(ste.delta_bar.mean().item()),
            "coverage": float(ste.n_sel.float().mean().item()) / ((int(cache.seq_lens[0]) + P - 1) // P)}


# ----------------------------------------------------------------------------- sequence sharding (N > 1)
def run_seq_sharded(args, rank, world, dev, k_pages):
    """configs[3]'s multi-GPU form: ONE 1M-token sequence whose pages are striped over the N
    ranks (page p on rank p mod N); every step = local scoring + top-k, global top-k merge,
    K scores, z_max all-reduce, multisection tau rounds (all-reduce of the partial
    sum (z - x)_+^beta), power-sum tau, numerator/denominator all-reduce.  Two collective
    modes, both timed: "nccl" = NCCL all-reduce / all-gather through torch.distributed between
    the library's kernels (host loop over the rounds); "in_kernel" = the
    library's own kernels exchange over NVLink peer memory (CUDA IPC buffers, remote stores
    + flags), no host read, the step replayed as a CUDA graph.  The in-kernel output is
    checked against the NCCL output on every rank; the headline is the faster valid mode.
    Timed with CUDA events per rank, max over ranks (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2605_21649_b200 import binding as ekv
    from paper_2605_21649_b200 import sharding
    wl = workload_for(args, 0, dev)                       # the same sequence on every rank
    cache = sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, rank, world)
    gl = wl.seq_lens.to(torch.int32).to(dev)
    q = wl.q.to(dev)
    del wl
    torch.cuda.empty_cache()
    sel = ekv.select_params("topk", k_pages)
    attn = ekv.attn_params(args.alpha)
    ws = ekv.shard_workspace(cache, HQ, sel, world)
    s = torch.cuda.Stream(device=dev)
    res = {"local_pages": int(cache.page_table.shape[1])}

    def timed(comm, graph):
        st = ekv.DecodeStats(1, HQ, dev, delta_bar=False)
        out = torch.empty(1, HQ, D, dtype=torch.float32, device=dev)
        run = lambda: ekv.decode_sharded(cache, gl, q, sel, attn, comm, ws, out=out, stats=st, stream=s)
        with torch.cuda.stream(s):
            for _ in range(max(3, args.warmup)):
                run()
        torch.cuda.synchronize()
        g = None
        if graph:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                run()
            torch.cuda.synchronize()
            dist.barrier()
            with torch.cuda.stream(s):
                g.replay()
            torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(args.steps):
                g.replay() if g is not None else run()
            e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) * 1e3 / args.steps], device=dev)
        tt = t.cpu() if os.environ.get("EKV_SAME_DEVICE") == "1" else t
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item()), out, st

    us_n, out_n, st_n = timed(sharding.TorchComm(), False)
    res["nccl"] = {"us_per_step": us_n, "how": "NCCL collectives via torch.distributed between the kernels, "
                                               "host loop over the multisection rounds"}
    try:
        pc = sharding.ipc_peer_comm(ekv.peer_buffer_size(cache, HQ, sel, world))
        us_k, out_k, st_k = timed(pc, True)
        err = (out_k - out_n).abs().max().item()
        same_supp = bool(torch.equal(st_k.supp_count, st_n.supp_count))
        ok = torch.tensor([1.0 if (err <= 1e-5 and same_supp) else 0.0],
                          device="cpu" if os.environ.get("EKV_SAME_DEVICE") == "1" else dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        res["in_kernel"] = {"us_per_step": us_k, "max_abs_vs_nccl": err, "supports_equal": same_supp,
                            "valid_on_all_ranks": bool(ok.item() == 1.0),
                            "how": "in-kernel collectives over NVLink peer memory (CUDA IPC buffers, remote "
                                   "stores + flags, rank-order reduction), no host read, CUDA-graph replay"}
    except Exception as e:  # reported; the NCCL mode stands
        res["in_kernel"] = {"error": f"{type(e).__name__}: {e}"}
    best = "nccl"
    if res["in_kernel"].get("valid_on_all_ranks") and res["in_kernel"]["us_per_step"] < us_n:
        best = "in_kernel"
    res["mode"] = best
    res["us_per_step"] = res[best]["us_per_step"]
    res["outputs_finite"] = bool(torch.isfinite(out_n).all().item())
    res["supp_mean"] = float(st_n.supp_count.float().mean().item())
    return res


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun on this node
        # (the arguments travel in the environment: torchrun's own parser would claim abbreviations
        # such as --n that follow the script name)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)]
        sys.exit(subprocess.call(cmd, env=dict(os.environ, EKV_BENCH_ARGV=json.dumps(sys.argv[1:]))))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import numpy as np
    import torch
    import torch.distributed as dist
    same = os.environ.get("EKV_SAME_DEVICE") == "1"     # test knob: N ranks on cuda:0 over gloo
    if world > 1:
        dist.init_process_group("gloo" if same else "nccl", init_method="env://")
    if same:
        local = 0
    torch.cuda.set_device(local)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.destroy_process_group()
        return

    from paper_2605_21649_b200 import binding as ekv
    from paper_2605_21649_b200.workload import new_tokens

    dev = torch.device("cuda", local)
    n = args.n
    M = (n + P - 1) // P
    k_pages = k_pages_for(args)
    # appended tokens grow the sequence; start slightly below n so that the context stays
    # within the 65536-page table
    spare = args.steps + args.warmup + 64 + max(5, args.steps // 2) + 16
    n0 = n - spare if (n + spare + P - 1) // P > 65536 else n
    wl = workload_for(args, rank, dev, n_tokens=n0, spare=n - n0 if n0 < n else spare)
    cache = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens, bound=args.bounds, stat=args.stats)
    ekv.rebuild_page_stats(cache)
    sel = ekv.select_params(args.policy, k_pages, 0.99, 0.0)
    attn = ekv.attn_params(args.alpha)
    ws = ekv.alloc_workspace(cache, HQ, sel)
    stats = ekv.DecodeStats(1, HQ, dev, delta_bar=True, gauss=args.policy == "gauss")
    # the query the heavy hitters were planted for (planted workload; randn: q ~ N(0, I) either
    # way); the appended token's k/v are fresh draws
    _, kn, vn = new_tokens(1, HQ, HKV, seed=7 + rank, device=dev)
    q = wl.q.contiguous()
    out = torch.empty(1, HQ, D, dtype=torch.float32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.synchronize()

    def step():
        ekv.append_kv(cache, kn, vn, stream=stream)
        ekv.decode(cache, q, sel, attn, ws, out=out, stats=stats, stream=stream)

    with torch.cuda.stream(stream):
        for _ in range(3):
            step()
        launches_decode = ekv.last_launch_count()
    stream.synchronize()
    # the step as one CUDA graph (the library is capture-safe: no sync, no alloc)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    stream.synchronize()
    launches_per_step = 1 + launches_decode

    with torch.cuda.stream(stream):        # replay() launches on the current stream
        for _ in range(args.warmup):
            g.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(args.steps):
                g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
    t_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([t_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t.item())
        dist.barrier()
    us_step = t_ms * 1e3 / args.steps
    time_graph = make_timer(stream)
    reps = max(10, args.steps)

    # ---- the dominant kernel (k_score, kmin/kmax of every page) timed alone, live
    box, _, _ = ekv.score_pages(cache, q, modes=1)
    pi, ns, _ = ekv.select(cache, HQ, ekv.select_params("topk", k_pages), alpha=args.alpha, box=box)
    torch.cuda.synchronize()
    phases = {}
    phases["score_pages"] = time_graph(lambda: ekv.score_pages_into(cache, q, box, stream=stream), reps)
    if not args.no_extras:
        phases["select_topk"] = time_graph(
            lambda: ekv.select_into(cache, HQ, ekv.select_params("topk", k_pages), args.alpha, box, pi, ns,
                                    stream=stream), reps)
        phases["sparse_attend"] = time_graph(
            lambda: ekv.sparse_attend(cache, q, pi, ns, attn, workspace=ws, stream=stream), reps)
    torch.cuda.synchronize()
    n_tok = int(cache.seq_lens[0].item())
    meta_bytes = M * HKV * 2 * D * (1 if args.bounds == "e4m3" else 2)   # kmin + kmax of every page
    score_gbs = meta_bytes / (phases["score_pages"] * 1e-6) / 1e9
    peak, peak_kind = peaks()

    # bytes of the sparse step (algorithmic): metadata + K of the union + V of support
    ekv.decode(cache, q, sel, attn, ws, out=out, stats=stats, stream=stream)
    torch.cuda.synchronize()
    union = union_pages(pi, ns) if args.policy == "topk" else None
    supp = int(stats.supp_count.sum().item())
    kv_sparse = (union or 0) * P * D * 2 + supp * D * 2
    step_bytes = meta_bytes + kv_sparse + HQ * D * 2 + HQ * D * 4
    full_bytes = n_tok * HKV * 2 * D * 2

    line_extra = {}
    if not args.no_extras:
        # ---- the paper's approximate threshold (N1, R23: histogram init + 2 Halley steps)
        attn_apx = ekv.attn_params(args.alpha, tau_halley=2)
        outa = torch.empty_like(out)
        stats_a = ekv.DecodeStats(1, HQ, dev, delta_bar=True, gauss=args.policy == "gauss")
        approx_us = time_graph(lambda: ekv.decode(cache, q, sel, attn_apx, ws, out=outa, stats=stats_a,
                                                  stream=stream), reps)
        torch.cuda.synchronize()
        ekv.decode(cache, q, sel, attn, ws, out=out, stats=stats, stream=stream)
        torch.cuda.synchronize()
        line_extra["decode_approx_tau"] = {
            "us": approx_us, "tau_halley": 2, "maxabs_vs_exact": float((outa - out).abs().max().item()),
            "note": "decode only (no append), the paper's histogram + Halley threshold (P:485)"}

    # ---- full-cache entmax baselines (a5) on the same cache
    full_us = full_dense_us = None
    full_out = None
    if not args.no_full:
        wsf = ekv.alloc_workspace(cache, HQ, None)
        fo = torch.empty(1, HQ, D, dtype=torch.float32, device=dev)
        ft = torch.empty(1, HQ, dtype=torch.float64, device=dev)
        fsu = torch.empty(1, HQ, dtype=torch.int32, device=dev)
        full_us = time_graph(lambda: ekv.full_attend(cache, q, attn, workspace=wsf, out=fo, tau=ft, supp=fsu,
                                                     stream=stream), max(5, reps // 5))
        attn_d = ekv.attn_params(args.alpha, dense_v=True)
        full_dense_us = time_graph(lambda: ekv.full_attend(cache, q, attn_d, workspace=wsf, out=fo, tau=ft,
                                                           supp=fsu, stream=stream), max(5, reps // 5))
        torch.cuda.synchronize()
        full_out = fo.clone()
        del wsf

    if not args.no_extras:
        # ---- selection quality at the headline point and the budget sweep (planted: recall claim)
        decode_only_us = time_graph(lambda: ekv.decode(cache, q, sel, attn, ws, out=out, stats=stats, stream=stream),
                                    reps)
        line_extra["quality"] = quality(ekv, cache, q, sel, attn, dev)
        sweep = []
        for bud in (0.01, 0.02, 0.05, 0.10):
            kb = max(1, math.ceil(bud * M))
            sb = ekv.select_params("topk", kb)
            wsb = ekv.alloc_workspace(cache, HQ, sb)
            stb = ekv.DecodeStats(1, HQ, dev, delta_bar=True)
            ob = torch.empty_like(out)
            us_b = time_graph(lambda: ekv.decode(cache, q, sb, attn, wsb, out=ob, stats=stb, stream=stream), reps)
            qb = quality(ekv, cache, q, sb, attn, dev)
            qb.update(budget=bud, k_pages=kb, decode_us=us_b,
                      speedup_vs_full_dense_v=(full_dense_us / us_b) if full_dense_us else None,
                      speedup_vs_full_support_v=(full_us / us_b) if full_us else None)
            sweep.append(qb)
            del wsb
        line_extra["budget_sweep"] = sweep
        ok = [s for s in sweep if s["rho_pooled"] >= 0.99 and s["rho_min"] >= 0.99]
        line_extra["recall_point"] = (
            {"budget": ok[0]["budget"], "k_pages": ok[0]["k_pages"], "rho_pooled": ok[0]["rho_pooled"],
             "rho_min": ok[0]["rho_min"], "decode_us": ok[0]["decode_us"],
             "speedup_vs_full_dense_v": ok[0]["speedup_vs_full_dense_v"],
             "speedup_vs_full_support_v": ok[0]["speedup_vs_full_support_v"]} if ok else None)
        line_extra["decode_only_us"] = decode_only_us
        # ---- the Gaussian-aware selector (the paper's 1M variant) on the same cache
        try:
            sg = ekv.select_params("gauss", 0, 0.99, 0.0)
            wsg = ekv.alloc_workspace(cache, HQ, sg)
            stg = ekv.DecodeStats(1, HQ, dev, delta_bar=False, gauss=True)
            og = torch.empty_like(out)
            g_us = time_graph(lambda: ekv.decode(cache, q, sg, attn, wsg, out=og, stats=stg, stream=stream),
                              max(5, reps // 5))
            qg = quality(ekv, cache, q, sg, attn, dev)
            qg.update(decode_us=g_us, q_page=0.99, margin=0.0,
                      speedup_vs_full_dense_v=(full_dense_us / g_us) if full_dense_us else None)
            # the paper's Gaussian kernel: tau_hat passed to the decode kernel + one Halley
            # refinement on the selected scores (R25) instead of the exact threshold
            a1 = ekv.attn_params(args.alpha, tau_halley=1)
            og1 = torch.empty_like(out)
            g1_us = time_graph(lambda: ekv.decode(cache, q, sg, a1, wsg, out=og1, stats=stg, stream=stream),
                               max(5, reps // 5))
            ekv.decode(cache, q, sg, attn, wsg, out=og, stats=stg, stream=stream)
            ekv.decode(cache, q, sg, a1, wsg, out=og1, stats=stg, stream=stream)
            torch.cuda.synchronize()
            rel = lambda x, y: float(((x - y).norm(dim=-1) / y.norm(dim=-1).clamp_min(1e-30)).mean().item())
            qg["tau_hat_halley1"] = {"decode_us": g1_us, "R_vs_exact_sparse_mean": rel(og1, og)}
            if full_out is not None:
                qg["R_vs_full_mean"] = rel(og, full_out)
                qg["tau_hat_halley1"]["R_vs_full_mean"] = rel(og1, full_out)
            line_extra["gaussian_selector"] = qg
            del wsg
        except Exception as e:  # reported, the headline stands
            line_extra["gaussian_selector"] = {"error": f"{type(e).__name__}: {e}"}
        # ---- N4: certified conservative box selection (Prop. B.2) -- exact full-cache entmax
        try:
            sc = ekv.select_params("certified", k_pages)
            wsc = ekv.alloc_workspace(cache, HQ, sc)
            stc = ekv.DecodeStats(1, HQ, dev, delta_bar=True, gauss=True)
            oc = torch.empty_like(out)
            c_us = time_graph(lambda: ekv.decode(cache, q, sc, attn, wsc, out=oc, stats=stc, stream=stream),
                              max(3, reps // 10))
            ekv.decode(cache, q, sc, attn, wsc, out=oc, stats=stc, stream=stream)
            torch.cuda.synchronize()
            line_extra["certified_selection"] = {
                "decode_us": c_us, "first_pass_k_pages": k_pages,
                "coverage": float(stc.n_sel.float().mean().item()) / M,
                "delta_bar_max": float(stc.delta_bar.max().item()),
                "maxabs_vs_full": float((oc - full_out).abs().max().item()) if full_out is not None else None,
                "speedup_vs_full_dense_v": (full_dense_us / c_us) if full_dense_us else None,
                "note": "Prop. B.2: pages with (alpha-1) box > tau~ of a top-k pass; output = full-cache entmax"}
            del wsc
        except Exception as e:
            line_extra["certified_selection"] = {"error": f"{type(e).__name__}: {e}"}
        # ---- N4: Gaussian selector at a non-integer beta (alpha = 1.7: beta = 1.43, numerical expectation)
        try:
            a17 = ekv.attn_params(1.7)
            sg = ekv.select_params("gauss", 0, 0.99, 0.0)
            wsn = ekv.alloc_workspace(cache, HQ, sg)
            stn = ekv.DecodeStats(1, HQ, dev, delta_bar=False, gauss=True)
            on = torch.empty_like(out)
            n_us = time_graph(lambda: ekv.decode(cache, q, sg, a17, wsn, out=on, stats=stn, stream=stream),
                              max(3, reps // 10))
            ekv.decode(cache, q, sg, a17, wsn, out=on, stats=stn, stream=stream)
            torch.cuda.synchronize()
            line_extra["gaussian_non_integer_beta"] = {
                "alpha": 1.7, "beta": 1.0 / (float(np.float32(1.7)) - 1.0), "decode_us": n_us,
                "coverage": float(stn.n_sel.float().mean().item()) / M,
                "outputs_finite": bool(torch.isfinite(on).all().item())}
            del wsn
        except Exception as e:
            line_extra["gaussian_non_integer_beta"] = {"error": f"{type(e).__name__}: {e}"}

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    qh_p = q.cpu().pin_memory()
    kh, vh = kn.cpu().pin_memory(), vn.cpu().pin_memory()
    oh = torch.empty(1, HQ, D, dtype=torch.float32).pin_memory()
    qd, kd, vd = torch.empty_like(q), torch.empty_like(kn), torch.empty_like(vn)
    e2e_steps = max(5, args.steps // 2)

    def e2e_step():
        qd.copy_(qh_p, non_blocking=True)
        kd.copy_(kh, non_blocking=True)
        vd.copy_(vh, non_blocking=True)
        ekv.append_kv(cache, kd, vd, stream=stream)
        ekv.decode(cache, qd, sel, attn, ws, out=out, stats=stats, stream=stream)
        oh.copy_(out, non_blocking=True)

    # (1) the user's step captured once and replayed, synchronised on the host every step
    ge = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        e2e_step()
    stream.synchronize()
    with torch.cuda.graph(ge, stream=stream):
        e2e_step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        a.record(stream)
        for _ in range(e2e_steps):
            ge.replay()
            stream.synchronize()
        b.record(stream)
    torch.cuda.synchronize()
    e2e_us = a.elapsed_time(b) * 1e3 / e2e_steps
    # (2) eager: every call through ctypes and the C ABI (validation + launches) each step
    with torch.cuda.stream(stream):
        for _ in range(3):
            e2e_step()
            stream.synchronize()
        a.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
            stream.synchronize()
        b.record(stream)
    torch.cuda.synchronize()
    e2e_eager_us = a.elapsed_time(b) * 1e3 / e2e_steps
    h2d = qh_p.numel() * 2 + kh.numel() * 2 + vh.numel() * 2
    d2h = oh.numel() * 4

    # ---- the CPU oracle on the SAME cache state: parity of the timed configuration + baseline
    cpu = None
    oracle_check = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.policy == "topk":
        try:
            st_chk = ekv.DecodeStats(1, HQ, dev, delta_bar=True, supp_cap=8192)
            out_chk = ekv.decode(cache, q, sel, attn, ws, stats=st_chk, stream=stream)
            pi_chk, ns_chk, _ = ekv.select(cache, HQ, ekv.select_params("topk", k_pages), alpha=args.alpha,
                                           box=ekv.score_pages(cache, q, modes=1, stream=stream)[0], stream=stream)
            torch.cuda.synchronize()
            seq_len = int(cache.seq_lens[0].item())
            caches = host_group_caches(cache.K, cache.V, cache.page_table, seq_len, args.bounds, args.stats)
            qh = q.float().cpu().numpy()
            cores = os.cpu_count() or 1
            threads = min(cores, HQ)
            refs = oracle_step(caches, qh, args.alpha, k_pages, threads)
            o_gpu = out_chk.cpu().numpy()
            worst, pages_eq, supp_eq, tau_err = 0.0, 0, 0, 0.0
            for h in range(HQ):
                r = refs[h]
                worst = max(worst, float(np.max(np.abs(o_gpu[0, h] - r["o"]))))
                if args.policy == "topk":
                    pages_eq += int(pi_chk[0, h, :int(ns_chk[0, h])].cpu().tolist() == r["pages"].tolist())
                att = caches[h // (HQ // HKV)].attend(qh[0, h], 0, 0, r["pages"], args.alpha, want_p=True)
                supp_eq += int(st_chk.support(0, h).cpu().tolist() == np.nonzero(att["p"])[0].tolist())
                tau_err = max(tau_err, abs(float(st_chk.tau[0, h]) - r["tau"]) / max(1.0, abs(r["tau"])))
            oracle_check = {"rows": HQ, "max_abs": worst, "page_sets_equal": pages_eq if args.policy == "topk" else None,
                            "support_sets_equal": supp_eq, "tau_max_rel_err": tau_err,
                            "state": f"the timed cache after its {seq_len - n0} appended tokens (seq_len {seq_len})"}
            t_thr = time_oracle(caches, qh, args.alpha, k_pages, threads, reps=3)
            t_one = time_oracle(caches, qh, args.alpha, k_pages, 1, reps=1, heads=list(range(HQ // HKV)))
            cpu = {"value": t_thr * 1e6, "unit": "us", "cores": threads, "kind": "oracle",
                   "sample": f"the whole 32-head step on the timed cache state, one query head per thread on "
                             f"{threads} of {cores} host cores, median of 3",
                   "single_thread_us": t_one * HKV * 1e6,
                   "single_thread_sample": "1 of 8 KV groups (4 query heads) on one core, x8"}
            del caches
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "us", "cores": 1, "kind": "oracle", "sample": f"failed: {type(e).__name__}: {e}"}

    seq = None
    if world > 1:
        try:
            seq = run_seq_sharded(args, rank, world, dev, k_pages)
        except Exception as e:  # reported, the batch-sharded line stands
            seq = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        step_gbs = step_bytes / (us_step * 1e-6) / 1e9
        line = {
            "metric": METRIC, "value": us_step, "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": us_step / 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": f"synthetic ({args.workload})",
            "config": {"workload": f"C4: 1 seq x {args.n} ctx per GPU, 32q/8kv heads, d=128, P=16, bf16, "
                                   f"alpha={args.alpha}, {args.policy} {args.budget:.0%} (k={k_pages} pages), "
                                   f"{args.workload}, page bounds {args.bounds}, stats {args.stats}; step = append + score + select + sparse entmax + delta_bar; "
                                   f"CUDA-graph replay",
                       "l2": "inputs larger than L2 (K/V 4 GiB, metadata 1.5 GiB per GPU): no flush",
                       "parallelism": f"batch-sharded x{world} (one sequence per GPU, no collective)"},
            "roofline": {"bound": "hbm", "kernel": "score_pages (k_score)", "achieved": score_gbs, "peak": peak,
                         "unit": "GB/s", "frac": score_gbs / peak, "traffic": ncu_traffic("k_score"),
                         "peak_kind": peak_kind, "algorithmic_bytes_per_launch": meta_bytes,
                         "kernel_us": phases["score_pages"]},
            "step_roofline": {"bytes": step_bytes, "achieved_gbs": step_gbs, "frac_measured_peak": step_gbs / peak,
                              "frac_nominal_8tbs": step_gbs / NOMINAL_HBM_GBS},
            "phases_us": phases,
            "bytes_read_vs_full": step_bytes / full_bytes,
            # a5 baseline (SURVEY 8(c) reading 17): dense-V full-cache entmax (all K and all V, the
            # paper's reference P:1343); the support-V variant (all K, V of the support) beside it
            "full_entmax_us": full_dense_us,
            "speedup_vs_full_entmax": (full_dense_us / us_step) if full_dense_us else None,
            "full_entmax_support_v_us": full_us,
            "speedup_vs_full_entmax_support_v": (full_us / us_step) if full_us else None,
            "full_entmax_dense_v_roofline_us": full_bytes / (peak * 1e3),
            "full_entmax_dense_v_frac": (full_bytes / (peak * 1e3)) / full_dense_us if full_dense_us else None,
            "speedup_vs_full_entmax_roofline": full_bytes / (peak * 1e3) / us_step,
            "cpu_baseline": cpu,
            "oracle_check": oracle_check,
            "e2e": {"value": e2e_us, "unit": "us", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "how": "public API step (pinned-host q/k/v in, append_kv, decode, out to host) captured in a "
                           "CUDA graph, host sync every step"},
            "e2e_eager": {"value": e2e_eager_us, "unit": "us",
                          "how": "the same step issued eagerly through ctypes + the C ABI every step"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "support_per_head_mean": supp / HQ, "union_pages": union,
        }
        line.update(line_extra)
        if seq is not None:
            line["batch_sharded"] = {"us_per_step": us_step, "scaling": "weak",
                                     "parallelism": f"batch-sharded x{world} (one 1M sequence per GPU)"}
            line["seq_sharded"] = seq
            if "us_per_step" in seq:
                # headline at N > 1: the one 1M sequence sequence-sharded over the N GPUs (configs[3])
                line["value"] = seq["us_per_step"]
                line["ms_per_step"] = seq["us_per_step"] / 1e3
                line["scaling"] = "strong"
                line["config"]["workload"] = (f"C4: ONE {args.n}-token sequence, pages striped over {world} GPUs, "
                                              f"32q/8kv, d=128, P=16, bf16, alpha={args.alpha}, top-k "
                                              f"{args.budget:.0%} (k={k_pages}), {args.workload}; step = local "
                                              f"score + top-k, all-gather merge, K scores, tau exchange ({seq.get('mode')}), "
                                              f"num/den all-reduce")
                line["config"]["parallelism"] = (f"sequence-sharded x{world} ("
                                                 + ("in-kernel collectives over NVLink peer memory"
                                                    if seq.get("mode") == "in_kernel" else "NCCL via torch.distributed")
                                                 + ")")
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
