#!/usr/bin/env python
"""Benchmark of the EntmaxKV sparse decode step on B200.

Default workload (BASELINE.json configs[3], the 1M-context config the metric is
quoted on; it fits one GPU): one 1,048,576-token sequence, Llama-3.1-8B attention
shape (32 q / 8 KV heads, d = 128), bf16, page 16, alpha = 1.5, top-k 1% of the
pages (k = 656), the paper's randn efficiency workload.

One step = append the new token's k/v (a0) + page scoring (a1) + top-k selection
(a2) + exact sparse alpha-entmax attention with delta_bar (a3, a4), replayed from a
CUDA graph.  The full-cache entmax baseline (a5) is timed on the same cache.
Inputs are larger than L2 (K/V 4 GiB, metadata 1.5 GiB), so no flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun): every rank decodes its own 1M sequence (batch sharding, weak
scaling, no collective in the step); the time is the max over ranks.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "µs per decode step (sparse vs full entmax) at 128K–1M ctx; HBM GB/s vs peak"


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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full", action="store_true")
    return ap.parse_args()


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
                                          "--format=csv,noheader,nounits", "-lms", "100"],
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


# ----------------------------------------------------------------------------- reference arm
def cpu_oracle_sample(n, Hq, Hkv, k_pages, alpha, seed, budget_s=20.0, wl=None):
    """Time the CPU oracle (as it stands) decoding one KV group (G query heads) of the
    workload: score all pages, top-k, sparse entmax.  Returns per-step microseconds
    extrapolated to all Hkv groups, cores used and a description."""
    import numpy as np
    import torch

    import oracle
    from paper_2605_21649_b200.workload import gather_head, make_workload

    if wl is None:
        wl = make_workload(1, n, Hq, Hkv, seed=seed, device="cuda" if torch.cuda.is_available() else "cpu")
    Kh, Vh = gather_head(wl, 0, 0)
    M = Kh.shape[0]
    hc = oracle.HostCache(Kh.float().cpu().numpy()[:, None], Vh.float().cpu().numpy()[:, None],
                          np.arange(M, dtype=np.int32)[None], np.array([int(wl.seq_lens[0])], np.int32))
    hc.build_stats()   # cache state (maintained incrementally by append), not per-step work
    G = Hq // Hkv
    qh = wl.q.float().cpu().numpy()
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        for g in range(G):
            oracle.decode_head(hc, qh[0, g], 0, 0, alpha, k_pages=k_pages)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_start > budget_s or len(times) >= 5:
            break
    per_group = statistics.median(times)
    return per_group * Hkv * 1e6, 1, f"1 of {Hkv} KV groups ({G} query heads) of the {n}-token step, " \
                                      f"median of {len(times)} runs, extrapolated x{Hkv}"


def run_reference(args, rank, world):
    import torch
    if world > 1 and rank != 0:
        return
    k_pages = max(1, math.ceil(args.budget * args.n / 16))
    steps = []
    for _ in range(args.warmup):
        pass
    us, cores, sample = cpu_oracle_sample(args.n, 32, 8, k_pages, args.alpha, seed=0, budget_s=20.0)
    steps = [us]
    line = {"impl": "reference", "metric": METRIC, "value": us, "unit": "us", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"C4 1M ctx, 32q/8kv, d=128, P=16, alpha={args.alpha}, top-k {args.budget:.0%}"
                                   f" (k={k_pages}), randn"},
            "cpu_baseline": {"value": us, "unit": "us", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": us, "unit": "us", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- sequence sharding (N > 1)
def run_seq_sharded(args, rank, world, dev, k_pages):
    """configs[3]'s multi-GPU form: ONE 1M-token sequence whose pages are striped over the N
    ranks (page p on rank p mod N); every step = local scoring + top-k, all-gather merge,
    K scores, z_max all-reduce, multisection tau rounds (all-reduce of the partial
    sum (z - x)_+^beta), power-sum tau, numerator/denominator all-reduce (NCCL through
    torch.distributed).  Timed with CUDA events per rank, max over ranks (strong scaling)."""
    import torch
    import torch.distributed as dist
    from paper_2605_21649_b200 import binding as ekv
    from paper_2605_21649_b200 import sharding
    from paper_2605_21649_b200.workload import make_workload
    Hq, Hkv = 32, 8
    wl = make_workload(1, args.n, Hq, Hkv, seed=1000, device=dev)     # same sequence on every rank
    cache = sharding.shard_cache(wl.K, wl.V, wl.page_table, wl.seq_lens, rank, world)
    gl = wl.seq_lens.to(torch.int32).to(dev)
    q = wl.q.to(dev)
    del wl
    torch.cuda.empty_cache()
    sel = ekv.select_params("topk", k_pages)
    attn = ekv.attn_params(args.alpha)
    ws = ekv.shard_workspace(cache, Hq, sel, world)
    st = ekv.DecodeStats(1, Hq, dev, delta_bar=False)
    out = torch.empty(1, Hq, 128, dtype=torch.float32, device=dev)
    comm = sharding.TorchComm()
    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        for _ in range(max(3, args.warmup)):
            ekv.decode_sharded(cache, gl, q, sel, attn, comm, ws, out=out, stats=st, stream=s)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(args.steps):
            ekv.decode_sharded(cache, gl, q, sel, attn, comm, ws, out=out, stats=st, stream=s)
        e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e3 / args.steps], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ok = bool(torch.isfinite(out).all().item())
    return {"us_per_step": float(t.item()), "local_pages": int(cache.page_table.shape[1]),
            "outputs_finite": ok, "supp_mean": float(st.supp_count.float().mean().item())}


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
    from paper_2605_21649_b200.workload import make_workload, new_tokens

    dev = torch.device("cuda", local)
    n, Hq, Hkv, d = args.n, 32, 8, 128
    P = 16
    M = (n + P - 1) // P
    k_pages = max(1, math.ceil(args.budget * M))
    # appended tokens grow the sequence; start slightly below n so that the context
    # stays within the 65536-page table (n = 2^20 -> 1,048,576 - spare ... 1,048,576 tokens)
    spare = args.steps + args.warmup + 64 + max(5, args.steps // 2) + 16
    n0 = n - spare if (n + spare + P - 1) // P > 65536 else n
    wl = make_workload(1, n0, Hq, Hkv, seed=1000 + rank, device=dev, spare_tokens=n - n0 if n0 < n else spare)
    cache = ekv.PagedCache.allocate_meta(wl.K, wl.V, wl.page_table, wl.seq_lens)
    ekv.rebuild_page_stats(cache)
    sel = ekv.select_params(args.policy, k_pages, 0.99, 0.0)
    attn = ekv.attn_params(args.alpha)
    ws = ekv.alloc_workspace(cache, Hq, sel)
    stats = ekv.DecodeStats(1, Hq, dev, delta_bar=True, gauss=args.policy == "gauss")
    q, kn, vn = new_tokens(1, Hq, Hkv, seed=7 + rank, device=dev)
    out = torch.empty(1, Hq, d, dtype=torch.float32, device=dev)
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

    # ---- per-kernel attribution (each phase replayed alone from its own graph)
    phases = {}

    def time_graph(fn, reps):
        gg = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            fn()
        stream.synchronize()
        with torch.cuda.graph(gg, stream=stream):
            fn()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for _ in range(3):
                gg.replay()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(reps):
                gg.replay()
            b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / reps

    box, mu, s2 = ekv.score_pages(cache, q, modes=1)
    pi, ns, _ = ekv.select(cache, Hq, sel, alpha=args.alpha, box=box)
    torch.cuda.synchronize()
    reps = max(10, args.steps)
    phases["score_pages"] = time_graph(lambda: ekv.score_pages_into(cache, q, box, stream=stream), reps)
    phases["select_topk"] = time_graph(lambda: ekv.select_into(cache, Hq, sel, args.alpha, box, pi, ns, stream=stream),
                                       reps)
    phases["sparse_attend"] = time_graph(
        lambda: ekv.sparse_attend(cache, q, pi, ns, attn, workspace=ws, stream=stream), reps)
    torch.cuda.synchronize()
    n_tok = int(cache.seq_lens[0].item())
    meta_bytes = M * Hkv * 2 * d * 2                      # kmin + kmax, bf16
    score_gbs = meta_bytes / (phases["score_pages"] * 1e-6) / 1e9
    peak, peak_kind = peaks()

    # bytes of the sparse step (algorithmic): metadata + K of the union + V of support
    G = Hq // Hkv
    union = 0
    for gk in range(Hkv):
        rows = [pi[0, gk * G + j, :int(ns[0, gk * G + j])] for j in range(G)]
        union += int(torch.unique(torch.cat(rows)).numel())
    supp = stats.supp_count.sum().item()
    kv_sparse = union * P * d * 2 + supp * d * 2
    step_bytes = meta_bytes + kv_sparse + Hq * d * 2 + Hq * d * 4
    full_bytes = n_tok * Hkv * 2 * d * 2

    # ---- the paper's approximate threshold (N1, R23: histogram init + 2 Halley steps)
    attn_apx = ekv.attn_params(args.alpha, tau_halley=2)
    outa = torch.empty_like(out)
    stats_a = ekv.DecodeStats(1, Hq, dev, delta_bar=True, gauss=args.policy == "gauss")
    approx_us = time_graph(lambda: ekv.decode(cache, q, sel, attn_apx, ws, out=outa, stats=stats_a, stream=stream), reps)
    torch.cuda.synchronize()
    ekv.decode(cache, q, sel, attn, ws, out=out, stats=stats, stream=stream)
    torch.cuda.synchronize()
    approx_maxabs = float((outa - out).abs().max().item())

    # ---- full-cache entmax baseline (a5)
    full_us = full_dense_us = None
    if not args.no_full:
        wsf = ekv.alloc_workspace(cache, Hq, None)
        fo = torch.empty(1, Hq, d, dtype=torch.float32, device=dev)
        ft = torch.empty(1, Hq, dtype=torch.float64, device=dev)
        fsu = torch.empty(1, Hq, dtype=torch.int32, device=dev)
        full_us = time_graph(lambda: ekv.full_attend(cache, q, attn, workspace=wsf, out=fo, tau=ft, supp=fsu,
                                                     stream=stream), max(5, reps // 5))
        attn_d = ekv.attn_params(args.alpha, dense_v=True)
        full_dense_us = time_graph(lambda: ekv.full_attend(cache, q, attn_d, workspace=wsf, out=fo, tau=ft,
                                                           supp=fsu, stream=stream), max(5, reps // 5))
        del wsf

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    qh = q.cpu().pin_memory()
    kh, vh = kn.cpu().pin_memory(), vn.cpu().pin_memory()
    oh = torch.empty(1, Hq, d, dtype=torch.float32).pin_memory()
    qd, kd, vd = torch.empty_like(q), torch.empty_like(kn), torch.empty_like(vn)
    e2e_steps = max(5, args.steps // 2)

    def e2e_step():
        qd.copy_(qh, non_blocking=True)
        kd.copy_(kh, non_blocking=True)
        vd.copy_(vh, non_blocking=True)
        ekv.append_kv(cache, kd, vd, stream=stream)
        ekv.decode(cache, qd, sel, attn, ws, out=out, stats=stats, stream=stream)
        oh.copy_(out, non_blocking=True)

    # the public API is graph-capturable: the user's step (pinned-host copies in, append,
    # decode, copy out) captured once and replayed, synchronised on the host every step
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
    h2d = qh.numel() * 2 + kh.numel() * 2 + vh.numel() * 2
    d2h = oh.numel() * 4

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cus, cores, sample = cpu_oracle_sample(args.n, Hq, Hkv, k_pages, args.alpha, seed=1000, budget_s=20.0)
            cpu = {"value": cus, "unit": "us", "cores": cores, "kind": "oracle", "sample": sample}
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "us", "cores": 1, "kind": "oracle", "sample": f"failed: {e}"}

    seq = None
    if world > 1:
        try:
            seq = run_seq_sharded(args, rank, world, dev, k_pages)
        except Exception as e:  # reported, the batch-sharded line stands
            seq = {"error": f"{type(e).__name__}: {e}"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": us_step, "unit": "us", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": us_step / 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"C4: 1 seq x {args.n} ctx per GPU, 32q/8kv heads, d=128, P=16, bf16, "
                                   f"alpha={args.alpha}, {args.policy} {args.budget:.0%} (k={k_pages} pages), randn "
                                   f"(P:629); step = append + score + select + sparse entmax; CUDA-graph replay",
                       "l2": "inputs larger than L2 (K/V 4 GiB, metadata 1.5 GiB per GPU)",
                       "parallelism": f"batch-sharded x{world} (one sequence per GPU, no collective)"},
            "roofline": {"bound": "hbm", "kernel": "score_pages (k_score)", "achieved": score_gbs, "peak": peak,
                         "unit": "GB/s", "frac": score_gbs / peak, "traffic": ncu_traffic("k_score"), "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": meta_bytes},
            "phases_us": phases,
            "step_bytes": step_bytes, "step_gbs": step_bytes / (us_step * 1e-6) / 1e9,
            "bytes_read_vs_full": step_bytes / full_bytes,
            # a5 baseline (SURVEY 8(c) reading 17): dense-V full-cache entmax (all K and all V, the
            # paper's reference P:1343); the support-V variant (all K, V of the support) beside it
            "full_entmax_us": full_dense_us,
            "speedup_vs_full_entmax": (full_dense_us / us_step) if full_dense_us else None,
            "full_entmax_support_v_us": full_us,
            "speedup_vs_full_entmax_support_v": (full_us / us_step) if full_us else None,
            # the dense-V baseline's own floor: all K + all V bytes at the HBM peak
            "full_entmax_dense_v_roofline_us": full_bytes / (peak * 1e3),
            "speedup_vs_full_entmax_roofline": full_bytes / (peak * 1e3) / us_step,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_us, "unit": "us", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "decode_approx_tau": {"us": approx_us, "tau_halley": 2, "maxabs_vs_exact": approx_maxabs,
                                  "note": "decode only (no append), the paper's histogram + Halley threshold"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "support_per_head_mean": supp / Hq, "union_pages": union,
        }
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
                                              f"{args.budget:.0%} (k={k_pages}); step = local score + top-k, "
                                              f"all-gather merge, K scores, NCCL multisection tau, num/den "
                                              f"all-reduce")
                line["config"]["parallelism"] = f"sequence-sharded x{world} (NCCL via torch.distributed)"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
