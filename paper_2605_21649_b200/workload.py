"""Seeded synthetic inputs for the EntmaxKV decode step.

This module holds NONE of the method's arithmetic: it only draws the inputs
(paged K/V caches, page tables, queries) that the CUDA path and the CPU oracle
both consume.  It is importable without the CUDA extension.

Workloads (recipes restated in DESIGN.md "Input recipe"):

* ``randn``   -- the paper's efficiency workload: q, k, v ~ N(0, I) rounded to the
  KV dtype.  Used for timing only.
* ``planted`` -- a Llama-shaped cache with planted heavy-hitter keys (the north
  star's "synthetic Llama-shaped paged KV caches with planted heavy-hitter
  keys"): anisotropic channel scales, 64 planted spans of 4 tokens per
  (sequence, kv head) aligned to one query head of the group, plus a sink at
  token 0.  Used for quality (recall) claims.  Background keys are i.i.d. over token
  positions: the worst case for page-level bounds (every page's box is the envelope of 16
  independent draws).
* ``llama``   -- ``planted`` on a background with token locality: the background key
  sequence of each (sequence, kv head) is an AR(1) process along token positions,
  k_t = phi k_{t-1} + sqrt(1 - phi^2) e_t (phi = 0.9, truncated to 64 taps), scaled per
  channel as in ``planted``.  Adjacent keys of real LLM caches are similar -- the premise
  of page-level (Quest-style) bounds the paper builds on -- so this is
  the north star's "Llama-shaped" cache; ``planted`` stays as the locality-free stress case.

Physical pages are a random permutation of the page pool (no locality), as in a
vLLM-style paged allocator.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch


@dataclass
class Workload:
    K: torch.Tensor            # [n_phys][Hkv][P][d]
    V: torch.Tensor            # [n_phys][Hkv][P][dv]
    page_table: torch.Tensor   # [B][max_pages] int32 (every entry a valid physical page)
    seq_lens: torch.Tensor     # [B] int32
    q: torch.Tensor            # [B][Hq][d] (KV dtype)
    Hq: int
    Hkv: int
    P: int
    d: int
    dv: int
    planted: dict = field(default_factory=dict)

    @property
    def B(self):
        return self.page_table.shape[0]

    @property
    def max_pages(self):
        return self.page_table.shape[1]


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def make_workload(B, seq_lens, Hq, Hkv, d=128, dv=128, P=16, dtype=torch.bfloat16, seed=0,
                  kind="randn", spare_tokens=0, device="cpu", n_spans=64, span_len=4,
                  kappa=(2.0, 8.0)) -> Workload:
    """Build a paged cache of B sequences.

    seq_lens: int (all equal) or list of ints.  spare_tokens: extra capacity per
    sequence (page-table entries already mapped to free physical pages) so that
    ``append_kv`` can grow the sequences.
    """
    if isinstance(seq_lens, int):
        seq_lens = [seq_lens] * B
    assert len(seq_lens) == B
    g = _gen(device, seed)
    max_pages = max((n + spare_tokens + P - 1) // P for n in seq_lens)
    max_pages = max(max_pages, 1)
    n_phys = B * max_pages
    perm = torch.randperm(n_phys, generator=g, device=device).to(torch.int32)
    page_table = perm.view(B, max_pages).contiguous()
    K32 = torch.randn(n_phys, Hkv, P, d, generator=g, device=device)
    V32 = torch.randn(n_phys, Hkv, P, dv, generator=g, device=device)
    q32 = torch.randn(B, Hq, d, generator=g, device=device)
    planted = {}
    if kind in ("planted", "llama"):
        K32, planted = _plant(K32, q32, page_table, seq_lens, Hq, Hkv, P, d, g, device,
                              n_spans, span_len, kappa, phi=0.9 if kind == "llama" else 0.0)
    elif kind != "randn":
        raise ValueError(f"unknown workload {kind!r}")
    sl = torch.tensor(seq_lens, dtype=torch.int32, device=device)
    return Workload(K=K32.to(dtype).contiguous(), V=V32.to(dtype).contiguous(), page_table=page_table,
                    seq_lens=sl, q=q32.to(dtype).contiguous(), Hq=Hq, Hkv=Hkv, P=P, d=d, dv=dv,
                    planted=planted)


def _ar_filter(x, phi, taps=64):
    """x [N][d] i.i.d. N(0, 1) rows -> AR(1) rows along N: y_t = sqrt(1 - phi^2) *
    sum_{j <= taps} phi^j x_{t-j} (unit variance up to phi^(2 taps + 2) ~ 1e-6)."""
    N, d = x.shape
    w = (math.sqrt(1.0 - phi * phi) * phi ** torch.arange(taps, -1, -1, dtype=torch.float32,
                                                            device=x.device))
    y = torch.nn.functional.conv1d(torch.nn.functional.pad(x.t().unsqueeze(0), (taps, 0)),
                                   w.view(1, 1, -1).expand(d, 1, taps + 1).contiguous(), groups=d)
    return y[0].t()


def _plant(K32, q32, page_table, seq_lens, Hq, Hkv, P, d, g, device, n_spans, span_len, kappa,
           phi=0.0):
    """Planted heavy hitters (DESIGN.md "Input recipe" W-llama-planted).

    Per (b, kv head): channel scales sigma_ch ~ logU[0.25, 4]; background keys
    k = sigma_ch * N(0, I) (phi > 0: k = sigma_ch * AR(1) along token positions, ``llama``); n_spans spans of span_len consecutive tokens at uniform
    positions plus a sink at token 0.  A planted key for query head h becomes
        k <- 0.6 k + kappa * sigma_bg,h * sqrt(d) * q_h / ||q_h||^2,
    so its score against q_h is raised by kappa * sigma_bg,h, where
    sigma_bg,h = ||sigma_ch * q_h|| / sqrt(d) is the background score std.
    kappa ~ U[kappa_lo, kappa_hi] per token; spans are assigned to the G query
    heads of the group round-robin; the sink is planted for every head.
    """
    G = Hq // Hkv
    B = page_table.shape[0]
    lo, hi = math.log(0.25), math.log(4.0)
    planted = {}
    for b in range(B):
        n = seq_lens[b]
        for kv in range(Hkv):
            sig_ch = torch.exp(lo + (hi - lo) * torch.rand(d, generator=g, device=device))
            # background for all tokens of this (b, kv)
            M = (n + P - 1) // P
            phys = page_table[b, :M].long()
            if phi > 0.0:
                bg = _ar_filter(K32[phys, kv].reshape(M * P, d), phi)
                K32[phys, kv] = bg.view(M, P, d) * sig_ch
            else:
                K32[phys, kv] = K32[phys, kv] * sig_ch
            starts = torch.randint(1, max(2, n - span_len), (n_spans,), generator=g, device=device)
            kap = kappa[0] + (kappa[1] - kappa[0]) * torch.rand(n_spans, span_len, generator=g, device=device)
            kap_sink = kappa[0] + (kappa[1] - kappa[0]) * torch.rand(G, generator=g, device=device)
            toks, heads = [], []
            for i in range(n_spans):
                h = kv * G + (i % G)
                qh = q32[b, h]
                sbg = torch.linalg.vector_norm(sig_ch * qh) / math.sqrt(d)
                u_dir = qh * (math.sqrt(d) / torch.dot(qh, qh))
                for t in range(span_len):
                    j = int(starts[i]) + t
                    if j >= n:
                        continue
                    ph, slot = page_table[b, j // P].long(), j % P
                    K32[ph, kv, slot] = 0.6 * K32[ph, kv, slot] + kap[i, t] * sbg * u_dir
                    toks.append(j)
                    heads.append(h)
            # sink at token 0 for every head of the group
            ph = page_table[b, 0].long()
            add = torch.zeros(d, device=device)
            for gi in range(G):
                qh = q32[b, kv * G + gi]
                sbg = torch.linalg.vector_norm(sig_ch * qh) / math.sqrt(d)
                add = add + kap_sink[gi] * sbg * qh * (math.sqrt(d) / torch.dot(qh, qh))
            K32[ph, kv, 0] = 0.6 * K32[ph, kv, 0] + add
            planted[(b, kv)] = (toks, heads)
    return K32, planted


def new_tokens(B, Hq, Hkv, d=128, dv=128, dtype=torch.bfloat16, seed=0, device="cpu"):
    """One decode step's fresh (q, k_new, v_new) ~ N(0, I) (the paper's randn workload)."""
    g = _gen(device, seed)
    q = torch.randn(B, Hq, d, generator=g, device=device).to(dtype)
    k = torch.randn(B, Hkv, d, generator=g, device=device).to(dtype)
    v = torch.randn(B, Hkv, dv, generator=g, device=device).to(dtype)
    return q, k, v


def gather_head(wl: Workload, b: int, kv: int):
    """Contiguous copy of one (sequence, kv head)'s pages, in logical order:
    K [M][P][d], V [M][P][dv] (indexing only; used to feed the oracle one head
    at full size)."""
    n = int(wl.seq_lens[b])
    M = (n + wl.P - 1) // wl.P
    phys = wl.page_table[b, :M].long()
    return wl.K[phys, kv].contiguous(), wl.V[phys, kv].contiguous()
