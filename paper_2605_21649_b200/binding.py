"""Thin ctypes binding over libentmaxkv.so (include/entmaxkv.h).

Argument marshalling only: torch tensors are passed as raw device pointers plus
sizes, the current CUDA stream as ``cudaStream_t``.  Every step of the decode
path runs in the library's CUDA kernels.  There is no CPU fallback: if the
shared library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libentmaxkv.so")

EKV_OK, EKV_ERR_INVALID_ARG, EKV_ERR_UNSUPPORTED, EKV_ERR_CAPACITY, EKV_ERR_EMPTY, EKV_ERR_CUDA, EKV_ERR_COMM = range(7)
EKV_BF16, EKV_F32 = 0, 1
EKV_ENTMAX, EKV_SOFTMAX = 0, 1
EKV_TOPK, EKV_GAUSS, EKV_ALL, EKV_CERTIFIED = 0, 1, 2, 3
EKV_SCORE_BOX, EKV_SCORE_GAUSS = 1, 2

EXPORTED = [
    "entmaxkv_last_error", "entmaxkv_version", "entmaxkv_workspace_size", "entmaxkv_select_capacity",
    "entmaxkv_workspace_status",
    "entmaxkv_append_kv", "entmaxkv_rebuild_page_stats", "entmaxkv_score_pages", "entmaxkv_select",
    "entmaxkv_sparse_attend", "entmaxkv_full_attend", "entmaxkv_decode", "entmaxkv_last_launch_count",
    "entmaxkv_shard_workspace_size", "entmaxkv_decode_sharded", "entmaxkv_peer_buffer_size",
]


class EkvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"entmaxkv status {status}: {msg}")
        self.status = status


class ekv_cache(ctypes.Structure):
    _fields_ = [("dtype", ctypes.c_int32), ("batch", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("value_dim", ctypes.c_int32), ("page_size", ctypes.c_int32),
                ("max_pages_per_seq", ctypes.c_int32), ("n_phys_pages", ctypes.c_int32),
                ("k_pages", ctypes.c_void_p), ("v_pages", ctypes.c_void_p),
                ("kmin", ctypes.c_void_p), ("kmax", ctypes.c_void_p),
                ("ksum", ctypes.c_void_p), ("ksumsq", ctypes.c_void_p), ("kavg", ctypes.c_void_p),
                ("kvar", ctypes.c_void_p), ("page_table", ctypes.c_void_p), ("seq_lens", ctypes.c_void_p),
                ("bound_dtype", ctypes.c_int32), ("stat_dtype", ctypes.c_int32)]


EKV_BOUND_KV, EKV_BOUND_E4M3 = 0, 1
EKV_STAT_F32, EKV_STAT_BF16 = 0, 1


EKV_ATTN_DENSE_V = 1
EKV_ATTN_CANONICAL = 2


class ekv_attn_params(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_float), ("transform", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("tau_halley", ctypes.c_int32)]


class ekv_select_params(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("k_pages", ctypes.c_int32), ("q_page", ctypes.c_double),
                ("margin", ctypes.c_double)]


class ekv_decode_stats(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_void_p), ("supp_count", ctypes.c_void_p), ("n_sel", ctypes.c_void_p),
                ("delta_bar", ctypes.c_void_p), ("tau_hat", ctypes.c_void_p), ("eval_exact", ctypes.c_int32),
                ("delta", ctypes.c_void_p), ("recovered", ctypes.c_void_p), ("full_supp", ctypes.c_void_p),
                ("tau_full", ctypes.c_void_p), ("supp_tok", ctypes.c_void_p), ("supp_cap", ctypes.c_int32)]


ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_void_p, ctypes.c_void_p)
ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                                ctypes.c_void_p)


class ekv_comm(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("allreduce", ALLREDUCE_FN),
                ("allgather", ALLGATHER_FN), ("user", ctypes.c_void_p), ("fixed_rounds", ctypes.c_int32),
                ("peers", ctypes.c_void_p * 8)]


_lib = None


def lib():
    """Load libentmaxkv.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` or `make`")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        vp, i32, f32, f64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_float, ctypes.c_double
        L.entmaxkv_last_error.restype = ctypes.c_char_p
        L.entmaxkv_version.restype = ctypes.c_char_p
        L.entmaxkv_workspace_size.argtypes = [P(ekv_cache), i32, P(ekv_select_params)]
        L.entmaxkv_workspace_size.restype = ctypes.c_size_t
        L.entmaxkv_select_capacity.argtypes = [P(ekv_cache), P(ekv_select_params)]
        L.entmaxkv_select_capacity.restype = i32
        L.entmaxkv_append_kv.argtypes = [P(ekv_cache), vp, vp, i32, vp]
        L.entmaxkv_rebuild_page_stats.argtypes = [P(ekv_cache), vp]
        L.entmaxkv_score_pages.argtypes = [P(ekv_cache), vp, i32, i32, vp, vp, vp, vp, vp]
        L.entmaxkv_select.argtypes = [P(ekv_cache), i32, vp, vp, vp, P(ekv_select_params), f32, vp, vp, i32, vp, vp, vp]
        L.entmaxkv_sparse_attend.argtypes = [P(ekv_cache), vp, i32, vp, vp, i32, vp, P(ekv_attn_params), vp, vp, vp, vp,
                                             vp]
        L.entmaxkv_full_attend.argtypes = [P(ekv_cache), vp, i32, P(ekv_attn_params), vp, vp, vp, vp, vp]
        L.entmaxkv_decode.argtypes = [P(ekv_cache), vp, i32, P(ekv_select_params), P(ekv_attn_params), vp,
                                      P(ekv_decode_stats), vp, vp]
        L.entmaxkv_last_launch_count.restype = i32
        L.entmaxkv_workspace_status.argtypes = [P(ekv_cache), i32, P(ekv_select_params), vp, P(i32), vp]
        L.entmaxkv_workspace_status.restype = ctypes.c_int
        L.entmaxkv_shard_workspace_size.argtypes = [P(ekv_cache), i32, P(ekv_select_params), i32]
        L.entmaxkv_shard_workspace_size.restype = ctypes.c_size_t
        L.entmaxkv_peer_buffer_size.argtypes = [P(ekv_cache), i32, P(ekv_select_params), i32]
        L.entmaxkv_peer_buffer_size.restype = ctypes.c_size_t
        L.entmaxkv_decode_sharded.argtypes = [P(ekv_cache), vp, vp, i32, P(ekv_select_params), P(ekv_attn_params),
                                              P(ekv_comm), vp, P(ekv_decode_stats), vp, vp]
        for name in ("entmaxkv_decode_sharded", "entmaxkv_append_kv", "entmaxkv_rebuild_page_stats", "entmaxkv_score_pages", "entmaxkv_select",
                     "entmaxkv_sparse_attend", "entmaxkv_full_attend", "entmaxkv_decode"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status):
    if status != EKV_OK:
        raise EkvError(status, lib().entmaxkv_last_error().decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def version() -> str:
    return lib().entmaxkv_version().decode()


def last_launch_count() -> int:
    return int(lib().entmaxkv_last_launch_count())


# ----------------------------------------------------------------------------- cache object
_DT = {torch.bfloat16: EKV_BF16, torch.float32: EKV_F32}


@dataclass
class PagedCache:
    """Device-resident paged KV cache + page metadata (caller-owned torch tensors)."""
    K: torch.Tensor          # [n_phys][Hkv][P][d]
    V: torch.Tensor          # [n_phys][Hkv][P][dv]
    page_table: torch.Tensor  # [B][max_pages] int32
    seq_lens: torch.Tensor   # [B] int32
    kmin: torch.Tensor
    kmax: torch.Tensor
    ksum: torch.Tensor
    ksumsq: torch.Tensor
    kavg: torch.Tensor
    kvar: torch.Tensor
    bound: str = "kv"        # "kv": kmin/kmax in the KV dtype; "e4m3": outward-rounded fp8 bytes (R24)
    stat: str = "f32"        # "f32" | "bf16": kavg / kvar storage

    @classmethod
    def allocate_meta(cls, K, V, page_table, seq_lens, bound="kv", stat="f32"):
        n_phys, Hkv, P, d = K.shape
        dev = K.device
        if bound not in ("kv", "e4m3") or stat not in ("f32", "bf16"):
            raise ValueError(f"bound {bound!r} / stat {stat!r}")
        mk = lambda dt: torch.zeros(n_phys, Hkv, d, dtype=dt, device=dev)
        bdt = torch.uint8 if bound == "e4m3" else K.dtype
        sdt = torch.bfloat16 if stat == "bf16" else torch.float32
        return cls(K, V, page_table.to(torch.int32).contiguous(), seq_lens.to(torch.int32).contiguous(),
                   mk(bdt), mk(bdt), mk(torch.float32), mk(torch.float32), mk(sdt), mk(sdt), bound, stat)

    def bounds_f32(self):
        """kmin, kmax as fp32 values (decodes the e4m3 bytes)."""
        if self.bound == "e4m3":
            return (self.kmin.view(torch.float8_e4m3fn).float(), self.kmax.view(torch.float8_e4m3fn).float())
        return self.kmin.float(), self.kmax.float()

    @property
    def batch(self):
        return self.page_table.shape[0]

    @property
    def n_kv_heads(self):
        return self.K.shape[1]

    @property
    def max_pages(self):
        return self.page_table.shape[1]

    def c_struct(self) -> ekv_cache:
        if self.K.dtype not in _DT:
            raise TypeError(f"unsupported KV dtype {self.K.dtype}")
        for t in (self.K, self.V, self.page_table, self.seq_lens, self.kmin, self.kmax, self.ksum, self.ksumsq,
                  self.kavg, self.kvar):
            if not t.is_cuda or not t.is_contiguous():
                raise ValueError("cache tensors must be contiguous CUDA tensors")
        n_phys, Hkv, P, d = self.K.shape
        return ekv_cache(_DT[self.K.dtype], self.batch, Hkv, d, self.V.shape[3], P, self.max_pages, n_phys,
                         self.K.data_ptr(), self.V.data_ptr(), self.kmin.data_ptr(), self.kmax.data_ptr(),
                         self.ksum.data_ptr(), self.ksumsq.data_ptr(), self.kavg.data_ptr(), self.kvar.data_ptr(),
                         self.page_table.data_ptr(), self.seq_lens.data_ptr(),
                         EKV_BOUND_E4M3 if self.bound == "e4m3" else EKV_BOUND_KV,
                         EKV_STAT_BF16 if self.stat == "bf16" else EKV_STAT_F32)


def select_params(policy="topk", k_pages=64, q_page=0.99, margin=0.0) -> ekv_select_params:
    pol = {"topk": EKV_TOPK, "gauss": EKV_GAUSS, "all": EKV_ALL, "certified": EKV_CERTIFIED}[policy]
    return ekv_select_params(pol, int(k_pages), float(q_page), float(margin))


def attn_params(alpha=1.5, transform="entmax", dense_v=False, tau_halley=0, canonical=False) -> ekv_attn_params:
    """tau_halley > 0: the paper's approximate threshold (histogram init + that many Halley steps).
    canonical: the full path scores in R1's order instead of on tensor cores (R26)."""
    return ekv_attn_params(float(alpha), {"entmax": EKV_ENTMAX, "softmax": EKV_SOFTMAX}[transform],
                           (EKV_ATTN_DENSE_V if dense_v else 0) | (EKV_ATTN_CANONICAL if canonical else 0),
                           int(tau_halley))


def workspace_size(cache: PagedCache, n_q_heads: int, sel: ekv_select_params | None) -> int:
    cs = cache.c_struct()
    n = lib().entmaxkv_workspace_size(ctypes.byref(cs), int(n_q_heads), None if sel is None else ctypes.byref(sel))
    if n == 0:
        raise EkvError(EKV_ERR_INVALID_ARG, lib().entmaxkv_last_error().decode())
    return int(n)


def workspace_status(cache: PagedCache, n_q_heads, sel, workspace, stream=None, raise_on_capacity=False) -> int:
    """Device status word of the last call on `workspace` (EKV_STATUS_* bits; synchronises the stream)."""
    cs = cache.c_struct()
    f = ctypes.c_int32(0)
    st = lib().entmaxkv_workspace_status(ctypes.byref(cs), int(n_q_heads), None if sel is None else ctypes.byref(sel),
                                         _ptr(workspace), ctypes.byref(f), _stream(stream))
    if st != EKV_OK and (st != EKV_ERR_CAPACITY or raise_on_capacity):
        _check(st)
    return int(f.value)


EKV_STATUS_CAPACITY = 1
EKV_STATUS_TIMEOUT = 2


def select_capacity(cache: PagedCache, sel: ekv_select_params) -> int:
    cs = cache.c_struct()
    return int(lib().entmaxkv_select_capacity(ctypes.byref(cs), ctypes.byref(sel)))


def alloc_workspace(cache, n_q_heads, sel=None, eval_exact=False):
    """One workspace serves decode (incl. eval_exact), select, sparse_attend and full_attend."""
    n = workspace_size(cache, n_q_heads, sel)
    return torch.empty(n, dtype=torch.uint8, device=cache.K.device)


# ----------------------------------------------------------------------------- entry points
def append_kv(cache: PagedCache, k_new, v_new, stream=None):
    """k_new/v_new: [B][n_tokens][Hkv][d] (or [B][Hkv][d] for one token)."""
    if k_new.dim() == 3:
        k_new, v_new = k_new.unsqueeze(1), v_new.unsqueeze(1)
    k_new, v_new = k_new.contiguous(), v_new.contiguous()
    cs = cache.c_struct()
    _check(lib().entmaxkv_append_kv(ctypes.byref(cs), _ptr(k_new), _ptr(v_new), int(k_new.shape[1]), _stream(stream)))


def rebuild_page_stats(cache: PagedCache, stream=None):
    cs = cache.c_struct()
    _check(lib().entmaxkv_rebuild_page_stats(ctypes.byref(cs), _stream(stream)))


def score_pages(cache: PagedCache, q, modes=EKV_SCORE_BOX, stream=None):
    B, Hq, _ = q.shape
    dev = q.device
    box = torch.empty(B, Hq, cache.max_pages, dtype=torch.float32, device=dev) if modes & 1 else None
    mu = torch.empty(B, Hq, cache.max_pages, dtype=torch.float32, device=dev) if modes & 2 else None
    s2 = torch.empty(B, Hq, cache.max_pages, dtype=torch.float32, device=dev) if modes & 2 else None
    cs = cache.c_struct()
    _check(lib().entmaxkv_score_pages(ctypes.byref(cs), _ptr(q.contiguous()), Hq, int(modes), _ptr(box), _ptr(mu),
                                      _ptr(s2), None, _stream(stream)))
    return box, mu, s2


def select(cache: PagedCache, n_q_heads, sel: ekv_select_params, alpha=1.5, box=None, mu=None, sigma2=None,
           stream=None, workspace=None):
    """workspace: needed by the Gaussian selector for a non-integer beta (its moment table);
    allocated here when None."""
    cap = select_capacity(cache, sel)
    if workspace is None and sel.policy == EKV_GAUSS:
        workspace = alloc_workspace(cache, n_q_heads, sel)
    dev = cache.K.device
    page_idx = torch.full((cache.batch, n_q_heads, cap), -1, dtype=torch.int32, device=dev)
    n_sel = torch.zeros(cache.batch, n_q_heads, dtype=torch.int32, device=dev)
    tau_hat = torch.zeros(cache.batch, n_q_heads, dtype=torch.float64, device=dev)
    cs = cache.c_struct()
    _check(lib().entmaxkv_select(ctypes.byref(cs), int(n_q_heads), _ptr(box), _ptr(mu), _ptr(sigma2), ctypes.byref(sel),
                                 float(alpha), _ptr(page_idx), _ptr(n_sel), cap, _ptr(tau_hat), _ptr(workspace),
                                 _stream(stream)))
    return page_idx, n_sel, tau_hat


def sparse_attend(cache: PagedCache, q, page_idx, n_sel, attn: ekv_attn_params, workspace=None, stream=None,
                  tau_init=None):
    B, Hq, _ = q.shape
    dev = q.device
    stride = page_idx.shape[2]
    if workspace is None:
        workspace = alloc_workspace(cache, Hq, select_params("topk", stride))
    out = torch.empty(B, Hq, cache.V.shape[3], dtype=torch.float32, device=dev)
    tau = torch.empty(B, Hq, dtype=torch.float64, device=dev)
    supp = torch.empty(B, Hq, dtype=torch.int32, device=dev)
    cs = cache.c_struct()
    _check(lib().entmaxkv_sparse_attend(ctypes.byref(cs), _ptr(q.contiguous()), Hq, _ptr(page_idx.contiguous()),
                                        _ptr(n_sel.contiguous()), stride,
                                        _ptr(None if tau_init is None else tau_init.contiguous()),
                                        ctypes.byref(attn), _ptr(out), _ptr(tau),
                                        _ptr(supp), _ptr(workspace), _stream(stream)))
    return out, tau, supp


def full_attend(cache: PagedCache, q, attn: ekv_attn_params, workspace=None, out=None, tau=None, supp=None,
                stream=None):
    B, Hq, _ = q.shape
    dev = q.device
    if workspace is None:
        workspace = alloc_workspace(cache, Hq, None)
    out = torch.empty(B, Hq, cache.V.shape[3], dtype=torch.float32, device=dev) if out is None else out
    tau = torch.empty(B, Hq, dtype=torch.float64, device=dev) if tau is None else tau
    supp = torch.empty(B, Hq, dtype=torch.int32, device=dev) if supp is None else supp
    cs = cache.c_struct()
    _check(lib().entmaxkv_full_attend(ctypes.byref(cs), _ptr(q.contiguous()), Hq, ctypes.byref(attn), _ptr(out),
                                      _ptr(tau), _ptr(supp), _ptr(workspace), _stream(stream)))
    return out, tau, supp


class DecodeStats:
    """Device buffers for ekv_decode_stats ([B][Hq] each)."""

    def __init__(self, B, Hq, device, delta_bar=True, eval_exact=False, gauss=False, supp_cap=0):
        f64 = lambda: torch.zeros(B, Hq, dtype=torch.float64, device=device)
        i32 = lambda: torch.zeros(B, Hq, dtype=torch.int32, device=device)
        self.tau, self.supp_count, self.n_sel = f64(), i32(), i32()
        self.delta_bar = f64() if delta_bar else None
        self.tau_hat = f64() if gauss else None
        self.eval_exact = bool(eval_exact)
        self.delta = f64() if eval_exact else None
        self.recovered = i32() if eval_exact else None
        self.full_supp = i32() if eval_exact else None
        self.tau_full = f64() if eval_exact else None
        self.supp_cap = int(supp_cap)
        self.supp_tok = (torch.full((B, Hq, self.supp_cap), -1, dtype=torch.int32, device=device)
                         if self.supp_cap > 0 else None)

    def c_struct(self):
        return ekv_decode_stats(_ptr(self.tau), _ptr(self.supp_count), _ptr(self.n_sel), _ptr(self.delta_bar),
                                _ptr(self.tau_hat), int(self.eval_exact), _ptr(self.delta), _ptr(self.recovered),
                                _ptr(self.full_supp), _ptr(self.tau_full), _ptr(self.supp_tok), self.supp_cap)

    def support(self, b, h):
        """Support token positions of row (b, h) (ascending; needs supp_cap > 0)."""
        n = min(int(self.supp_count[b, h]), self.supp_cap)
        return self.supp_tok[b, h, :n]


def decode(cache: PagedCache, q, sel: ekv_select_params, attn: ekv_attn_params, workspace, out=None,
           stats: DecodeStats | None = None, stream=None):
    """Fused decode step (score -> select -> sparse attend [+ stats]); returns out [B][Hq][dv] fp32."""
    B, Hq, _ = q.shape
    if out is None:
        out = torch.empty(B, Hq, cache.V.shape[3], dtype=torch.float32, device=q.device)
    cs = cache.c_struct()
    st = stats.c_struct() if stats is not None else None
    _check(lib().entmaxkv_decode(ctypes.byref(cs), _ptr(q), Hq, ctypes.byref(sel), ctypes.byref(attn), _ptr(out),
                                 None if st is None else ctypes.byref(st), _ptr(workspace), _stream(stream)))
    return out


def score_pages_into(cache: PagedCache, q, box=None, mu=None, sigma2=None, stream=None):
    """score_pages writing into caller buffers (modes from which buffers are given)."""
    modes = (EKV_SCORE_BOX if box is not None else 0) | (EKV_SCORE_GAUSS if mu is not None else 0)
    cs = cache.c_struct()
    _check(lib().entmaxkv_score_pages(ctypes.byref(cs), _ptr(q), int(q.shape[1]), modes, _ptr(box), _ptr(mu),
                                      _ptr(sigma2), None, _stream(stream)))


def select_into(cache: PagedCache, n_q_heads, sel: ekv_select_params, alpha, box, page_idx, n_sel, mu=None,
                sigma2=None, tau_hat=None, stream=None):
    cs = cache.c_struct()
    _check(lib().entmaxkv_select(ctypes.byref(cs), int(n_q_heads), _ptr(box), _ptr(mu), _ptr(sigma2),
                                 ctypes.byref(sel), float(alpha), _ptr(page_idx), _ptr(n_sel), int(page_idx.shape[2]),
                                 _ptr(tau_hat), None, _stream(stream)))


# ----------------------------------------------------------------------------- sequence sharding
def shard_workspace(cache: PagedCache, n_q_heads, sel: ekv_select_params, world: int):
    n = lib().entmaxkv_shard_workspace_size(ctypes.byref(cache.c_struct()), int(n_q_heads), ctypes.byref(sel),
                                            int(world))
    if n == 0:
        raise EkvError(EKV_ERR_INVALID_ARG, lib().entmaxkv_last_error().decode())
    return torch.empty(int(n), dtype=torch.uint8, device=cache.K.device)


def peer_buffer_size(cache: PagedCache, n_q_heads, sel: ekv_select_params, world: int) -> int:
    n = lib().entmaxkv_peer_buffer_size(ctypes.byref(cache.c_struct()), int(n_q_heads), ctypes.byref(sel), int(world))
    if n == 0:
        raise EkvError(EKV_ERR_INVALID_ARG, lib().entmaxkv_last_error().decode())
    return int(n)


def decode_sharded(cache: PagedCache, global_seq_lens, q, sel: ekv_select_params, attn: ekv_attn_params, comm,
                   workspace, out=None, stats: DecodeStats | None = None, stream=None, fixed_rounds=0):
    """One sequence-sharded decode step on this rank's local cache (include/entmaxkv.h).
    `comm` provides rank, world and either the collectives (callback mode: the library calls
    them back between its kernels) or `peers`, the W exchange-buffer pointers of the in-kernel
    collective mode (see paper_2605_21649_b200.sharding).  Returns out [B][Hq][dv] fp32 (replicated)."""
    B, Hq, _ = q.shape
    if out is None:
        out = torch.empty(B, Hq, cache.V.shape[3], dtype=torch.float32, device=q.device)
    s = stream if stream is not None else torch.cuda.current_stream(q.device)
    comm.bind(workspace, s)
    cm = ekv_comm(int(comm.rank), int(comm.world), comm.c_allreduce, comm.c_allgather, None, int(fixed_rounds))
    for i, p in enumerate(getattr(comm, "peers", None) or []):
        cm.peers[i] = int(p)
    cs = cache.c_struct()
    st = stats.c_struct() if stats is not None else None
    try:
        _check(lib().entmaxkv_decode_sharded(ctypes.byref(cs), _ptr(global_seq_lens), _ptr(q), Hq, ctypes.byref(sel),
                                             ctypes.byref(attn), ctypes.byref(cm), _ptr(out),
                                             None if st is None else ctypes.byref(st), _ptr(workspace),
                                             ctypes.c_void_p(s.cuda_stream)))
    finally:
        comm.unbind()
    if comm.error is not None:
        raise comm.error
    return out
