"""EntmaxKV sparse alpha-entmax decode step for B200 (sm_100a).

The compute path lives in ``libentmaxkv.so`` (C ABI, include/entmaxkv.h);
``binding`` is the ctypes layer over it and ``workload`` draws seeded
synthetic inputs.  Importing the package does not load the library; the first
call into ``binding`` does, and raises if it is missing (no CPU fallback).
"""
__all__ = ["binding", "workload"]
